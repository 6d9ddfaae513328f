// evox_kernels.cu -- sm_100a kernels of the PSO/CSO generation.
//
// Hot path: one fused kernel per PSO generation reads
// X, V and (unless the row's pbest copy is pending) P once, draws r1/r2 with
// Philox in registers, moves + clips, writes X', V' (and the pending P copy),
// evaluates f(X') from registers, applies the per-row tell and reduces the
// generation's argmin (warp -> CTA -> one atomicMin per CTA); the last CTA to
// finish publishes gbest.  20 B/element of HBM traffic per generation.
//
// Row engine geometry (a function of ld only, so every result is bitwise the
// same for every shard count, R-11):
//   * LPR lanes walk one row (LPR = 4 / 8 for ld <= 128 / 256, else 32); a warp holds
//     RPW = 32/LPR consecutive rows; or
//   * WPR = 8 warps (one CTA) share one row, each owning a contiguous segment
//     (ld > 4096).
// Lanes walk their segment in chunks of LPR float4 quads (one LDG.128/STG.128
// per lane per array per chunk), U chunks in flight.  The HBM stream is kept
// ahead of the loads with cp.async.bulk.prefetch.L2 (SASS UBLKPF): the next
// rows of the warp when they are short (mode A), or a sliding window of
// AHEAD quads inside long rows (mode B).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "evox_device.cuh"
#include "evox_internal.h"

namespace evox {

namespace {

#ifndef EVOX_U
#define EVOX_U 4
#endif
#ifndef EVOX_MINB
#define EVOX_MINB 2
#endif
#ifndef EVOX_AHEAD
#define EVOX_AHEAD 4  // mode-B prefetch window, in lane groups
#endif
#ifndef EVOX_PF
// L2 bulk-prefetch switches (measured): bit 0 mode A (a warp's next short
// rows: +2-4 points at dim <= 1000; on), bit 1 mode B (sliding window inside long rows:
// -13 points at dim 1e5; off), bit 2 CSO winner/loser rows of the next item (neutral; off),
// bit 3 the first rows of a PDL-launched generation (neutral; off).
#define EVOX_PF 1
#endif
constexpr int U = EVOX_U;          // max chunks in flight per lane group (register slots)
constexpr int WARPS = 8;           // warps per CTA (256 threads) in every geometry
constexpr long long MODE_A_MAX = 384;  // quads per warp-iteration prefetched whole (mode A)
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <int LPR_, int WPR_, int U_ = U, bool EFL_ = true>
struct Geom {
    static constexpr bool EFL = EFL_;             // evict-first loads (stores always are)
    static constexpr int LPR = LPR_;              // lanes per row segment
    static constexpr int WPR = WPR_;              // warps per row
    static constexpr int NU = U_ < U ? U_ : U;    // chunks in flight per lane group
    static constexpr int RPW = 32 / LPR_;         // rows per warp (WPR == 1)
    static constexpr int RPC = WPR_ == 1 ? WARPS * RPW : WARPS / WPR_;  // rows per CTA pass
    static constexpr int GROUP = LPR_ * NU;       // quads per lane-group iteration
};

// Row segment [qb, qe) of warp `wr` (of WPR) over NQ quads.
__device__ __forceinline__ void row_segment(long long NQ, int wpr, int wr, long long& qb,
                                            long long& qe) {
    const long long seg = (NQ + wpr - 1) / wpr;
    qb = (long long)wr * seg;
    if (qb > NQ) qb = NQ;
    qe = qb + seg < NQ ? qb + seg : NQ;
}

__device__ __forceinline__ float4 bound4(const float* b, float b0, int uniform, long long q) {
    if (uniform) return make_float4(b0, b0, b0, b0);
    return __ldg(reinterpret_cast<const float4*>(b) + q);
}
// Compile-time specialisation: uniform bounds feed FMNMX straight from the
// constant bank; per-column bounds are two L1-resident LDG.128 per quad.
template <bool UNI>
__device__ __forceinline__ float4 bound4t(const float* b, float b0, long long q) {
    if constexpr (UNI) return make_float4(b0, b0, b0, b0);
    else return __ldg(reinterpret_cast<const float4*>(b) + q);
}

__device__ __forceinline__ float clipf(float x, float lo, float hi) {
    return fminf(fmaxf(x, lo), hi);
}

// Bulk L2 prefetch (Hopper+ cp.async.bulk.prefetch): pulls a whole run of a row
// from HBM into L2 with one instruction, so later LDGs of it hit L2.
__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
    if (bytes > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)bytes)
                     : "memory");
}

// The PSO velocity/position update of one element (R-1, R-4), exact op order.
// c1 = phi_p r1 and c2 = phi_g r2 arrive already scaled (scaled_u24).
__device__ __forceinline__ void pso_elem(float& x, float& v, float p, float g, float c1, float c2,
                                         float w, float lo, float hi) {
    const float a = __fsub_rn(p, x);
    const float b = __fsub_rn(g, x);
    const float vn = __fmaf_rn(c2, b, __fmaf_rn(c1, a, __fmul_rn(w, v)));
    x = clipf(__fadd_rn(x, vn), lo, hi);
    v = vn;
}

__device__ __forceinline__ void zero_pad(float4& x, float4& v, long long q, long long D) {
    if (4 * q + 3 >= D) {  // padding columns stay 0
        const long long j0 = 4 * q;
        if (j0 + 1 >= D) { x.y = 0.f; v.y = 0.f; }
        if (j0 + 2 >= D) { x.z = 0.f; v.z = 0.f; }
        if (j0 + 3 >= D) { x.w = 0.f; v.w = 0.f; }
    }
}

// Griewank column constants h_j = 1/(2 pi sqrt(j+1)) for one CTA, computed in
// fp64 and rounded once (geometries with ld <= HTAB; else computed per element).
constexpr int HTAB = 4096;
template <int P, class G>
struct HTable {
    __device__ __forceinline__ static const float* fill(float*, long long) { return nullptr; }
};
template <class G>
struct HTable<GRIEWANK, G> {
    __device__ __forceinline__ static const float* fill(float* sh, long long ld) {
        if constexpr (G::WPR > 1) {
            return nullptr;
        } else {
            if (ld > HTAB) return nullptr;
            for (long long j = threadIdx.x; j < ld; j += blockDim.x)
                sh[j] = (float)(0.15915494309189534 / sqrt((double)(j + 1)));
            __syncthreads();
            return sh;
        }
    }
};
template <int P>
struct HStore {
    float v[1];
};
template <>
struct HStore<GRIEWANK> {
    float v[HTAB];
};

// Programmatic dependent launch (PDL): a generation kernel lets the next one be
// scheduled as soon as its CTAs start retiring; the next one prefetches its
// first rows into L2 and then waits for the full completion (and memory
// flush) of this grid before touching anything this generation wrote.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// First-row L2 prefetch of a warp (X and V only: whether P is needed depends
// on imp, which the previous generation is still writing).
template <class G>
__device__ __forceinline__ void prefetch_first_rows(const float* X, const float* V, long long rows,
                                                    long long ld, long long wfirst, long long qb,
                                                    long long qe) {
    if (!(EVOX_PF & 8) || lane_id() != 0 || wfirst >= rows) return;
    const long long nr = rows - wfirst < G::RPW ? rows - wfirst : G::RPW;
    const long long o = wfirst * ld * 4 + qb * 16;
    long long bytes = G::WPR == 1 ? nr * ld * 4 : (qe - qb) * 16;
    if (bytes > 64 * 1024) bytes = 64 * 1024;  // long rows: the window prefetcher takes over
    prefetch_l2(reinterpret_cast<const char*>(X) + o, bytes);
    prefetch_l2(reinterpret_cast<const char*>(V) + o, bytes);
}

struct NoPrefetch {
    __device__ __forceinline__ void operator()(long long) {}
};

// ---------------------------------------------------------------------------
// Row engine: walks one row segment [qb, qe) chunk by chunk; `mv` loads/moves a
// quad and returns the value to evaluate; folds the fitness (with the
// Rosenbrock cross-quad halo).  Every lane of the warp executes every chunk
// iteration (qb/qe are warp-uniform); lanes of an absent row (`row_ok` false)
// do no memory work.  `pf(base)` is called by the warp at each group start.
template <int P, class G, class Mover, class PF>
__device__ __forceinline__ void walk_segment(Mover& mv, long long qb, long long qe, long long D,
                                             bool row_ok, Fit<P>& acc, float& head_x,
                                             float& tail_x, bool& tail_valid, PF& pf,
                                             const float* htab = nullptr) {
    const int sl = lane_id() & (G::LPR - 1);
    float pend_x = 0.0f;
    bool pend = false;  // last sub-lane: x_{4q+3} waiting for x_{4q+4} of the next chunk
    head_x = 0.0f;
    tail_valid = false;
    tail_x = 0.0f;
    for (long long base = qb; base < qe; base += G::GROUP) {
        pf(base);
#pragma unroll
        for (int u = 0; u < G::NU; ++u) {
            const long long q = base + G::LPR * u + sl;
            if (row_ok && q < qe) mv.template load<G::EFL>(u, q);
        }
#pragma unroll
        for (int u = 0; u < G::NU; ++u) {
            const long long cb = base + G::LPR * u;  // first quad of this chunk
            if (cb >= qe) break;                     // warp-uniform
            const long long q = cb + sl;
            const bool valid = row_ok && q < qe;
            float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid) {
                xn = mv.step(u, q);
                fit_quad<P>(acc, xn, 4 * q, D, htab);
            }
            if constexpr (P == ROSENBROCK) {
                const float nb = __shfl_down_sync(FULL, xn.x, 1, G::LPR);
                const float f0 = __shfl_sync(FULL, xn.x, 0, G::LPR);
                if (cb == qb) head_x = f0;
                if (sl == G::LPR - 1 && pend) {
                    acc.pair(pend_x, f0);
                    pend = false;
                }
                if (valid) {
                    const bool has_next = 4 * q + 4 < D;
                    if (q + 1 < qe) {
                        if (sl < G::LPR - 1) {
                            if (has_next) acc.pair(xn.w, nb);
                        } else {
                            pend = has_next;
                            pend_x = xn.w;
                        }
                    } else {  // last quad of the segment: successor is the next segment's head
                        tail_valid = has_next;
                        tail_x = xn.w;
                    }
                }
            }
        }
    }
}

// Reduce a row's fitness over its lanes (xor butterfly of width LPR) and, for
// WPR > 1, over the row's warps in fixed order through shared memory.  Returns
// f in sub-lane 0 (WPR == 1) / thread 0 (WPR > 1).
template <int P, class G>
__device__ __forceinline__ float reduce_row(Fit<P> acc, long long D, float head_x, float tail_x,
                                            bool tail_valid, Fit<P>* sh_acc, float* sh_head) {
    const int lane = lane_id();
    if constexpr (G::WPR > 1 && P == ROSENBROCK) {
        const int wr = threadIdx.x >> 5;
        if (lane == 0) sh_head[wr] = head_x;
        __syncthreads();
        if (tail_valid && wr + 1 < G::WPR) acc.pair(tail_x, sh_head[wr + 1]);
    }
#pragma unroll
    for (int m = G::LPR / 2; m >= 1; m >>= 1) {
        Fit<P> o = acc;
        o.shfl_xor(m, G::LPR);
        acc.combine(o);
    }
    if constexpr (G::WPR == 1) {
        return acc.finish(D);
    } else {
        const int wr = threadIdx.x >> 5;
        if (lane == 0) sh_acc[wr] = acc;
        __syncthreads();
        float f = 0.0f;
        if (threadIdx.x == 0) {
            Fit<P> t = sh_acc[0];
#pragma unroll 1
            for (int k = 1; k < G::WPR; ++k) t.combine(sh_acc[k]);
            f = t.finish(D);
        }
        __syncthreads();  // sh_acc / sh_head reusable for the next row
        return f;
    }
}

// Thread-to-row mapping of a geometry.
template <class G>
struct RowMap {
    long long first, stride;  // this thread's first row and the row stride per iteration
    long long wfirst;         // the warp's first row (WPR == 1: rows wfirst..wfirst+RPW-1)
    int sl;                   // sub-lane within the row group
    bool leader;              // the thread that owns the row's scalar results
    long long qb, qe;         // this warp's segment of the row
    __device__ __forceinline__ RowMap(long long NQ) {
        const int wid = threadIdx.x >> 5, lane = lane_id();
        sl = lane & (G::LPR - 1);
        if constexpr (G::WPR == 1) {
            wfirst = ((long long)blockIdx.x * WARPS + wid) * G::RPW;
            first = wfirst + lane / G::LPR;
            stride = (long long)gridDim.x * G::RPC;
            leader = sl == 0;
            qb = 0;
            qe = NQ;
        } else {
            wfirst = (long long)blockIdx.x * (WARPS / G::WPR) + wid / G::WPR;
            first = wfirst;
            stride = (long long)gridDim.x * G::RPC;
            leader = (threadIdx.x % (G::WPR * 32)) == 0;
            row_segment(NQ, G::WPR, wid % G::WPR, qb, qe);
        }
    }
};

// ---------------------------------------------------------------------------
// Movers
struct MoverEval {
    const float4* Xr;
    float4 x[U];
    template <bool EF>
    __device__ __forceinline__ void load(int u, long long q) { x[u] = ld_stream<EF>(Xr + q); }
    __device__ __forceinline__ float4 step(int u, long long) { return x[u]; }
};

// PSO move of one row (A1, A3, A4, lazy A5).  Holds a reference to the kernel
// parameter block (resolved to constant-bank operands once inlined: the
// Philox round keys, w, phi*2^-24 and the bounds feed instructions directly).
template <bool UNI, bool G_COHERENT = false>
struct MoverPso {
    const PsoArgs& a;
    float4* Xr;
    float4* Vr;
    float4* Pr;
    uint32_t row_g;  // global row (Philox counter word 1)
    uint32_t t;      // generation of the source population (counter word 2)
    bool pend;       // pbest copy pending: P := X_t, P not read
    float4 x[U], v[U], p[U];
    __device__ __forceinline__ MoverPso(const PsoArgs& a_, long long row, uint32_t t_, bool pend_)
        : a(a_) {
        Xr = reinterpret_cast<float4*>(a.X + row * a.ld);
        Vr = reinterpret_cast<float4*>(a.V + row * a.ld);
        Pr = reinterpret_cast<float4*>(a.P + row * a.ld);
        row_g = (uint32_t)(a.row0 + row);
        t = t_;
        pend = pend_;
    }
    template <bool EF>
    __device__ __forceinline__ void load(int u, long long q) {
        x[u] = ld_stream<EF>(Xr + q);
        v[u] = ld_stream<EF>(Vr + q);
        if (!pend) p[u] = ld_stream<EF>(Pr + q);
    }
    __device__ __forceinline__ float4 step(int u, long long q) {
        const float4 xo = x[u];
        const float4 pb = pend ? xo : p[u];
        if (pend) st_stream(Pr + q, xo);
        // G is read-only for a generation kernel (non-coherent path); the
        // persistent small-population kernel rewrites it between generations.
        const float4 g = G_COHERENT ? __ldcg(reinterpret_cast<const float4*>(a.G) + q)
                                    : __ldg(reinterpret_cast<const float4*>(a.G) + q);
        const float4 lo = bound4t<UNI>(a.lb, a.lb0, q);
        const float4 hi = bound4t<UNI>(a.ub, a.ub0, q);
        const uint4 b1 = Philox::run(make_uint4((uint32_t)q, row_g, t, 2u), a.rk);
        const uint4 b2 = Philox::run(make_uint4((uint32_t)q, row_g, t, 3u), a.rk);
        float4 xn = xo, vn = v[u];
        const float w = a.w, cp = a.cp, cg = a.cg;
        pso_elem(xn.x, vn.x, pb.x, g.x, scaled_u24(b1.x, cp), scaled_u24(b2.x, cg), w, lo.x, hi.x);
        pso_elem(xn.y, vn.y, pb.y, g.y, scaled_u24(b1.y, cp), scaled_u24(b2.y, cg), w, lo.y, hi.y);
        pso_elem(xn.z, vn.z, pb.z, g.z, scaled_u24(b1.z, cp), scaled_u24(b2.z, cg), w, lo.z, hi.z);
        pso_elem(xn.w, vn.w, pb.w, g.w, scaled_u24(b1.w, cp), scaled_u24(b2.w, cg), w, lo.w, hi.w);
        zero_pad(xn, vn, q, a.D);
        st_stream(Xr + q, xn);
        st_stream(Vr + q, vn);
        return xn;
    }
};

// Mode-B prefetcher (long row segments): keeps a window of AHEAD quads of
// X, V and (unless the pbest copy is pending) P in flight ahead of the
// loads, crossing into the warp's next row.  Lane 0 issues; the cursor is
// relative to the current row segment (c in [0, 2 seg)).
struct WindowPrefetch {
    const char* X;
    const char* V;
    const char* P;
    long long ld_bytes, qb, seg, ahead;
    long long row, nxt;  // current and next row of the warp (nxt >= rows: none)
    bool pend_cur, pend_nxt, on;
    long long c;         // next unprefetched quad, relative to qb of the current row
    __device__ __forceinline__ void issue(long long r, long long q0, long long n, bool pend) {
        const long long o = r * ld_bytes + (qb + q0) * 16;
        prefetch_l2(X + o, n * 16);
        prefetch_l2(V + o, n * 16);
        if (!pend) prefetch_l2(P + o, n * 16);
    }
    __device__ __forceinline__ void operator()(long long base) {
        if (!on) return;
        long long target = (base - qb) + ahead;
        const long long lim = nxt >= 0 ? 2 * seg : seg;
        if (target > lim) target = lim;
        if (c >= target) return;
        if (c < seg) {
            const long long e = target < seg ? target : seg;
            issue(row, c, e - c, pend_cur);
            c = e;
        }
        if (c < target) {  // into the next row
            issue(nxt, c - seg, target - c, pend_nxt);
            c = target;
        }
    }
};

// ---------------------------------------------------------------------------
// Grid-level argmin + finalize (A12/A13).
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long k) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const unsigned long long o = __shfl_xor_sync(FULL, k, m);
        k = o < k ? o : k;
    }
    return k;
}

// Every thread calls it after its last row; returns true in the (whole) last
// CTA to finish, with the generation's min key in *out_key.
__device__ __forceinline__ bool grid_argmin(Ctl* ctl, unsigned long long my_key,
                                            unsigned long long* out_key, bool sys = false) {
    __shared__ unsigned long long sh_k[32];
    __shared__ int sh_last;
    const int lane = lane_id(), wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    my_key = warp_min_u64(my_key);
    if (lane == 0) sh_k[wid] = my_key;
    // this thread's population stores visible device-wide (system-wide when peers
    // on other GPUs read this shard in the next generation)
    if (sys) __threadfence_system();
    else __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = sh_k[0];
        for (int i = 1; i < nw; ++i) k = sh_k[i] < k ? sh_k[i] : k;
        if (k != ~0ull) atomicMin(&ctl->gen_key, k);
        __threadfence();
        const unsigned int prev = atomicAdd(&ctl->ticket, 1u);
        sh_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!sh_last) return false;
    __threadfence();
    *out_key = atomicAdd(&ctl->gen_key, 0ull);
    return true;
}

// Peer-memory exchange primitives (system scope: the mailboxes of other ranks
// are NVLink peer memory mapped into this address space).
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The last CTA's winner record -> every rank's mailbox slot[par][rank]; wait for
// the world records of this generation; strict gbest selection (A13, fused).
// Every rank selects from the same world records: identical G on all ranks.
__device__ void peer_exchange(const PsoArgs& a, unsigned long long key, unsigned long long t_new) {
    __shared__ int sh_w, sh_better;
    __shared__ unsigned long long sh_key;
    Ctl* ctl = a.ctl;
    const long long NQ = a.ld >> 2;
    const int par = (int)(t_new & 1);
    const unsigned long long flag = t_new + 1;  // mailboxes start zeroed: 0 = nothing yet
    const bool any = key != ~0ull;
    const long long grow = (long long)(uint32_t)(key & 0xffffffffu);
    const float4* src = reinterpret_cast<const float4*>(a.X + (any ? grow - a.row0 : 0) * a.ld);
    const long long my_off = ((long long)par * a.world + a.rank) * a.mb_slot;
    for (long long q = threadIdx.x; q < NQ; q += blockDim.x) {
        const float4 v = any ? __ldcg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int p = 0; p < a.world; ++p)
            reinterpret_cast<float4*>(a.mbox[p] + my_off + 16)[q] = v;
    }
    if (threadIdx.x == 0)
        for (int p = 0; p < a.world; ++p)
            *reinterpret_cast<unsigned long long*>(a.mbox[p] + my_off + 8) = key;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int p = 0; p < a.world; ++p)
            st_release_sys(reinterpret_cast<unsigned long long*>(a.mbox[p] + my_off), flag);
        // wait for every rank's record of this generation in our own mailbox
        const unsigned long long t0 = globaltimer_ns();
        unsigned long long kmin = ~0ull;
        int w = -1;
        for (int r = 0; r < a.world; ++r) {
            const unsigned char* slot = a.mbox[a.rank] + ((long long)par * a.world + r) * a.mb_slot;
            while (ld_acquire_sys(reinterpret_cast<const unsigned long long*>(slot)) != flag) {
                if (globaltimer_ns() - t0 > a.peer_timeout_ns) {
                    ctl->err = 1;
                    break;
                }
                __nanosleep(256);
            }
            const unsigned long long kr = __ldcg(reinterpret_cast<const unsigned long long*>(slot + 8));
            if (kr < kmin) { kmin = kr; w = r; }
        }
        const bool ok = kmin != ~0ull;
        const float fmin = ok ? unord_f32((uint32_t)(kmin >> 32)) : __int_as_float(0x7f800000);
        sh_key = kmin;
        sh_w = w;
        sh_better = ok && fmin < ctl->gf;  // strict improvement (R-5)
    }
    __syncthreads();
    if (sh_better) {
        const float4* wr = reinterpret_cast<const float4*>(
            a.mbox[a.rank] + ((long long)par * a.world + sh_w) * a.mb_slot + 16);
        float4* G = reinterpret_cast<float4*>(a.G);
        for (long long q = threadIdx.x; q < NQ; q += blockDim.x) G[q] = __ldcg(wr + q);
    }
    if (threadIdx.x == 0) {
        const unsigned long long k = sh_key;
        const float fmin = k != ~0ull ? unord_f32((uint32_t)(k >> 32)) : __int_as_float(0x7f800000);
        if (sh_better) {
            ctl->gf = fmin;
            ctl->gidx = (long long)(uint32_t)(k & 0xffffffffu);
        }
        ctl->hist[t_new] = fmin;
    }
}

// End-of-generation barrier of a row-sharded population whose shards read each
// other (DE donors, CSO cross-shard pairs): publish this rank's min key in every
// rank's mailbox (slot[par][rank] = {flag, key}), wait for all, return the
// global min.  No rank starts generation t+1 (which may overwrite rows peers
// read in generation t) before every rank finished generation t.  One thread.
__device__ unsigned long long peer_min(unsigned char* const* mbox, int rank, int world,
                                       unsigned long long timeout_ns, Ctl* ctl,
                                       unsigned long long key, unsigned long long t_new) {
    const int par = (int)(t_new & 1);
    const unsigned long long flag = t_new + 1;
    const long long my = ((long long)par * world + rank) * 16;
    for (int w = 0; w < world; ++w) *reinterpret_cast<unsigned long long*>(mbox[w] + my + 8) = key;
    __threadfence_system();
    for (int w = 0; w < world; ++w)
        st_release_sys(reinterpret_cast<unsigned long long*>(mbox[w] + my), flag);
    unsigned long long kmin = ~0ull;
    const unsigned long long t0 = globaltimer_ns();
    for (int w = 0; w < world; ++w) {
        const unsigned char* slot = mbox[rank] + ((long long)par * world + w) * 16;
        while (ld_acquire_sys(reinterpret_cast<const unsigned long long*>(slot)) != flag) {
            if (globaltimer_ns() - t0 > timeout_ns) {
                ctl->err = 1;
                break;
            }
            __nanosleep(256);
        }
        const unsigned long long kw = __ldcg(reinterpret_cast<const unsigned long long*>(slot + 8));
        kmin = kw < kmin ? kw : kmin;
    }
    return kmin;
}

// In the last CTA: gbest update (strict, R-5), hist, or the winner record for
// the exchange.  `t_new` is the index of the population just evaluated.
__device__ void pso_finalize(const PsoArgs& a, unsigned long long key, unsigned long long t_new) {
    Ctl* ctl = a.ctl;
    const long long NQ = a.ld >> 2;
    const bool any = key != ~0ull;
    const long long grow = (long long)(uint32_t)(key & 0xffffffffu);
    const float fmin = any ? unord_f32((uint32_t)(key >> 32)) : __int_as_float(0x7f800000);
    if (a.peer) {
        peer_exchange(a, key, t_new);
    } else if (a.exchange) {
        // winner record {u64 key; u32 pad[2]; f32 row[ld]} into this rank's slot
        unsigned char* rec = a.rec + (long long)a.rank * a.rec_stride;
        const float4* src = reinterpret_cast<const float4*>(a.X + (any ? grow - a.row0 : 0) * a.ld);
        float4* dst = reinterpret_cast<float4*>(rec + 16);
        for (long long q = threadIdx.x; q < NQ; q += blockDim.x)
            dst[q] = any ? __ldcg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (threadIdx.x == 0) *reinterpret_cast<unsigned long long*>(rec) = key;
    } else {
        __shared__ int sh_better;
        if (threadIdx.x == 0) sh_better = any && fmin < ctl->gf;  // strict improvement
        __syncthreads();
        const bool better = sh_better != 0;
        if (better) {
            const float4* src = reinterpret_cast<const float4*>(a.X + (grow - a.row0) * a.ld);
            float4* G = reinterpret_cast<float4*>(a.G);
            for (long long q = threadIdx.x; q < NQ; q += blockDim.x) G[q] = __ldcg(src + q);
        }
        if (threadIdx.x == 0) {
            if (better) {
                ctl->gf = fmin;
                ctl->gidx = grow;
            }
            ctl->hist[t_new] = fmin;
        }
    }
    if (threadIdx.x == 0) {
        ctl->gen_key = ~0ull;
        ctl->ticket = 0u;
        ctl->t = t_new;
    }
}

// ---------------------------------------------------------------------------
// Kernels

// A2: X0 = fmaf(u, ub-lb, lb) (Philox tag 0, t = 0), V0 = 0 (+ P0 = X0 for PSO).
__device__ __forceinline__ void init_population(float* X, float* V, float* P, long long rows,
                                                long long row0, long long D, long long ld,
                                                const float* lb, const float* ub, float lb0,
                                                float ub0, int uniform, const PhiloxKey& rk) {
    const long long NQ = ld >> 2;
    const long long total = rows * NQ;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / NQ, q = i - r * NQ;
        const uint4 b = Philox::run(make_uint4((uint32_t)q, (uint32_t)(row0 + r), 0u, 0u), rk);
        const float4 lo = bound4(lb, lb0, uniform, q);
        const float4 hi = bound4(ub, ub0, uniform, q);
        float4 x, v = make_float4(0.f, 0.f, 0.f, 0.f);
        x.x = __fmaf_rn(u24(b.x), __fsub_rn(hi.x, lo.x), lo.x);
        x.y = __fmaf_rn(u24(b.y), __fsub_rn(hi.y, lo.y), lo.y);
        x.z = __fmaf_rn(u24(b.z), __fsub_rn(hi.z, lo.z), lo.z);
        x.w = __fmaf_rn(u24(b.w), __fsub_rn(hi.w, lo.w), lo.w);
        zero_pad(x, v, q, D);
        reinterpret_cast<float4*>(X)[i] = x;
        reinterpret_cast<float4*>(V)[i] = v;
        if (P) reinterpret_cast<float4*>(P)[i] = x;
    }
}

__global__ void k_pso_init(PsoArgs a) {
    init_population(a.X, a.V, a.P, a.rows, a.row0, a.D, a.ld, a.lb, a.ub, a.lb0, a.ub0,
                    a.uniform_bounds, a.rk);
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        a.pf[r] = __int_as_float(0x7f800000);
        a.f[r] = __int_as_float(0x7f800000);
        a.imp[r] = 0;
    }
}

// evox_eval: fit[r] = f(X[r]).
template <int P, class G>
__global__ void __launch_bounds__(256) k_eval(const float* __restrict__ X, long long rows,
                                              long long D, long long ld,
                                              float* __restrict__ fit) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P> sh_h;
    const float* htab = HTable<P, G>::fill(sh_h.v, ld);
    const RowMap<G> m(ld >> 2);
    NoPrefetch pf;
    for (long long it = 0;; ++it) {
        const long long wrow = m.wfirst + it * m.stride;
        if (wrow >= rows) break;  // warp-uniform (CTA-uniform for WPR > 1)
        const long long row = m.first + it * m.stride;
        const bool ok = row < rows;
        MoverEval mv;
        mv.Xr = reinterpret_cast<const float4*>(X + (ok ? row : 0) * ld);
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P, G>(mv, m.qb, m.qe, D, ok, acc, hx, tx, tv, pf, htab);
        const float f = reduce_row<P, G>(acc, D, hx, tx, tv, sh_acc, sh_head);
        if (m.leader && ok) fit[row] = f;
    }
}

// Fused PSO generation: lazy pbest + move + clip + evaluate + tell + argmin.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, EVOX_MINB) k_pso_gen(PsoArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P> sh_h;
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    const int lane = lane_id();
    prefetch_first_rows<G>(a.X, a.V, a.rows, a.ld, m.wfirst, m.qb, m.qe);
    pdl_wait();               // the previous generation (G, imp, pf, t) is complete
    pdl_launch_dependents();  // the next generation may be scheduled as our CTAs retire
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const long long seg = m.qe - m.qb;
    // prefetch mode: A = the warp's whole next rows (short rows), B = sliding window
    const bool mode_a = seg * G::RPW <= MODE_A_MAX;
    WindowPrefetch wp;
    wp.X = reinterpret_cast<const char*>(a.X);
    wp.V = reinterpret_cast<const char*>(a.V);
    wp.P = reinterpret_cast<const char*>(a.P);
    wp.ld_bytes = a.ld * 4;
    wp.qb = m.qb;
    wp.seg = seg;
    wp.ahead = seg < EVOX_AHEAD * G::GROUP ? seg : EVOX_AHEAD * G::GROUP;
    wp.on = !mode_a && lane == 0 && (EVOX_PF & 2);
    wp.c = 0;
    unsigned long long best = ~0ull;
    // pbest-pending flags one and two iterations ahead (imp[r] is rewritten only
    // by the thread group that owns row r, later in this kernel, so these reads
    // see the previous generation's decisions).
    long long row = m.first;
    bool pend_cur = row < a.rows ? a.imp[row] != 0 : true;
    bool pend_nxt = row + m.stride < a.rows ? a.imp[row + m.stride] != 0 : true;
    for (long long it = 0;; ++it, row += m.stride) {
        const long long wrow = m.wfirst + it * m.stride;
        if (wrow >= a.rows) break;  // warp-uniform (CTA-uniform for WPR > 1)
        const bool ok = row < a.rows;
        const long long nxt = row + m.stride, nn = nxt + m.stride;
        const bool nxt_ok = nxt < a.rows;
        if (mode_a && (EVOX_PF & 1)) {
            // the warp's next rows, HBM -> L2 now (X, V contiguous; P per row unless pending)
            const long long wn = wrow + m.stride;
            if (lane == 0 && wn < a.rows) {
                long long nr = a.rows - wn < G::RPW ? a.rows - wn : G::RPW;
                const long long o = wn * a.ld * 4 + m.qb * 16;
                const long long bytes = G::WPR == 1 ? nr * a.ld * 4 : seg * 16;
                prefetch_l2(reinterpret_cast<const char*>(a.X) + o, bytes);
                prefetch_l2(reinterpret_cast<const char*>(a.V) + o, bytes);
            }
            if (m.sl == 0 && nxt_ok && !pend_nxt)
                prefetch_l2(reinterpret_cast<const char*>(a.P) + nxt * a.ld * 4 + m.qb * 16,
                            seg * 16);
        } else if (!mode_a) {
            wp.row = row;
            wp.nxt = nxt_ok ? nxt : -1;
            wp.pend_cur = pend_cur;
            wp.pend_nxt = pend_nxt;
        }
        const bool pend_nn = nn < a.rows ? a.imp[nn] != 0 : true;
        float pf_old = 0.0f;
        if (m.leader && ok) pf_old = a.pf[row];
        MoverPso<UNI> mv(a, ok ? row : 0, (uint32_t)t, pend_cur);
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P, G>(mv, m.qb, m.qe, a.D, ok, acc, hx, tx, tv, wp, htab);
        const float f = reduce_row<P, G>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
        if (m.leader && ok) {
            // per-row tell (A11): strict improvement, NaN never improves
            const bool imp = f < pf_old;
            a.f[row] = f;
            a.imp[row] = imp ? 1 : 0;
            if (imp) a.pf[row] = f;
            const unsigned long long k = make_key(f, a.row0 + row);
            best = k < best ? k : best;
        }
        pend_cur = pend_nxt;
        pend_nxt = pend_nn;
        wp.c = wp.c > seg ? wp.c - seg : 0;
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key)) pso_finalize(a, key, t + 1);
}


// Persistent single-CTA PSO for tiny populations (latency-bound, e.g. C1:
// 100 x 10): all n generations in one launch, a CTA barrier instead of the
// grid-wide argmin.  Per-row arithmetic, reduction order and decisions are
// those of k_pso_gen, so the trajectory is bitwise identical.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256) k_pso_run_small(PsoArgs a, long long n_gens) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P> sh_h;
    __shared__ unsigned long long sh_k[WARPS];
    __shared__ int sh_better;
    __shared__ long long sh_row;
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    Ctl* ctl = a.ctl;
    unsigned long long t = ctl->t;
    float gf = ctl->gf;
    long long gidx = ctl->gidx;
    NoPrefetch pf;
    for (long long g = 0; g < n_gens; ++g) {
        unsigned long long best = ~0ull;
        for (long long it = 0;; ++it) {
            const long long wrow = m.wfirst + it * m.stride;
            if (wrow >= a.rows) break;
            const long long row = m.first + it * m.stride;
            const bool ok = row < a.rows;
            const bool pend = ok ? a.imp[row] != 0 : true;
            float pf_old = 0.0f;
            if (m.leader && ok) pf_old = a.pf[row];
            MoverPso<UNI, true> mv(a, ok ? row : 0, (uint32_t)t, pend);
            Fit<P> acc;
            float hx, tx;
            bool tv;
            walk_segment<P, G>(mv, m.qb, m.qe, a.D, ok, acc, hx, tx, tv, pf, htab);
            const float f = reduce_row<P, G>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
            if (m.leader && ok) {
                const bool imp = f < pf_old;
                a.f[row] = f;
                a.imp[row] = imp ? 1 : 0;
                if (imp) a.pf[row] = f;
                const unsigned long long k = make_key(f, a.row0 + row);
                best = k < best ? k : best;
            }
        }
        best = warp_min_u64(best);
        if (lane == 0) sh_k[wid] = best;
        __syncthreads();  // also orders this generation's X stores before the G copy
        if (threadIdx.x == 0) {
            unsigned long long k = sh_k[0];
            for (int i = 1; i < WARPS; ++i) k = sh_k[i] < k ? sh_k[i] : k;
            const bool any = k != ~0ull;
            const float fmin = any ? unord_f32((uint32_t)(k >> 32)) : __int_as_float(0x7f800000);
            const bool better = any && fmin < gf;  // strict improvement
            sh_better = better;
            sh_row = (long long)(uint32_t)(k & 0xffffffffu) - a.row0;
            if (better) {
                gf = fmin;
                gidx = (long long)(uint32_t)(k & 0xffffffffu);
            }
            ctl->hist[t + 1] = fmin;
        }
        __syncthreads();
        if (sh_better) {
            const float4* src = reinterpret_cast<const float4*>(a.X + sh_row * a.ld);
            float4* Gd = reinterpret_cast<float4*>(a.G);
            for (long long q = threadIdx.x; q < (a.ld >> 2); q += blockDim.x) Gd[q] = __ldcg(src + q);
        }
        __syncthreads();
        ++t;
    }
    if (threadIdx.x == 0) {
        ctl->t = t;
        ctl->gf = gf;
        ctl->gidx = gidx;
    }
}

// ---------------------------------------------------------------------------
// TMA-staged fused PSO generation (warp-per-row geometry, ld <= 4096).
// Each warp owns a 2-stage shared-memory ring of {X, V, P} x 128 quads (one
// lane group).  Lane 0 fills it with cp.async.bulk (1-D TMA, SASS UBLKCP)
// completing on a per-stage mbarrier: while the warp computes group g from
// shared memory, group g+1 (possibly the first group of the warp's next row)
// is in flight -- no registers held by in-flight loads, and the 4 chunks of a
// group are still computed straight-line (cross-chunk Philox ILP).  Stores go
// straight from registers (evict-first).  Same arithmetic, reduction tree and
// decisions as k_pso_gen: bitwise identical (tested).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

constexpr int TMA_GQ = 32 * U;  // quads per group (= G32::GROUP)
struct TmaStage {
    float4 x[TMA_GQ], v[TMA_GQ], p[TMA_GQ];
};
constexpr size_t TMA_SMEM = sizeof(TmaStage) * 2 * WARPS;  // 96 KB per CTA

template <int P, bool UNI>
__global__ void __launch_bounds__(256, EVOX_MINB) k_pso_gen_tma(PsoArgs a) {
    using G = Geom<32, 1>;  // the warp-per-row geometry (G32)
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    __shared__ __align__(8) uint64_t bars[WARPS][2];
    __shared__ Fit<P> sh_acc[1];
    __shared__ float sh_head[1];
    __shared__ __align__(16) HStore<P> sh_h;
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    TmaStage* stg = reinterpret_cast<TmaStage*>(dyn_smem) + 2 * wid;
    uint64_t* bar = bars[wid];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    pdl_launch_dependents();
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const long long NQ = a.ld >> 2;
    const long long NG = (NQ + TMA_GQ - 1) / TMA_GQ;  // groups per row
    const long long n_it = m.wfirst < a.rows ? (a.rows - 1 - m.wfirst) / m.stride + 1 : 0;
    const long long total = n_it * NG;
    const float4* X4 = reinterpret_cast<const float4*>(a.X);
    const float4* V4 = reinterpret_cast<const float4*>(a.V);
    const float4* P4 = reinterpret_cast<const float4*>(a.P);
    // pbest-pending flags of the current row and the next two rows of the warp
    long long row = m.first;
    bool pend[3];
    pend[0] = row < a.rows ? a.imp[row] != 0 : true;
    pend[1] = row + m.stride < a.rows ? a.imp[row + m.stride] != 0 : true;
    pend[2] = row + 2 * m.stride < a.rows ? a.imp[row + 2 * m.stride] != 0 : true;
    // lane 0: put group g of the warp's stream in flight (it_cur = current row iteration)
    auto issue = [&](long long g, long long it_cur) {
        const long long it = g / NG, gg = g - it * NG;
        const long long r = m.first + it * m.stride;
        const long long q0 = gg * TMA_GQ;
        const long long nq = NQ - q0 < TMA_GQ ? NQ - q0 : TMA_GQ;
        const int st = (int)(g & 1);
        const long long d = it - it_cur;
        const bool pd = d == 0 ? pend[0] : (d == 1 ? pend[1] : pend[2]);
        const uint32_t bytes = (uint32_t)(nq * 16);
        fence_proxy_async_smem();  // the warp's generic reads of this stage are done
        mbar_expect_tx(&bar[st], bytes * (pd ? 2u : 3u));
        const long long o = r * NQ + q0;
        tma_load_1d(stg[st].x, X4 + o, bytes, &bar[st]);
        tma_load_1d(stg[st].v, V4 + o, bytes, &bar[st]);
        if (!pd) tma_load_1d(stg[st].p, P4 + o, bytes, &bar[st]);
    };
    if (lane == 0 && total > 0) issue(0, 0);
    float pf_old = 0.0f;
    if (lane == 0 && row < a.rows) pf_old = a.pf[row];
    Fit<P> acc;
    float pend_x = 0.0f, head_x = 0.0f;
    bool hpend = false;
    unsigned long long best = ~0ull;
    const float w = a.w, cp = a.cp, cg = a.cg;
    long long it = 0, gg = 0;
    for (long long g = 0; g < total; ++g) {
        if (lane == 0 && g + 1 < total) issue(g + 1, it);  // stage (g+1)&1 was freed by g-1
        const int st = (int)(g & 1);
        mbar_wait(&bar[st], (uint32_t)((g >> 1) & 1));
        const bool ok = row < a.rows;
        const bool pd = pend[0];
        const long long q0 = gg * TMA_GQ;
        const uint32_t row_g = (uint32_t)(a.row0 + row);
        float4* Xr = reinterpret_cast<float4*>(a.X) + row * NQ;
        float4* Vr = reinterpret_cast<float4*>(a.V) + row * NQ;
        float4* Pr = reinterpret_cast<float4*>(a.P) + row * NQ;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long cb = q0 + 32 * u;
            if (cb >= NQ) break;  // warp-uniform
            const long long q = cb + lane;
            const bool valid = ok && q < NQ;
            float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid) {
                const int k = 32 * u + lane;
                const float4 xo = stg[st].x[k];
                float4 vn = stg[st].v[k];
                const float4 pb = pd ? xo : stg[st].p[k];
                if (pd) st_stream(Pr + q, xo);
                const float4 g4 = __ldg(reinterpret_cast<const float4*>(a.G) + q);
                const float4 lo = bound4t<UNI>(a.lb, a.lb0, q);
                const float4 hi = bound4t<UNI>(a.ub, a.ub0, q);
                const uint4 b1 = Philox::run(make_uint4((uint32_t)q, row_g, (uint32_t)t, 2u), a.rk);
                const uint4 b2 = Philox::run(make_uint4((uint32_t)q, row_g, (uint32_t)t, 3u), a.rk);
                xn = xo;
                pso_elem(xn.x, vn.x, pb.x, g4.x, scaled_u24(b1.x, cp), scaled_u24(b2.x, cg), w, lo.x, hi.x);
                pso_elem(xn.y, vn.y, pb.y, g4.y, scaled_u24(b1.y, cp), scaled_u24(b2.y, cg), w, lo.y, hi.y);
                pso_elem(xn.z, vn.z, pb.z, g4.z, scaled_u24(b1.z, cp), scaled_u24(b2.z, cg), w, lo.z, hi.z);
                pso_elem(xn.w, vn.w, pb.w, g4.w, scaled_u24(b1.w, cp), scaled_u24(b2.w, cg), w, lo.w, hi.w);
                zero_pad(xn, vn, q, a.D);
                st_stream(Xr + q, xn);
                st_stream(Vr + q, vn);
                fit_quad<P>(acc, xn, 4 * q, a.D, htab);
            }
            if constexpr (P == ROSENBROCK) {
                const float nb = __shfl_down_sync(FULL, xn.x, 1);
                const float f0 = __shfl_sync(FULL, xn.x, 0);
                if (cb == 0) head_x = f0;
                if (lane == 31 && hpend) {
                    acc.pair(pend_x, f0);
                    hpend = false;
                }
                if (valid && q + 1 < NQ) {
                    const bool has_next = 4 * q + 4 < a.D;
                    if (lane < 31) {
                        if (has_next) acc.pair(xn.w, nb);
                    } else {
                        hpend = has_next;
                        pend_x = xn.w;
                    }
                }
            }
        }
        __syncwarp();  // all lanes are done reading stage st (reused by group g+2)
        if (gg == NG - 1) {  // end of the row
            const float f = reduce_row<P, G>(acc, a.D, head_x, 0.0f, false, sh_acc, sh_head);
            if (lane == 0 && ok) {
                const bool imp = f < pf_old;  // per-row tell (A11)
                a.f[row] = f;
                a.imp[row] = imp ? 1 : 0;
                if (imp) a.pf[row] = f;
                const unsigned long long k = make_key(f, a.row0 + row);
                best = k < best ? k : best;
            }
            acc = Fit<P>();
            hpend = false;
            pend_x = head_x = 0.0f;
            ++it;
            gg = 0;
            row += m.stride;
            pend[0] = pend[1];
            pend[1] = pend[2];
            const long long r2 = row + 2 * m.stride;
            pend[2] = r2 < a.rows ? a.imp[r2] != 0 : true;
            if (lane == 0 && row < a.rows) pf_old = a.pf[row];
        } else {
            ++gg;
        }
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key)) pso_finalize(a, key, t + 1);
}

// Unfused ask: move X_t -> X_{t+1} (no evaluation).
template <class G, bool UNI>
__global__ void __launch_bounds__(256) k_pso_move(PsoArgs a, unsigned long long t) {
    __shared__ Fit<SPHERE> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    (void)sh_acc;
    (void)sh_head;
    const RowMap<G> m(a.ld >> 2);
    NoPrefetch pf;
    for (long long it = 0;; ++it) {
        const long long wrow = m.wfirst + it * m.stride;
        if (wrow >= a.rows) break;
        const long long row = m.first + it * m.stride;
        const bool ok = row < a.rows;
        const bool pend = ok ? a.imp[row] != 0 : false;
        MoverPso<UNI> mv(a, ok ? row : 0, (uint32_t)t, pend);
        Fit<SPHERE> acc;  // unused
        float hx, tx;
        bool tv;
        walk_segment<SPHERE, G>(mv, m.qb, m.qe, a.D, ok, acc, hx, tx, tv, pf);
        __syncwarp();
        if constexpr (G::WPR > 1) __syncthreads();
        if (m.leader && ok) a.imp[row] = 0;
    }
}

// Tell with given fitness (t = 0 after init, or after an unfused ask).
__global__ void __launch_bounds__(256) k_pso_tell(PsoArgs a, const float* __restrict__ fit,
                                                  unsigned long long t) {
    unsigned long long best = ~0ull;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        const float f = fit[r];
        const bool imp = f < a.pf[r];
        a.f[r] = f;
        a.imp[r] = imp ? 1 : 0;
        if (imp) a.pf[r] = f;
        const unsigned long long k = make_key(f, a.row0 + r);
        best = k < best ? k : best;
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key)) pso_finalize(a, key, t);
}

// world > 1: after the all-gather of the W winner records, pick the min key
// (fitness, then global index) and apply the strict gbest improvement (A13).
__global__ void __launch_bounds__(256) k_gbest_select(PsoArgs a) {
    __shared__ int sh_w;
    __shared__ unsigned long long sh_key;
    Ctl* ctl = a.ctl;
    if (threadIdx.x == 0) {
        unsigned long long k = ~0ull;
        int w = -1;
        for (int r = 0; r < a.world; ++r) {
            const unsigned long long kr =
                *reinterpret_cast<const unsigned long long*>(a.rec + (long long)r * a.rec_stride);
            if (kr < k) { k = kr; w = r; }
        }
        sh_w = w;
        sh_key = k;
    }
    __syncthreads();
    const unsigned long long key = sh_key;
    const bool any = key != ~0ull;
    const float fmin = any ? unord_f32((uint32_t)(key >> 32)) : __int_as_float(0x7f800000);
    const bool better = any && fmin < ctl->gf;
    if (better) {
        const float4* src =
            reinterpret_cast<const float4*>(a.rec + (long long)sh_w * a.rec_stride + 16);
        float4* G = reinterpret_cast<float4*>(a.G);
        for (long long q = threadIdx.x; q < (a.ld >> 2); q += blockDim.x) G[q] = src[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (better) {
            ctl->gf = fmin;
            ctl->gidx = (long long)(uint32_t)(key & 0xffffffffu);
        }
        ctl->hist[ctl->t] = fmin;
    }
}

// Materialise pending pbest rows: P_i <- X_i, imp_i <- 0 (bitwise-neutral).
__global__ void __launch_bounds__(256) k_pso_materialize(PsoArgs a) {
    const long long NQ = a.ld >> 2;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    for (long long row = (long long)blockIdx.x * WARPS + wid; row < a.rows;
         row += (long long)gridDim.x * WARPS) {
        if (!a.imp[row]) continue;
        const float4* x = reinterpret_cast<const float4*>(a.X + row * a.ld);
        float4* p = reinterpret_cast<float4*>(a.P + row * a.ld);
        for (long long q = lane; q < NQ; q += 32) p[q] = x[q];
        __syncwarp();
        if (lane == 0) a.imp[row] = 0;
    }
}

// ---------------------------------------------------------------------------
// CSO (Table II; R-8)

// Keyed bijection of [0,Bb): 4-round Feistel on 2h bits + cycle walking.
struct CsoPerm {
    uint32_t k[4];
    uint32_t h, mask, Bb;
    __device__ __forceinline__ void init(uint32_t blk, uint32_t t, uint32_t Bb_,
                                         const PhiloxKey& rk) {
        const uint4 r = Philox::run(make_uint4(blk, 0u, t, 4u), rk);
        k[0] = r.x; k[1] = r.y; k[2] = r.z; k[3] = r.w;
        Bb = Bb_;
        uint32_t b = 0;
        while (b < 32 && (1ull << b) < (unsigned long long)Bb) ++b;
        if (b < 2) b = 2;
        if (b & 1) ++b;
        h = b / 2;
        mask = (1u << h) - 1u;
    }
    __device__ __forceinline__ uint32_t enc(uint32_t x) const {
        uint32_t L = (x >> h) & mask, R = x & mask;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t F = ((R ^ k[r]) * 0x9E3779B1u) >> (32 - h);
            const uint32_t nR = (L ^ F) & mask;
            L = R;
            R = nR;
        }
        return (L << h) | R;
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        uint32_t y = enc(x);
        while (y >= Bb) y = enc(y);
        return y;
    }
};

// Loser update of one row (A15): v = fmaf(R2, xw-xl, R1*vl) [+ phi R3 (xbar-xl)], clip.
template <bool UNI>
struct MoverCso {
    const CsoArgs& a;
    float4* Xl;
    float4* Vl;
    const float4* Xw;
    uint32_t row_g, t;
    float4 x[U], v[U], xw[U];
    __device__ __forceinline__ MoverCso(const CsoArgs& a_) : a(a_) {}
    template <bool EF>
    __device__ __forceinline__ void load(int u, long long q) {
        x[u] = ld_stream<EF>(Xl + q);
        v[u] = ld_stream<EF>(Vl + q);
        xw[u] = ld_stream<EF>(Xw + q);
    }
    __device__ __forceinline__ static float upd(float xl, float vl, float xwv, float r1, float r2,
                                                float c3, float xb, bool use3, float lo, float hi,
                                                float& vout) {
        float v = __fmaf_rn(r2, __fsub_rn(xwv, xl), __fmul_rn(r1, vl));
        if (use3) v = __fmaf_rn(c3, __fsub_rn(xb, xl), v);
        vout = v;
        return clipf(__fadd_rn(xl, v), lo, hi);
    }
    __device__ __forceinline__ float4 step(int u, long long q) {
        const uint4 b1 = Philox::run(make_uint4((uint32_t)q, row_g, t, 5u), a.rk);
        const uint4 b2 = Philox::run(make_uint4((uint32_t)q, row_g, t, 6u), a.rk);
        const bool use3 = a.phi != 0.0f;
        float4 c3 = make_float4(0.f, 0.f, 0.f, 0.f), xb = c3;
        if (use3) {
            const uint4 b3 = Philox::run(make_uint4((uint32_t)q, row_g, t, 7u), a.rk);
            const float phi = a.phi;
            c3 = make_float4(__fmul_rn(phi, u24(b3.x)), __fmul_rn(phi, u24(b3.y)),
                             __fmul_rn(phi, u24(b3.z)), __fmul_rn(phi, u24(b3.w)));
            xb = __ldg(reinterpret_cast<const float4*>(a.xbar) + q);
        }
        const float4 lo = bound4t<UNI>(a.lb, a.lb0, q);
        const float4 hi = bound4t<UNI>(a.ub, a.ub0, q);
        float4 xn, vn;
        xn.x = upd(x[u].x, v[u].x, xw[u].x, u24(b1.x), u24(b2.x), c3.x, xb.x, use3, lo.x, hi.x, vn.x);
        xn.y = upd(x[u].y, v[u].y, xw[u].y, u24(b1.y), u24(b2.y), c3.y, xb.y, use3, lo.y, hi.y, vn.y);
        xn.z = upd(x[u].z, v[u].z, xw[u].z, u24(b1.z), u24(b2.z), c3.z, xb.z, use3, lo.z, hi.z, vn.z);
        xn.w = upd(x[u].w, v[u].w, xw[u].w, u24(b1.w), u24(b2.w), c3.w, xb.w, use3, lo.w, hi.w, vn.w);
        zero_pad(xn, vn, q, a.D);
        st_stream(Xl + q, xn);
        st_stream(Vl + q, vn);
        return xn;
    }
};

__device__ void cso_finalize(const CsoArgs& a, unsigned long long key, unsigned long long t_new) {
    if (threadIdx.x == 0) {
        Ctl* ctl = a.ctl;
        if (a.peer) key = peer_min(a.mbox, a.rank, a.world, a.peer_timeout_ns, ctl, key, t_new);
        ctl->min_key = key;
        if (a.exchange && !a.peer) {
            ctl->hkeys[t_new] = key;
        } else {
            ctl->hist[t_new] = key != ~0ull ? unord_f32((uint32_t)(key >> 32))
                                            : __int_as_float(0x7f800000);
        }
        ctl->gen_key = ~0ull;
        ctl->ticket = 0u;
        ctl->t = t_new;
    }
}

// The pair (or the unpaired odd member) of CSO work item `it` (R-8).
struct CsoItem {
    long long gw, gl;  // winner, loser global rows (gl < 0: unpaired member gw passes)
    float fw;
    bool valid;  // this rank updates the loser (or owns the unpaired member)
    bool wl;     // the winner (or the unpaired member) is one of this rank's rows
};

__device__ __forceinline__ int cso_owner(const CsoArgs& a, long long r) {
    int w = 0;
    while (w + 1 < a.nsh && r >= a.prow0[w + 1]) ++w;
    return w;
}
__device__ __forceinline__ float cso_f(const CsoArgs& a, long long r, int p) {
    const int w = cso_owner(a, r);
    return a.pf[w][p][r - a.prow0[w]];
}
// Blocks this rank scans: its own (aligned shards) or all of them (global pairing).
__device__ __forceinline__ long long cso_blk0(const CsoArgs& a) { return a.peer ? 0 : a.row0 / a.B; }
__device__ __forceinline__ long long cso_nitems(const CsoArgs& a) {
    const long long blk0 = cso_blk0(a);
    const long long end = a.peer ? a.pop : a.row0 + a.rows;
    return ((end + a.B - 1) / a.B - blk0) * ((a.B + 1) / 2);
}

// Item `it`: its pair (or the unpaired member), the decision, and whether this
// rank does the work (it owns the loser / the unpaired member).
__device__ __forceinline__ CsoItem cso_item(const CsoArgs& a, long long it, uint32_t t) {
    CsoItem r;
    r.valid = false;
    r.wl = false;
    r.gl = -1;
    r.gw = 0;
    r.fw = 0.f;
    const long long blk0 = cso_blk0(a);
    const long long ipb = (a.B + 1) / 2;
    const long long bl = it / ipb, p = it - bl * ipb;
    const long long blk = blk0 + bl;
    const long long base = blk * a.B;
    if (base >= a.pop) return r;
    const long long Bb = (base + a.B <= a.pop) ? a.B : a.pop - base;
    if (p >= (Bb + 1) / 2) return r;
    CsoPerm perm;
    perm.init((uint32_t)blk, t, (uint32_t)Bb, a.rk);
    const long long lo = a.row0, hi = a.row0 + a.rows;  // this rank's rows
    const int par = (int)(t & 1);
    const float* f = a.f2[par];
    if (2 * p + 1 >= Bb) {  // odd block: unpaired member passes unchanged
        r.gw = base + perm((uint32_t)(Bb - 1));
        r.valid = r.gw >= lo && r.gw < hi;
        r.wl = r.valid;
        if (r.valid) r.fw = f[r.gw - a.row0];
        return r;
    }
    const long long gi = base + perm((uint32_t)(2 * p));
    const long long gk = base + perm((uint32_t)(2 * p + 1));
    const bool li = gi >= lo && gi < hi, lk = gk >= lo && gk < hi;
    if (!li && !lk) return r;  // neither member is ours
    const float fi = li ? f[gi - a.row0] : cso_f(a, gi, par);
    const float fk = lk ? f[gk - a.row0] : cso_f(a, gk, par);
    const float oi = fi != fi ? __int_as_float(0x7f800000) : fi;
    const float ok = fk != fk ? __int_as_float(0x7f800000) : fk;
    const bool i_wins = oi < ok || (oi == ok && gi < gk);
    r.gw = i_wins ? gi : gk;
    r.gl = i_wins ? gk : gi;
    r.fw = i_wins ? fi : fk;
    r.valid = i_wins ? lk : li;  // the loser's owner updates it (and contributes the key)
    r.wl = i_wins ? li : lk;     // the winner's owner carries its fitness to the next parity
    return r;
}

// One CSO generation over this shard's whole blocks.  One work item per pair
// (plus one for the unpaired member of an odd block), mapped like a row.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, EVOX_MINB) k_cso_gen(CsoArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P> sh_h;
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const long long items = cso_nitems(a);
    NoPrefetch pf;
    unsigned long long best = ~0ull;
    const long long seg_off = m.qb * 16, seg_bytes = (m.qe - m.qb) * 16;
    // Items are resolved two iterations ahead: the pair's fitness loads land
    // during one iteration, the winner/loser rows are prefetched into L2 during
    // the next (the rows are scattered by the pairing, so there is no stream
    // to follow).  Pairs are disjoint, so no other item of this generation
    // writes the fitness read here.
    CsoItem ci_cur, ci_nxt;
    ci_cur.valid = ci_cur.wl = false;
    ci_nxt.valid = ci_nxt.wl = false;
    if (m.first < items) ci_cur = cso_item(a, m.first, (uint32_t)t);
    if (m.first + m.stride < items) ci_nxt = cso_item(a, m.first + m.stride, (uint32_t)t);
    for (long long k = 0;; ++k) {
        const long long witem = m.wfirst + k * m.stride;
        if (witem >= items) break;
        const long long it = m.first + k * m.stride;
        if ((EVOX_PF & 4) && m.sl == 0 && ci_nxt.valid && ci_nxt.gl >= 0) {
            const char* X = reinterpret_cast<const char*>(a.X);
            const long long ol = (ci_nxt.gl - a.row0) * a.ld * 4 + seg_off;
            prefetch_l2(X + ol, seg_bytes);
            prefetch_l2(reinterpret_cast<const char*>(a.V) + ol, seg_bytes);
            if (ci_nxt.gw >= a.row0 && ci_nxt.gw < a.row0 + a.rows)  // local winners only
                prefetch_l2(X + (ci_nxt.gw - a.row0) * a.ld * 4 + seg_off, seg_bytes);
        }
        CsoItem ci_nn;
        ci_nn.valid = ci_nn.wl = false;
        if (it + 2 * m.stride < items) ci_nn = cso_item(a, it + 2 * m.stride, (uint32_t)t);
        const CsoItem ci = ci_cur;
        const bool pair = ci.valid && ci.gl >= 0;
        MoverCso<UNI> mv(a);
        const long long lrow = pair ? ci.gl - a.row0 : 0, wrow = pair ? ci.gw - a.row0 : 0;
        mv.Xl = reinterpret_cast<float4*>(a.X + lrow * a.ld);
        mv.Vl = reinterpret_cast<float4*>(a.V + lrow * a.ld);
        if (pair && (ci.gw < a.row0 || ci.gw >= a.row0 + a.rows)) {  // winner on a peer GPU
            const int w = cso_owner(a, ci.gw);
            mv.Xw = reinterpret_cast<const float4*>(a.pX[w] + (ci.gw - a.prow0[w]) * a.ld);
        } else {
            mv.Xw = reinterpret_cast<const float4*>(a.X + wrow * a.ld);
        }
        mv.row_g = (uint32_t)(pair ? ci.gl : 0);
        mv.t = (uint32_t)t;
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P, G>(mv, m.qb, m.qe, a.D, pair, acc, hx, tx, tv, pf, htab);
        const float fl = reduce_row<P, G>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
        if (m.leader) {
            float* fnext = a.f2[(t + 1) & 1];
            if (ci.wl) fnext[ci.gw - a.row0] = ci.fw;  // winner / unpaired: unchanged
            if (ci.valid) {
                unsigned long long kk = make_key(ci.fw, ci.gw);
                if (pair) {
                    fnext[ci.gl - a.row0] = fl;
                    const unsigned long long kl = make_key(fl, ci.gl);
                    kk = kl < kk ? kl : kk;
                }
                best = kk < best ? kk : best;
            }
        }
        ci_cur = ci_nxt;
        ci_nxt = ci_nn;
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key, a.peer != 0)) cso_finalize(a, key, t + 1);
}

// Generation 0 (after the evaluation of X0): population minimum -> hist[0].
__global__ void __launch_bounds__(256) k_cso_tell0(CsoArgs a) {
    unsigned long long best = ~0ull;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = make_key(a.f2[0][r], a.row0 + r);
        best = k < best ? k : best;
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key, a.peer != 0)) cso_finalize(a, key, 0);
}

__global__ void k_cso_init(CsoArgs a) {
    init_population(a.X, a.V, nullptr, a.rows, a.row0, a.D, a.ld, a.lb, a.ub, a.lb0, a.ub0,
                    a.uniform_bounds, a.rk);
}

// Column means for the phi != 0 term: fixed row chunks of 1024, fp64 partial
// sums in row order, chunks combined in order (world == 1 only).
__global__ void k_colsum_partial(const float* __restrict__ X, long long rows, long long ld,
                                 double* __restrict__ part) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long c = blockIdx.y;
    if (j >= ld) return;
    const long long r0 = c * 1024, r1 = (r0 + 1024 < rows) ? r0 + 1024 : rows;
    double s = 0.0;
    for (long long r = r0; r < r1; ++r) s += (double)X[r * ld + j];
    part[c * ld + j] = s;
}
__global__ void k_colsum_final(const double* __restrict__ part, long long nchunk, long long rows,
                               long long ld, float* __restrict__ xbar) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ld) return;
    double s = 0.0;
    for (long long c = 0; c < nchunk; ++c) s += part[c * ld + j];
    xbar[j] = (float)(s / (double)rows);
}

// world > 1: hist[t] from the all-reduced (min) keys.
__global__ void k_keys_to_hist(Ctl* ctl, unsigned long long t0, long long n) {
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long k = ctl->hkeys[t0 + i];
        ctl->hist[t0 + i] =
            k != ~0ull ? unord_f32((uint32_t)(k >> 32)) : __int_as_float(0x7f800000);
    }
}

// argmin key of a fitness vector (one CTA; for best() queries, not hot).
__global__ void __launch_bounds__(1024) k_argmin_rows(const float* f, long long rows,
                                                      long long row0,
                                                      unsigned long long* key_out) {
    __shared__ unsigned long long sh[32];
    unsigned long long best = ~0ull;
    for (long long r = threadIdx.x; r < rows; r += blockDim.x) {
        const unsigned long long k = make_key(f[r], row0 + r);
        best = k < best ? k : best;
    }
    best = warp_min_u64(best);
    if (lane_id() == 0) sh[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = sh[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) k = sh[i] < k ? sh[i] : k;
        *key_out = k;
    }
}

// ---------------------------------------------------------------------------
// DE/rand/1/bin (the DE of the paper's experiment P:700; R-14)

// Donor indices of target i: rejection sampling over the word stream
// philox((c, i, t, 8))[l], each word mapped to [0,N) by (w * N) >> 32.
// Expected ~3 words: O(1) per target whatever N (the paper's EvoX DE stopped
// at N = 16,384 on its distinct-index sampling).
__device__ __forceinline__ void de_indices(const DeArgs& a, long long i, uint32_t t,
                                           long long r[3]) {
    int got = 0;
    for (uint32_t c = 0; got < 3; ++c) {
        const uint4 w = Philox::run(make_uint4(c, (uint32_t)i, t, 8u), a.rk);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            if (got < 3) {
                const long long v = (long long)(((unsigned long long)ws[l] * (unsigned long long)a.pop) >> 32);
                bool ok = v != i;
                for (int k = 0; k < got; ++k) ok = ok && v != r[k];
                if (ok) r[got++] = v;
            }
        }
    }
}

template <bool UNI>
struct MoverDe {
    const DeArgs& a;
    const float4* Xi;
    const float4* Xa;
    const float4* Xb;
    const float4* Xc;
    float4* Out;
    uint32_t row_g, t;
    long long jrand;
    float4 x[U], xa[U], xb[U], xc[U];
    __device__ __forceinline__ explicit MoverDe(const DeArgs& a_) : a(a_) {}
    template <bool EF>
    __device__ __forceinline__ void load(int u, long long q) {
        x[u] = ld_stream<EF>(Xi + q);
        xa[u] = __ldcg(Xa + q);  // donors: random rows, may be re-read by other targets
        xb[u] = __ldcg(Xb + q);
        xc[u] = __ldcg(Xc + q);
    }
    __device__ __forceinline__ static float trial(float xi, float va, float vb, float vc, float U,
                                                  float CR, float F, bool forced, float lo,
                                                  float hi) {
        const float v = __fmaf_rn(F, __fsub_rn(vb, vc), va);
        const float y = (U < CR || forced) ? v : xi;
        return clipf(y, lo, hi);
    }
    __device__ __forceinline__ float4 step(int u, long long q) {
        const uint4 b = Philox::run(make_uint4((uint32_t)q, row_g, t, 10u), a.rk);
        const float4 lo = bound4t<UNI>(a.lb, a.lb0, q);
        const float4 hi = bound4t<UNI>(a.ub, a.ub0, q);
        const long long j0 = 4 * q;
        const float F = a.F, CR = a.CR;
        float4 o;
        o.x = trial(x[u].x, xa[u].x, xb[u].x, xc[u].x, u24(b.x), CR, F, j0 == jrand, lo.x, hi.x);
        o.y = trial(x[u].y, xa[u].y, xb[u].y, xc[u].y, u24(b.y), CR, F, j0 + 1 == jrand, lo.y, hi.y);
        o.z = trial(x[u].z, xa[u].z, xb[u].z, xc[u].z, u24(b.z), CR, F, j0 + 2 == jrand, lo.z, hi.z);
        o.w = trial(x[u].w, xa[u].w, xb[u].w, xc[u].w, u24(b.w), CR, F, j0 + 3 == jrand, lo.w, hi.w);
        float4 dummy = o;
        zero_pad(o, dummy, q, a.D);
        st_stream(Out + q, o);
        return o;
    }
};

__device__ __forceinline__ float nan_inf(float v) { return v != v ? __int_as_float(0x7f800000) : v; }

// Owner rank of a global row (linear scan over <= kMaxPeers shard offsets).
__device__ __forceinline__ int de_owner(const DeArgs& a, long long r) {
    int w = 0;
    while (w + 1 < a.world && r >= a.prow0[w + 1]) ++w;
    return w;
}


__device__ __forceinline__ void de_finalize(const DeArgs& a, unsigned long long key,
                                            unsigned long long t_new) {
    if (threadIdx.x == 0) {
        Ctl* ctl = a.ctl;
        if (a.peer) key = peer_min(a.mbox, a.rank, a.world, a.peer_timeout_ns, ctl, key, t_new);
        ctl->hist[t_new] = key != ~0ull ? unord_f32((uint32_t)(key >> 32)) : __int_as_float(0x7f800000);
        ctl->min_key = key;
        ctl->gen_key = ~0ull;
        ctl->ticket = 0u;
        ctl->t = t_new;
    }
}

// One DE generation: trial of every target from the population at parity p,
// evaluation, greedy "<=" replacement by flipping the buffer-select flag.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, EVOX_MINB) k_de_gen(DeArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P> sh_h;
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const int p = (int)(t & 1);
    const unsigned char* sel = a.sel[p];
    NoPrefetch pf;
    unsigned long long best = ~0ull;
    // The next target's donors and the buffer flags of its rows are resolved one
    // iteration ahead: their loads (scattered bytes) land while this row streams,
    // so the row loads of the next iteration are not behind a 2-deep dependent
    // chain (indices -> flags -> rows).
    uint32_t nr[3] = {0, 0, 0}, nsb = 0;
    float nfx = 0.0f;
    auto resolve = [&](long long rw, uint32_t r3[3], uint32_t& sb, float& fx) {
        if (rw < a.rows) {
            long long r[3];
            de_indices(a, a.row0 + rw, (uint32_t)t, r);
            r3[0] = (uint32_t)r[0];
            r3[1] = (uint32_t)r[1];
            r3[2] = (uint32_t)r[2];
            int fl[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int w = de_owner(a, r[k]);
                fl[k] = a.psel[w][p][r[k] - a.prow0[w]];
            }
            sb = (uint32_t)sel[rw] | ((uint32_t)fl[0] << 1) | ((uint32_t)fl[1] << 2) |
                 ((uint32_t)fl[2] << 3);
            fx = a.f[p][rw];
        }
    };
    resolve(m.first, nr, nsb, nfx);
    for (long long it = 0;; ++it) {
        const long long wrow = m.wfirst + it * m.stride;
        if (wrow >= a.rows) break;
        const long long row = m.first + it * m.stride;
        const bool ok = row < a.rows;
        const uint32_t cr0 = nr[0], cr1 = nr[1], cr2 = nr[2], csb = nsb;
        const float cfx = nfx;
        resolve(row + m.stride, nr, nsb, nfx);
        MoverDe<UNI> mv(a);
        int si = 0;
        float fx = 0.0f;
        if (ok) {
            si = (int)(csb & 1u);
            auto donor = [&](uint32_t r, int k) {
                const int w = de_owner(a, r);
                return reinterpret_cast<const float4*>(a.pbuf[w][(csb >> (k + 1)) & 1u] +
                                                       ((long long)r - a.prow0[w]) * a.ld);
            };
            mv.Xi = reinterpret_cast<const float4*>(a.buf[si] + row * a.ld);
            mv.Xa = donor(cr0, 0);
            mv.Xb = donor(cr1, 1);
            mv.Xc = donor(cr2, 2);
            mv.Out = reinterpret_cast<float4*>(a.buf[si ^ 1] + row * a.ld);
            const uint4 jw = Philox::run(make_uint4(0u, (uint32_t)(a.row0 + row), (uint32_t)t, 9u), a.rk);
            mv.jrand = (long long)(((unsigned long long)jw.x * (unsigned long long)a.D) >> 32);
            fx = cfx;
        } else {
            mv.Xi = mv.Xa = mv.Xb = mv.Xc = nullptr;
            mv.Out = nullptr;
            mv.jrand = -1;
        }
        mv.row_g = (uint32_t)(a.row0 + row);
        mv.t = (uint32_t)t;
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P, G>(mv, m.qb, m.qe, a.D, ok, acc, hx, tx, tv, pf, htab);
        const float fu = reduce_row<P, G>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
        if (m.leader && ok) {
            const bool accept = nan_inf(fu) <= nan_inf(fx);  // S:325, NaN as +inf
            const float fn = accept ? fu : fx;
            a.sel[p ^ 1][row] = (unsigned char)(accept ? (si ^ 1) : si);
            a.f[p ^ 1][row] = fn;
            const unsigned long long k = make_key(fn, a.row0 + row);
            best = k < best ? k : best;
        }
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key, a.peer != 0)) de_finalize(a, key, t + 1);
}

__global__ void k_de_init(DeArgs a) {
    init_population(a.buf[0], a.buf[1], nullptr, a.rows, a.row0, a.D, a.ld, a.lb, a.ub, a.lb0,
                    a.ub0, a.uniform_bounds, a.rk);
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        a.sel[0][r] = 0;
        a.sel[1][r] = 0;
    }
}

// Generation 0 (after evaluating buf[0] into f[0]): hist[0] = min f.
__global__ void __launch_bounds__(256) k_de_tell0(DeArgs a) {
    unsigned long long best = ~0ull;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = make_key(a.f[0][r], a.row0 + r);
        best = k < best ? k : best;
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key, a.peer != 0)) de_finalize(a, key, 0);
}

// Gather the current population into buf[0] (rows held by buf[1] are copied and
// their flag reset): bitwise-neutral for later generations.
__global__ void __launch_bounds__(256) k_de_materialize(DeArgs a) {
    const int p = (int)(a.ctl->t & 1);
    const long long NQ = a.ld >> 2;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    for (long long row = (long long)blockIdx.x * WARPS + wid; row < a.rows;
         row += (long long)gridDim.x * WARPS) {
        if (!a.sel[p][row]) continue;
        const float4* s = reinterpret_cast<const float4*>(a.buf[1] + row * a.ld);
        float4* d = reinterpret_cast<float4*>(a.buf[0] + row * a.ld);
        for (long long q = lane; q < NQ; q += 32) d[q] = s[q];
        __syncwarp();
        if (lane == 0) a.sel[p][row] = 0;
    }
}

__global__ void k_debug_philox(const uint4* ctr, PhiloxKey rk, uint4* out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = Philox::run(ctr[i], rk);
}

// ----------------------------------------------------------------- dispatch
int sm_count(int device) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

using G4 = Geom<4, 1, U, false>;  // short rows: plain loads measured best (C4: +5 points)
using G8 = Geom<8, 1>;
using G32 = Geom<32, 1>;
using GW8 = Geom<32, 8, 3>;  // long rows: 3 chunks in flight measured best (C5)

// 3: 4 lanes per row (ld <= 128), 0: 8 lanes per row (ld <= 256), 1: a warp per
// row (ld <= 4096), 2: a CTA per row.  Narrow row groups keep short rows from
// idling lanes (dim 100 = 25 quads: 28 lane-slots with 4 lanes vs 32 with 8).
int geom_id(long long ld) {
    const long long NQ = ld >> 2;
    if (NQ <= 32) return 3;
    if (NQ <= 64) return 0;
    if (NQ <= 1024) return 1;
    return 2;
}

int grid_for(const void* fn, long long units, int device) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)sm_count(device) * per_sm;
    if (units < g) g = units;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

int wpr_for_dim(long long ld) { return geom_id(ld) == 2 ? 8 : 1; }

#define EVOX_DISPATCH_GEOM(ld, ...)     \
    do {                                \
        switch (geom_id(ld)) {          \
            case 3: {                   \
                using G_ = G4;          \
                __VA_ARGS__;            \
            } break;                    \
            case 0: {                   \
                using G_ = G8;          \
                __VA_ARGS__;            \
            } break;                    \
            case 1: {                   \
                using G_ = G32;         \
                __VA_ARGS__;            \
            } break;                    \
            default: {                  \
                using G_ = GW8;         \
                __VA_ARGS__;            \
            } break;                    \
        }                               \
    } while (0)

#define EVOX_DISPATCH_PROB(p, ...)             \
    do {                                       \
        switch (p) {                           \
            case SPHERE: {                     \
                constexpr int P_ = SPHERE;     \
                __VA_ARGS__;                   \
            } break;                           \
            case ACKLEY: {                     \
                constexpr int P_ = ACKLEY;     \
                __VA_ARGS__;                   \
            } break;                           \
            case RASTRIGIN: {                  \
                constexpr int P_ = RASTRIGIN;  \
                __VA_ARGS__;                   \
            } break;                           \
            case GRIEWANK: {                   \
                constexpr int P_ = GRIEWANK;   \
                __VA_ARGS__;                   \
            } break;                           \
            default: {                         \
                constexpr int P_ = ROSENBROCK; \
                __VA_ARGS__;                   \
            } break;                           \
        }                                      \
    } while (0)

#define EVOX_DISPATCH_UNI(u, ...)         \
    do {                                  \
        if (u) {                          \
            constexpr bool U_ = true;     \
            __VA_ARGS__;                  \
        } else {                          \
            constexpr bool U_ = false;    \
            __VA_ARGS__;                  \
        }                                 \
    } while (0)

template <class G>
static long long row_units(long long rows) {
    return (rows + G::RPC - 1) / G::RPC;
}

cudaError_t launch_pso_init(const PsoArgs& a, cudaStream_t st) {
    const long long total = a.rows * (a.ld >> 2);
    long long g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_pso_init<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_eval(int problem, const float* X, long long rows, long long D, long long ld,
                        float* fit, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        const int g = grid_for((const void*)k_eval<P_, G_>, row_units<G_>(rows), dev);
        k_eval<P_, G_><<<g, 256, 0, st>>>(X, rows, D, ld, fit);
    }));
    return cudaGetLastError();
}

int pso_gen_grid(int problem, long long ld, long long rows, int device) {
    int g = 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        g = grid_for((const void*)k_pso_gen<P_, G_, true>, row_units<G_>(rows), device);
    }));
    return g;  // the TMA variant uses the same grid (2 CTAs/SM: 2 x 96 KB of staging)
}

// Generation kernels are launched with programmatic stream serialization (PDL):
// kernel t+1 becomes resident while kernel t retires (EVOX_NO_PDL=1: plain launch).
template <class K, class A>
static cudaError_t launch_pdl(K kernel, int grid, const A& a, cudaStream_t st, size_t smem = 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = getenv("EVOX_NO_PDL") ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

// The TMA-staged kernel is an opt-in variant (EVOX_TMA=1) of the warp-per-row
// geometry: measured 4-5 points BELOW the LDG + bulk-L2-prefetch kernel at H
// and C2, so the LDG kernel is the default.
static bool use_tma(long long ld) {
    const char* v = getenv("EVOX_TMA");
    return geom_id(ld) == 1 && U == 4 && v && *v == '1';
}

template <class K>
static void tma_attr(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM);
}

cudaError_t launch_pso_gen(int problem, const PsoArgs& a, int grid, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (use_tma(a.ld)) {
        EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, {
            tma_attr(k_pso_gen_tma<P_, U_>);
            e = launch_pdl(k_pso_gen_tma<P_, U_>, grid, a, st, TMA_SMEM);
        }));
    } else {
        EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
            e = launch_pdl(k_pso_gen<P_, G_, U_>, grid, a, st);
        })));
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

bool pso_small(long long rows, long long ld) { return rows * ld <= 65536; }

cudaError_t launch_pso_run_small(int problem, const PsoArgs& a, long long n, cudaStream_t st) {
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
        k_pso_run_small<P_, G_, U_><<<1, 256, 0, st>>>(a, n);
    })));
    return cudaGetLastError();
}

cudaError_t launch_pso_move(const PsoArgs& a, unsigned long long t, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_GEOM(a.ld, {
        const int g = grid_for((const void*)k_pso_move<G_, U_>, row_units<G_>(a.rows), dev);
        k_pso_move<G_, U_><<<g, 256, 0, st>>>(a, t);
    }));
    return cudaGetLastError();
}

cudaError_t launch_pso_tell(const PsoArgs& a, const float* fit, unsigned long long t,
                            cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int g = grid_for((const void*)k_pso_tell, (a.rows + 255) / 256, dev);
    k_pso_tell<<<g, 256, 0, st>>>(a, fit, t);
    return cudaGetLastError();
}

cudaError_t launch_gbest_select(const PsoArgs& a, cudaStream_t st) {
    k_gbest_select<<<1, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pso_materialize(const PsoArgs& a, cudaStream_t st) {
    long long g = (a.rows + WARPS - 1) / WARPS;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_pso_materialize<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_cso_init(const CsoArgs& a, cudaStream_t st) {
    const long long total = a.rows * (a.ld >> 2);
    long long g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_cso_init<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_cso_tell0(const CsoArgs& a, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int g = grid_for((const void*)k_cso_tell0, (a.rows + 255) / 256, dev);
    k_cso_tell0<<<g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

static long long cso_items(const CsoArgs& a) {
    const long long blk0 = a.peer ? 0 : a.row0 / a.B;
    const long long end = a.peer ? a.pop : a.row0 + a.rows;
    return ((end + a.B - 1) / a.B - blk0) * ((a.B + 1) / 2);
}

int cso_gen_grid(int problem, const CsoArgs& a, int device) {
    int g = 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
        g = grid_for((const void*)k_cso_gen<P_, G_, true>, row_units<G_>(cso_items(a)), device);
    }));
    return g;
}

cudaError_t launch_cso_gen(int problem, const CsoArgs& a, int grid, cudaStream_t st) {
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
        k_cso_gen<P_, G_, U_><<<grid, 256, 0, st>>>(a);
    })));
    return cudaGetLastError();
}

cudaError_t launch_cso_colmean(const CsoArgs& a, float* xbar, double* scratch, cudaStream_t st) {
    const long long nchunk = (a.rows + 1023) / 1024;
    dim3 g1((unsigned)((a.ld + 127) / 128), (unsigned)nchunk);
    k_colsum_partial<<<g1, 128, 0, st>>>(a.X, a.rows, a.ld, scratch);
    k_colsum_final<<<(unsigned)((a.ld + 127) / 128), 128, 0, st>>>(scratch, nchunk, a.rows, a.ld,
                                                                    xbar);
    return cudaGetLastError();
}

cudaError_t launch_cso_hist_from_keys(const CsoArgs& a, unsigned long long t0, long long n,
                                      cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_keys_to_hist<<<1, 256, 0, st>>>(a.ctl, t0, n);
    return cudaGetLastError();
}

cudaError_t launch_argmin_rows(const float* f, long long rows, long long row0,
                               unsigned long long* key_out, cudaStream_t st) {
    k_argmin_rows<<<1, 1024, 0, st>>>(f, rows, row0, key_out);
    return cudaGetLastError();
}

cudaError_t launch_de_init(const DeArgs& a, cudaStream_t st) {
    const long long total = a.rows * (a.ld >> 2);
    long long g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_de_init<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_de_tell0(const DeArgs& a, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int g = grid_for((const void*)k_de_tell0, (a.rows + 255) / 256, dev);
    k_de_tell0<<<g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

int de_gen_grid(int problem, long long ld, long long rows, int device) {
    int g = 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        g = grid_for((const void*)k_de_gen<P_, G_, true>, row_units<G_>(rows), device);
    }));
    return g;
}

cudaError_t launch_de_gen(int problem, const DeArgs& a, int grid, cudaStream_t st) {
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
        k_de_gen<P_, G_, U_><<<grid, 256, 0, st>>>(a);
    })));
    return cudaGetLastError();
}

cudaError_t launch_de_materialize(const DeArgs& a, cudaStream_t st) {
    long long g = (a.rows + WARPS - 1) / WARPS;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_de_materialize<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_debug_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                                long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long g = (n + 255) / 256;
    if (g > 4096) g = 4096;
    const PhiloxKey rk = Philox::schedule(((uint64_t)k1 << 32) | k0);
    k_debug_philox<<<(int)g, 256, 0, st>>>(reinterpret_cast<const uint4*>(ctr), rk,
                                           reinterpret_cast<uint4*>(out), n);
    return cudaGetLastError();
}

}  // namespace evox
