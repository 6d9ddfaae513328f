// row_engine.cuh -- building blocks shared by every generation kernel:
// launch geometry, the row engine (walk_segment / reduce_row), bulk L2 prefetch,
// the grid argmin, the peer-memory barrier primitives, the population init and
// the dispatch helpers.  Header-only (internal linkage in each kernel TU).
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
#pragma once

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
#ifndef EVOX_ABL
#define EVOX_ABL 0  // ablation bits for measurement builds only; 0 in the product
#endif
#ifndef EVOX_MINB
#define EVOX_MINB 2
#endif
// CTAs per SM the generation kernels are register-capped for in the short-row
// (4 lanes/row, dim <= 128) geometry: tuning switches, measured in DESIGN.md §7
#ifndef EVOX_PSO_SHORT_MINB
#define EVOX_PSO_SHORT_MINB EVOX_MINB
#endif
#ifndef EVOX_DE_SHORT_MINB
#define EVOX_DE_SHORT_MINB 3  // with 2 chunks in flight: D1 0.665 -> 0.713 (r02_ab_de.txt)
#endif
#ifndef EVOX_ROW_MINB
#define EVOX_ROW_MINB 3  // CTA-per-row geometry (ld > 4096): C5 0.872 -> 0.909 (r02_pf.txt)
#endif
#ifndef EVOX_PDL
#define EVOX_PDL 1  // programmatic dependent launch of the generation kernels
#endif
#ifndef EVOX_AHEAD
#define EVOX_AHEAD 4  // mode-B prefetch window, in lane groups
#endif
#ifndef EVOX_PF
// L2 bulk-prefetch switches (measured): bit 0 unused (mode A, a warp's next
// short rows, is the runtime PsoArgs.pf_next: pso_prefetch_next), bit 1 mode B (sliding window inside long rows:
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
__device__ __forceinline__ float4 bound4t(const float* b, float b0, int q) {
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

__device__ __forceinline__ void zero_pad(float4& x, float4& v, int q, int D) {
    if (4 * q + 3 >= D) {  // padding columns stay 0
        const int j0 = 4 * q;
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
// Shared-memory column table: only the warp-row geometries (ld <= HTAB) of
// Griewank use it; the CTA-per-row geometry reads the global table of evox_eval
// (or computes h_j per element) and must not give up 16 KB of L1 for nothing.
template <int P, class G>
struct HStore {
    float v[1];
};
template <class G>
struct HStore<GRIEWANK, G> {
    float v[G::WPR > 1 ? 1 : HTAB];
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
__device__ __forceinline__ void walk_segment(Mover& mv, long long qb_, long long qe_, long long D_,
                                             bool row_ok, Fit<P>& acc, float& head_x,
                                             float& tail_x, bool& tail_valid, PF& pf,
                                             const float* htab = nullptr) {
    // in-row indices in 32 bits (ld < 2^31 is validated at init): fewer integer
    // instructions per chunk than 64-bit compares and adds
    const int sl = lane_id() & (G::LPR - 1);
    const int qb = (int)qb_, qe = (int)qe_, D = (int)D_;
    float pend_x = 0.0f;
    bool pend = false;  // last sub-lane: x_{4q+3} waiting for x_{4q+4} of the next chunk
    head_x = 0.0f;
    tail_valid = false;
    tail_x = 0.0f;
    // one chunk: move (Mover::step), fitness terms, Rosenbrock halo -- in chunk order
    auto chunk = [&](int u, int base) {
        const int cb = base + G::LPR * u;  // first quad of this chunk
        const int q = cb + sl;
        const bool valid = row_ok && q < qe;
        float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            xn = mv.step(u, q);
#if EVOX_ABL & 2  // ablation (measurement builds only): no fitness terms
#else
            fit_quad<P>(acc, xn, 4 * q, D, htab);
#endif
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
    };
    // Rosenbrock, interior group (every quad q of the group has q + 1 < qe and
    // 4q + 4 < D): the same terms in the same order as `chunk`, without the
    // per-element bounds and segment-end bookkeeping (E5-rosenbrock: ~23 -> ~10
    // lane-instructions per element).  Bitwise equal to `chunk`.
    auto chunk_interior = [&](int u, int base) {
      if constexpr (P == ROSENBROCK) {
        const int cb = base + G::LPR * u;
        const int q = cb + sl;
        float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row_ok) {
            xn = mv.step(u, q);
            acc.pair(xn.x, xn.y);
            acc.pair(xn.y, xn.z);
            acc.pair(xn.z, xn.w);
        }
        const float nb = __shfl_down_sync(FULL, xn.x, 1, G::LPR);
        const float f0 = __shfl_sync(FULL, xn.x, 0, G::LPR);
        if (cb == qb) head_x = f0;
        if (sl == G::LPR - 1) {
            if (pend) acc.pair(pend_x, f0);
            pend = row_ok;
            pend_x = xn.w;
        } else if (row_ok) {
            acc.pair(xn.w, nb);
        }
      }
    };
    auto load = [&](int u, int base) {
        const int q = base + G::LPR * u + sl;
        if (row_ok && q < qe) mv.template load<G::EFL>(u, q);
    };
    // loads that depend on a late-arriving per-row flag (PSO: P unless the pbest copy is
    // pending) go out after every independent load of the group, so the flag's latency
    // overlaps the other loads instead of stalling them
    auto load_late = [&](int u, int base) {
        const int q = base + G::LPR * u + sl;
        if (row_ok && q < qe) mv.template load_late<G::EFL>(u, q);
    };
    for (int base = qb; base < qe; base += G::GROUP) {
        pf(base);
#pragma unroll
        for (int u = 0; u < G::NU; ++u) load(u, base);
#pragma unroll
        for (int u = 0; u < G::NU; ++u) load_late(u, base);
        if constexpr (P == ROSENBROCK) {
            if (base + G::GROUP < qe && 4LL * (base + G::GROUP) < D) {  // warp-uniform
#pragma unroll
                for (int u = 0; u < G::NU; ++u) chunk_interior(u, base);
                continue;
            }
        }
#pragma unroll
        for (int u = 0; u < G::NU; ++u) {
            if (base + G::LPR * u >= qe) break;  // warp-uniform
            chunk(u, base);
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
    __device__ __forceinline__ void load(int u, int q) { x[u] = ld_stream<EF>(Xr + q); }
    template <bool EF>
    __device__ __forceinline__ void load_late(int, int) {}
    __device__ __forceinline__ float4 step(int u, long long) { return x[u]; }
};

// ---------------------------------------------------------------------------
// Flat-tile kernels (k_pso_gen_flat, k_de_gen_flat, k_cso_gen_flat): a CTA moves the quads of
// a tile of rows as one flat range, stages per-quad values in shared memory, then folds each
// row's fitness in the row geometry's order (bitwise the row-walk kernels' f).
//   staged layout: A[T][NQ] float4 (+ B[T][NQ] when pre_comps<P>() == 2), then htab.
// Rosenbrock stages x' and is folded by the row engine (pairs straddle quads); the other
// problems stage pre_quad's values (every expensive per-element term, computed by all 256
// threads in the flat phase) and a lane only applies fold_quad's accumulator operations.
struct MoverSmem {
    const float4* xr;
    float4 x[U];
    template <bool EF>
    __device__ __forceinline__ void load(int u, int q) { x[u] = xr[q]; }
    template <bool EF>
    __device__ __forceinline__ void load_late(int, int) {}
    __device__ __forceinline__ float4 step(int u, int) { return x[u]; }
};

template <int P>
__host__ __device__ constexpr int stage_comps() { return P == ROSENBROCK ? 1 : pre_comps<P>(); }

// Bytes of staging for T rows of ld floats (+ the Griewank column table).
template <int P>
inline size_t flat_stage_bytes(long long T, long long ld) {
    return (size_t)T * (size_t)ld * 4 * stage_comps<P>() + (P == GRIEWANK ? (size_t)ld * 4 : 0);
}

// Stage quad i (column quad q) of the tile.
template <int P>
__device__ __forceinline__ void stage_quad(float4* st, int tile_quads, int i, int q, float4 x,
                                           const float* htab) {
    if constexpr (P == ROSENBROCK) {
        st[i] = x;
    } else {
        float4 A, B;
        pre_quad<P>(x, 4 * q, htab, A, B);
        st[i] = A;
        if constexpr (pre_comps<P>() == 2) st[tile_quads + i] = B;
    }
}

// Fold staged row `lr` of the tile in geometry G's order (a lane group of LPR lanes per row,
// WPR == 1); returns f in sub-lane 0.  Every lane of the warp must call it (shuffles).
template <int P, class G>
__device__ __forceinline__ float fold_staged_row(const float4* st, int tile_quads, int lr, int NQ,
                                                 long long D, bool row_ok, const float* htab,
                                                 Fit<P>* sh_acc, float* sh_head) {
    static_assert(G::WPR == 1, "warp-row geometries only");
    Fit<P> acc;
    float hx = 0.f, tx = 0.f;
    bool tv = false;
    if constexpr (P == ROSENBROCK) {
        MoverSmem ms;
        ms.xr = st + lr * NQ;
        NoPrefetch pf;
        walk_segment<P, G>(ms, 0, NQ, D, row_ok, acc, hx, tx, tv, pf, htab);
    } else {
        const int sl = lane_id() & (G::LPR - 1);
        if (row_ok) {
            const float4* A = st + lr * NQ;
            const float4* B = st + tile_quads + lr * NQ;
            for (int q = sl; q < NQ; q += G::LPR) {
                const float4 a = A[q];
                const float4 b = pre_comps<P>() == 2 ? B[q] : a;
                fold_quad<P>(acc, a, b, 4 * q, (int)D);
            }
        }
    }
    return reduce_row<P, G>(acc, D, hx, tx, tv, sh_acc, sh_head);
}

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
// Grid-barrier primitives of the persistent kernels (GPU scope).
__device__ __forceinline__ void st_release_gpu_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_gpu_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
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

// ----------------------------------------------------------------- dispatch
inline int sm_count(int device) {
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
// A function of ld only: every reduction order -- hence every fitness bit -- is fixed by
// the dimension, whatever the population, shard count or launch grid (R-11).
inline int geom_id(long long ld) {
    const long long NQ = ld >> 2;
    if (NQ <= 32) return 3;
    if (NQ <= 64) return 0;
    if (NQ <= 1024) return 1;
    return 2;
}

// CSO generation: 8 lanes per row up to 1024 quads (one warp walks 4 independent pairs at
// once, so more scattered winner/loser rows are in flight: C3 71 -> 77 % of HBM peak; PSO
// and DE measured worse with it). Still a function of ld only (R-11).
inline int cso_geom_id(long long ld) {
    const int g = geom_id(ld);
    return g == 1 ? 0 : g;
}

// `waves` x (resident CTAs), at most one CTA per row unit.  The grid never changes a result
// bit (every reduction is per row; the argmin is exact), only the schedule.
inline int grid_for(const void* fn, long long units, int device, int waves = 1) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)sm_count(device) * per_sm * waves;
    if (units < g) g = units;
    return (int)(g < 1 ? 1 : g);
}

// Generation kernels are launched with programmatic stream serialization (PDL):
// kernel t+1 becomes resident while kernel t retires.
template <class K, class A>
inline cudaError_t launch_pdl(K kernel, int grid, const A& a, cudaStream_t st, size_t smem = 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = EVOX_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <class G>
inline long long row_units(long long rows) {
    return (rows + G::RPC - 1) / G::RPC;
}

}  // namespace

#define EVOX_DISPATCH_GEOM(ld, ...) EVOX_DISPATCH_GEOM_ID(geom_id(ld), __VA_ARGS__)
#define EVOX_DISPATCH_GEOM_ID(id, ...)  \
    do {                                \
        switch (id) {                   \
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

}  // namespace evox
