// pso_kernels.cu -- PSO: the fused generation kernel (A1-A12), its TMA-staged
// variant, the persistent small-population kernel, the unfused ask/tell kernels and the
// gbest exchange (A13: NCCL select or in-kernel peer-memory mailboxes).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "evox_device.cuh"
#include "evox_internal.h"
#include "row_engine.cuh"

namespace evox {

namespace {

// PSO move of one row (A1, A3, A4, lazy A5).  Holds a reference to the kernel
// parameter block (resolved to constant-bank operands once inlined: the
// Philox round keys, w, phi*2^-24 and the bounds feed instructions directly).
// STS: evict-first stores (the row-walk kernels); the kernels that bulk-prefetch their tile into
// L2 store (and load) with the default policy (profiles/r02_ab_hints.txt).
template <bool UNI, bool G_COHERENT = false, bool STS = true>
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
    // row pointers already at hand (the flat tiles: tile base + r * NQ, 32-bit offsets)
    __device__ __forceinline__ MoverPso(const PsoArgs& a_, float4* xr, float4* vr, float4* pr,
                                        uint32_t row_g_, uint32_t t_, bool pend_)
        : a(a_), Xr(xr), Vr(vr), Pr(pr), row_g(row_g_), t(t_), pend(pend_) {}
    template <bool EF>
    __device__ __forceinline__ void load(int u, int q) {
        x[u] = ld_stream<EF>(Xr + q);
        v[u] = ld_stream<EF>(Vr + q);
    }
    template <bool EF>
    __device__ __forceinline__ void load_late(int u, int q) {  // waits for imp (pend)
        if (!pend) p[u] = ld_stream<EF>(Pr + q);
    }
    __device__ __forceinline__ float4 step(int u, int q) {
        const float4 xo = x[u];
        const float4 pb = pend ? xo : p[u];
        if (pend) st_stream<STS>(Pr + q, xo);
        // G is read-only for a generation kernel (non-coherent path); the persistent
        // kernels rewrite it between generations: a plain (coherent, L1-cached) load,
        // ordered after the rewrite by the barrier's acquire + bar.sync.
#if EVOX_ABL & 4  // ablation (measurement builds only): no gbest load
        const float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#else
        const float4 g = G_COHERENT ? *(reinterpret_cast<const float4*>(a.G) + q)
                                    : __ldg(reinterpret_cast<const float4*>(a.G) + q);
#endif
        const float4 lo = bound4t<UNI>(a.lb, a.lb0, q);
        const float4 hi = bound4t<UNI>(a.ub, a.ub0, q);
#if EVOX_ABL & 1  // ablation: no Philox
        const uint4 b1 = make_uint4(q * 0x9E3779B9u, row_g * 0x85EBCA6Bu, q ^ row_g, t);
        const uint4 b2 = make_uint4(row_g * 0x9E3779B9u, q * 0x85EBCA6Bu, q + row_g, t);
#else
        const uint4 b1 = Philox::run(make_uint4((uint32_t)q, row_g, t, 2u), a.rk);
        const uint4 b2 = Philox::run(make_uint4((uint32_t)q, row_g, t, 3u), a.rk);
#endif
        float4 xn = xo, vn = v[u];
        const float w = a.w, cp = a.cp, cg = a.cg;
        pso_elem(xn.x, vn.x, pb.x, g.x, scaled_u24(b1.x, cp), scaled_u24(b2.x, cg), w, lo.x, hi.x);
        pso_elem(xn.y, vn.y, pb.y, g.y, scaled_u24(b1.y, cp), scaled_u24(b2.y, cg), w, lo.y, hi.y);
        pso_elem(xn.z, vn.z, pb.z, g.z, scaled_u24(b1.z, cp), scaled_u24(b2.z, cg), w, lo.z, hi.z);
        pso_elem(xn.w, vn.w, pb.w, g.w, scaled_u24(b1.w, cp), scaled_u24(b2.w, cg), w, lo.w, hi.w);
        zero_pad(xn, vn, q, a.D);
        st_stream<STS>(Xr + q, xn);
        st_stream<STS>(Vr + q, vn);
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

// In the last CTA: gbest update (strict, R-5), hist, or the winner record for
// the exchange.  `t_new` is the index of the population just evaluated.
__device__ void pso_finalize(const PsoArgs& a, unsigned long long key, unsigned long long t_new) {
    Ctl* ctl = a.ctl;
    const long long NQ = a.ld >> 2;
    const bool any = key != ~0ull;
    const long long grow = (long long)(uint32_t)(key & 0xffffffffu);
    const float fmin = any ? unord_f32((uint32_t)(key >> 32)) : __int_as_float(0x7f800000);
    if (a.exchange) {
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

// The rows of one fused PSO generation owned by this thread (lazy pbest + move +
// clip + evaluate + tell); returns this thread's argmin key.  COH: G is re-read
// through L2 (the persistent kernel rewrites it between generations).
template <int P, class G, bool UNI, bool COH>
__device__ __forceinline__ unsigned long long pso_gen_rows(const PsoArgs& a, const RowMap<G>& m,
                                                           unsigned long long t, const float* htab,
                                                           Fit<P>* sh_acc, float* sh_head) {
    const int lane = lane_id();
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
        if (mode_a && a.pf_next) {
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
        MoverPso<UNI, COH> mv(a, ok ? row : 0, (uint32_t)t, pend_cur);
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
    return best;
}

// Fused PSO generation: lazy pbest + move + clip + evaluate + tell + argmin.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, G::WPR > 1 ? EVOX_ROW_MINB : (G::LPR == 4 ? EVOX_PSO_SHORT_MINB : EVOX_MINB))
    k_pso_gen(PsoArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P, G> sh_h;
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    prefetch_first_rows<G>(a.X, a.V, a.rows, a.ld, m.wfirst, m.qb, m.qe);
    pdl_wait();               // the previous generation (G, imp, pf, t) is complete
    pdl_launch_dependents();  // the next generation may be scheduled as our CTAs retire
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const unsigned long long best = pso_gen_rows<P, G, UNI, false>(a, m, t, htab, sh_acc, sh_head);
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key) && !a.fin_kernel) pso_finalize(a, key, t + 1);
}

#ifndef EVOX_WAVE_MINB
#define EVOX_WAVE_MINB 4  // CTAs/SM of the wave kernel (warp-row geometries)
#endif
#ifndef EVOX_ROW_U
#define EVOX_ROW_U 3  // chunks in flight of the wave kernel, CTA-per-row geometry
#endif
#ifndef EVOX_WAVE_PF
#define EVOX_WAVE_PF 3  // warp-row wave kernel: L2 prefetch of the CTA's rows (bit 0 X, V; bit 1 P):
                        // H 0.935 -> 0.974, H-sphere 0.969 -> 0.989 (profiles/r02_ab_wave_pf.txt)
#endif
#ifndef EVOX_WAVE_PF_EF
#define EVOX_WAVE_PF_EF 0  // evict-first hints in the prefetching wave kernel (H: 0.963 with, 0.996 without)
#endif
#ifndef EVOX_WAVE_PF_MAX_LD
#define EVOX_WAVE_PF_MAX_LD 1024
#endif
#ifndef EVOX_WAVE_U
#define EVOX_WAVE_U 2  // chunks in flight per lane group in the wave kernel (warp-row geometries)
#endif

// Fused PSO generation on a "wave" grid: one CTA per row block (every thread at most one
// row), CTAs scheduled by the hardware in row order as slots free up.  Per row it runs
// exactly the code of k_pso_gen (same geometry, reduction order and decisions: bitwise the
// same trajectory); what it drops is the persistent loop's state (prefetch windows,
// next-row flags) and the end-of-grid fence + ticket: a CTA's minimum key goes to
// ctl->gen_key with one relaxed atomicMin, and the gbest publication runs in k_pso_fin,
// ordered after this grid by the kernel boundary (PDL griddepcontrol.wait).  The P load
// of a row waits on its imp flag; X and V of the row are already in flight by then
// (walk_segment's late loads).  Micro (profiles/r02_micro_np3.txt): this schedule streams
// the generation's access pattern at 6.48 TB/s against 6.13-6.33 for a persistent grid.
template <int P, class G, bool UNI, bool PF>
__global__ void __launch_bounds__(256, G::WPR > 1 ? EVOX_ROW_MINB : EVOX_WAVE_MINB)
    k_pso_gen_wave(PsoArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P, G> sh_h;
    __shared__ unsigned long long sh_k[WARPS];
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    const long long row = m.first;  // grid = row units: at most one row per thread
    const bool ok = row < a.rows;
    pdl_wait();               // the previous generation (G, imp, pf, t) is complete
    pdl_launch_dependents();
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const bool pend = ok ? a.imp[row] != 0 : true;
    // PF (chosen on the host only while the grid's tiles fit L2 comfortably: 8 rows x ld x 12 B
    // on ~600 resident CTAs is 58 MB at ld = 1024; at dim 1500 / 2048 / 4096 the prefetch
    // thrashes L2: 0.85 / 0.76 / 0.61-0.76 against 0.88 / 0.83 / 0.72-0.94 without,
    // profiles/r02_wave_threshold.txt)
    if constexpr (PF && G::WPR == 1) {
        // the CTA's rows HBM -> L2 at its start (X, V contiguous; P per row unless pending)
        const long long r0 = (long long)blockIdx.x * G::RPC;
        const long long nr = a.rows - r0 < G::RPC ? a.rows - r0 : G::RPC;
        if ((EVOX_WAVE_PF & 1) && threadIdx.x == 0 && nr > 0) {
            prefetch_l2(a.X + r0 * a.ld, nr * a.ld * 4);
            prefetch_l2(a.V + r0 * a.ld, nr * a.ld * 4);
        }
        if ((EVOX_WAVE_PF & 2) && m.leader && ok && !pend) prefetch_l2(a.P + row * a.ld, a.ld * 4);
    }
    float pf_old = 0.0f;
    if (m.leader && ok) pf_old = a.pf[row];
    unsigned long long best = ~0ull;
    if (m.wfirst < a.rows) {  // warp-uniform (CTA-uniform for WPR > 1)
        MoverPso<UNI, false, !(PF && !EVOX_WAVE_PF_EF)> mv(a, ok ? row : 0, (uint32_t)t, pend);
        Fit<P> acc;
        float hx, tx;
        bool tv;
        NoPrefetch pf;
        walk_segment<P, G>(mv, m.qb, m.qe, a.D, ok, acc, hx, tx, tv, pf, htab);
        const float f = reduce_row<P, G>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
        if (m.leader && ok) {
            const bool imp = f < pf_old;  // per-row tell (A11): strict, NaN never improves
            a.f[row] = f;
            a.imp[row] = imp ? 1 : 0;
            if (imp) a.pf[row] = f;
            best = make_key(f, a.row0 + row);
        }
    }
    best = warp_min_u64(best);
    if (lane_id() == 0) sh_k[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = sh_k[0];
#pragma unroll
        for (int i = 1; i < WARPS; ++i) k = sh_k[i] < k ? sh_k[i] : k;
        if (k != ~0ull) atomicMin(&a.ctl->gen_key, k);
    }
}

#ifndef EVOX_FLAT_K
#define EVOX_FLAT_K 1  // quads per thread per batch of the flat phase (with the tile's L2 prefetch)
#endif
#ifndef EVOX_FLAT_MINB
#define EVOX_FLAT_MINB 4  // its CTAs/SM (register cap)
#endif
#ifndef EVOX_FLAT_EF
#define EVOX_FLAT_EF 0  // evict-first loads and stores in the flat phase (C4r: 0.892 with, 0.909 without)
#endif
#ifndef EVOX_FLAT_PF
#define EVOX_FLAT_PF 3  // bulk L2 prefetch of the CTA's tile at its start: bit 0 X, V; bit 1 P rows
#endif
#ifndef EVOX_FLAT_G32
#define EVOX_FLAT_G32 0  // warp-per-row rows also take k_pso_gen_flat (tiles of 8 rows)
#endif
#ifndef EVOX_FLAT_PF_GRIEWANK
#define EVOX_FLAT_PF_GRIEWANK EVOX_FLAT_PF
#endif
#ifndef EVOX_FLAT_MINB_GRIEWANK
#define EVOX_FLAT_MINB_GRIEWANK EVOX_FLAT_MINB
#endif

// Fused PSO generation for short rows (4 / 8 lanes per row geometries, ld <= 256) on a wave
// grid of one CTA per G::RPC rows, in two phases:
//  1. flat: the CTA's RPC x NQ quads are contiguous in X, V, P, so its threads walk them as one
//     flat range (thread i: quads i, i + 256, ...; EVOX_FLAT_K in flight) -- every warp
//     instruction reads 512 contiguous bytes instead of 4-8 separate 64-byte row pieces, and
//     no lane idles on a row's ragged end.  Each quad is moved by exactly MoverPso::step (same
//     Philox counters (q, global row, t, tag), op order, clip, zero padding, lazy pbest) and its
//     x' is staged in shared memory;
//  2. the geometry's row engine (walk_segment / reduce_row over RowMap<G>, reading the staged
//     x') folds the fitness in the geometry's order: bitwise the f of k_pso_gen (R-11), then
//     the per-row tell and the CTA's argmin key (one relaxed atomicMin; gbest is published by
//     k_pso_fin, as for k_pso_gen_wave).
// The CTA's first act is a bulk L2 prefetch of its whole tile (X, V; P of the rows whose pbest
// copy is not pending), so the DRAM stream never waits on registers, nor on phase 2.
// Micro of this access pattern (scripts/micro/short.cu, profiles/r02_micro_short.txt):
// 6.84 TB/s with Philox against 5.86 for the 4-lanes-per-row persistent walk.  Measured
// (profiles/r02_ab_flat.txt, same box): C4g 0.767 -> 0.842, C4r 0.781 -> 0.911 of the HBM
// peak with the prefetch (0.81 / 0.79 without it; 2 quads per batch / 3 CTAs/SM lose).
// Per-problem knobs (measurement builds).  With x' folded in phase 2, Griewank measured best
// with 6 CTAs/SM and only X/V prefetched (0.874); since the flat phase computes its terms
// (pre_quad) the common defaults win for it too (C4g 0.910, profiles/r02_ab_flat2.txt).
template <int P>
__host__ __device__ constexpr int flat_minb() { return P == GRIEWANK ? EVOX_FLAT_MINB_GRIEWANK : EVOX_FLAT_MINB; }
template <int P>
__host__ __device__ constexpr int flat_pf() { return P == GRIEWANK ? EVOX_FLAT_PF_GRIEWANK : EVOX_FLAT_PF; }

template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, flat_minb<P>()) k_pso_gen_flat(PsoArgs a) {
    static_assert(G::WPR == 1, "flat phase: warp-row geometries only");
    extern __shared__ __align__(128) unsigned char flat_smem_buf[];
    float4* st = reinterpret_cast<float4*>(flat_smem_buf);  // staged tile (+ [ld] htab)
    __shared__ Fit<P> sh_acc[1];
    __shared__ float sh_head[1];
    __shared__ unsigned char sh_pend[G::RPC];
    __shared__ unsigned long long sh_k[WARPS];
    const int NQ = (int)(a.ld >> 2);
    const int tq = G::RPC * NQ;  // staged quads per component
    const float* htab =
        HTable<P, G>::fill(reinterpret_cast<float*>(st + tq * stage_comps<P>()), a.ld);
    const RowMap<G> m(NQ);
    const long long row0 = (long long)blockIdx.x * G::RPC;
    const int nrow = a.rows - row0 < G::RPC ? (int)(a.rows - row0) : G::RPC;
    pdl_wait();               // the previous generation (G, imp, pf, t) is complete
    pdl_launch_dependents();
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const int n = nrow * NQ;
    const float4* Xt = reinterpret_cast<const float4*>(a.X) + row0 * NQ;
    const float4* Vt = reinterpret_cast<const float4*>(a.V) + row0 * NQ;
    const float4* Pt = reinterpret_cast<const float4*>(a.P) + row0 * NQ;
    if (threadIdx.x < nrow) {
        const unsigned char pd = a.imp[row0 + threadIdx.x];
        sh_pend[threadIdx.x] = pd;
#if EVOX_FLAT_PF
        // the whole tile HBM -> L2 at once (X, V contiguous; P per row unless its pbest copy
        // is pending): the DRAM stream runs ahead of the register loads, phase 2 included
        if ((flat_pf<P>() & 1) && threadIdx.x == 0) {
            prefetch_l2(Xt, (long long)n * 16);
            prefetch_l2(Vt, (long long)n * 16);
        }
        if ((flat_pf<P>() & 2) && !pd) prefetch_l2(Pt + threadIdx.x * NQ, (long long)NQ * 16);
#endif
    }
    const long long row = m.first;
    const bool ok = row < a.rows;
    float pf_old = 0.0f;
    if (m.leader && ok) pf_old = a.pf[row];
    __syncthreads();
    // phase 1: flat walk of the tile (r = i / NQ exactly: i * NQ < 2^32)
    const uint32_t magic = (uint32_t)(0xffffffffu / (uint32_t)NQ) + 1u;
    constexpr int K = EVOX_FLAT_K;
    for (int b = 0; b < n; b += 256 * K) {
        float4 x[K], v[K], p[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = b + 256 * k + (int)threadIdx.x;
            if (i < n) {
                x[k] = ld_stream<EVOX_FLAT_EF != 0>(Xt + i);
                v[k] = ld_stream<EVOX_FLAT_EF != 0>(Vt + i);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = b + 256 * k + (int)threadIdx.x;
            if (i < n) {
                const int r = (int)__umulhi((uint32_t)i, magic);
                if (!sh_pend[r]) p[k] = ld_stream<EVOX_FLAT_EF != 0>(Pt + i);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = b + 256 * k + (int)threadIdx.x;
            if (i < n) {
                const int r = (int)__umulhi((uint32_t)i, magic);
                const int q = i - r * NQ;
                const int o = i - q;  // r * NQ
                MoverPso<UNI, false, EVOX_FLAT_EF != 0> mv(
                    a, const_cast<float4*>(Xt) + o, const_cast<float4*>(Vt) + o,
                    const_cast<float4*>(Pt) + o, (uint32_t)(a.row0 + row0) + (uint32_t)r,
                    (uint32_t)t, sh_pend[r] != 0);
                mv.x[0] = x[k];
                mv.v[0] = v[k];
                mv.p[0] = p[k];
                stage_quad<P>(st, tq, i, q, mv.step(0, q), htab);
            }
        }
    }
    __syncthreads();
    // phase 2: the geometry's fitness fold over the staged rows, tell, argmin key
    unsigned long long best = ~0ull;
    {
        const float f = fold_staged_row<P, G>(st, tq, ok ? (int)(row - row0) : 0, NQ, a.D, ok,
                                              htab, sh_acc, sh_head);
        if (m.leader && ok) {
            const bool imp = f < pf_old;  // per-row tell (A11): strict, NaN never improves
            a.f[row] = f;
            a.imp[row] = imp ? 1 : 0;
            if (imp) a.pf[row] = f;
            best = make_key(f, a.row0 + row);
        }
    }
    best = warp_min_u64(best);
    if (lane_id() == 0) sh_k[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = sh_k[0];
#pragma unroll
        for (int i = 1; i < WARPS; ++i) k = sh_k[i] < k ? sh_k[i] : k;
        if (k != ~0ull) atomicMin(&a.ctl->gen_key, k);
    }
}

// Copy `n` quads src -> dst with this grid's threads, 4 float4 loads in flight per thread.
__device__ __forceinline__ void grid_copy4(float4* dst, const float4* src, long long n) {
    const long long nth = (long long)gridDim.x * blockDim.x;
    long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + 3 * nth < n; q += 4 * nth) {
        const float4 v0 = __ldcg(src + q), v1 = __ldcg(src + q + nth);
        const float4 v2 = __ldcg(src + q + 2 * nth), v3 = __ldcg(src + q + 3 * nth);
        dst[q] = v0;
        dst[q + nth] = v1;
        dst[q + 2 * nth] = v2;
        dst[q + 3 * nth] = v3;
    }
    for (; q < n; q += nth) dst[q] = __ldcg(src + q);
}

// gbest publication after a generation (or tell) kernel that only reduced the generation's
// minimum key into ctl->gen_key (PsoArgs.fin_kernel): the last-CTA step of k_pso_gen, run by
// a small grid so the row copies are spread over several SMs.
//  * one rank: strict improvement -> G <- X[i*], gf, gidx; hist; t.
//  * NCCL exchange: this rank's winner record {key; row} for the all-gather.
//  * peer exchange, KEY FIRST (A13; the paper's per-iteration all-gather of fitness,
//    P:583-587): a rank whose local minimum can still improve gbest stages its row in its
//    OWN mailbox slot[par][rank] (local copy); every rank then writes only its 8-byte key +
//    release flag into every rank's mailbox; each rank picks the minimum key (lowest global
//    index on ties, R-11) and, on a strict improvement over gf, pulls that ONE row from the
//    winner's mailbox over NVLink into G.  One row crosses NVLink per rank per improving
//    generation (was: W rows pushed per rank every generation).  Parity double-buffering:
//    a rank overwrites slot[par] only at t_new + 2, after every peer published t_new + 1,
//    i.e. finished this pull (stream order).  Bounded waits (ctl->err, no hang).
__global__ void __launch_bounds__(256) k_pso_fin(PsoArgs a, long long t_arg) {
    __shared__ int sh_sel;
    pdl_wait();
    pdl_launch_dependents();
    Ctl* ctl = a.ctl;
    // every CTA reads the control block BEFORE CTA 0 rewrites it (arrival counter below)
    const unsigned long long t_new =
        t_arg >= 0 ? (unsigned long long)t_arg : *(volatile unsigned long long*)&ctl->t + 1;
    const unsigned long long key = *(volatile unsigned long long*)&ctl->gen_key;
    const float gf_old = *(volatile float*)&ctl->gf;
    const long long NQ = a.ld >> 2;
    const bool any = key != ~0ull;
    const long long grow = (long long)(uint32_t)(key & 0xffffffffu);
    const float fmin = any ? unord_f32((uint32_t)(key >> 32)) : __int_as_float(0x7f800000);
    const float4* xrow = reinterpret_cast<const float4*>(a.X + (any ? grow - a.row0 : 0) * a.ld);
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    const int par = (int)(t_new & 1);
    const unsigned long long flag = t_new + 1;  // mailboxes start zeroed: 0 = nothing yet
    const long long my_off = ((long long)par * a.world + a.rank) * a.mb_slot;
    if (a.peer) {  // 1. a possible winner stages its row in its own mailbox (local HBM)
        if (any && fmin < gf_old)
            grid_copy4(reinterpret_cast<float4*>(a.mbox[a.rank] + my_off + 16), xrow, NQ);
    } else if (a.exchange) {  // NCCL: winner record {u64 key; pad; f32 row[ld]} of this rank
        unsigned char* rec = a.rec + (long long)a.rank * a.rec_stride;
        if (any) {
            grid_copy4(reinterpret_cast<float4*>(rec + 16), xrow, NQ);
        } else {
            for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < NQ;
                 q += (long long)gridDim.x * blockDim.x)
                reinterpret_cast<float4*>(rec + 16)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (lead) *reinterpret_cast<unsigned long long*>(rec) = key;
    } else if (any && fmin < gf_old) {  // one rank: strict improvement (R-5)
        grid_copy4(reinterpret_cast<float4*>(a.G), xrow, NQ);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.peer) __threadfence_system();
        atomicAdd(&ctl->fin_cnt, 1u);
    }
    if (!lead && !a.peer) return;
    unsigned long long t0 = 0;
    if (lead) {
        t0 = globaltimer_ns();
        while (ld_acquire_gpu_u32(&ctl->fin_cnt) != gridDim.x) {  // every CTA has read ctl
            if (globaltimer_ns() - t0 > a.peer_timeout_ns) { ctl->err = 1; break; }
            __nanosleep(64);
        }
        ctl->fin_cnt = 0u;
        ctl->gen_key = ~0ull;
        ctl->ticket = 0u;
        ctl->t = t_new;
        if (!a.peer) {
            if (!a.exchange) {
                if (any && fmin < gf_old) {
                    ctl->gf = fmin;
                    ctl->gidx = grow;
                }
                ctl->hist[t_new] = fmin;
            }
            return;
        }
        // 2. the 8-byte key into every rank's slot, then the release flags
        for (int p = 0; p < a.world; ++p)
            *reinterpret_cast<unsigned long long*>(a.mbox[p] + my_off + 8) = key;
        __threadfence_system();
        for (int p = 0; p < a.world; ++p)
            st_release_sys(reinterpret_cast<unsigned long long*>(a.mbox[p] + my_off), flag);
        // 3. every rank's key of this generation, from our own mailbox
        unsigned long long kmin = ~0ull;
        int w = -1;
        for (int r = 0; r < a.world; ++r) {
            const unsigned char* slot =
                a.mbox[a.rank] + ((long long)par * a.world + r) * a.mb_slot;
            while (ld_acquire_sys(reinterpret_cast<const unsigned long long*>(slot)) != flag) {
                if (globaltimer_ns() - t0 > a.peer_timeout_ns) { ctl->err = 1; break; }
                __nanosleep(128);
            }
            const unsigned long long kr =
                __ldcg(reinterpret_cast<const unsigned long long*>(slot + 8));
            if (kr < kmin) { kmin = kr; w = r; }
        }
        const bool ok = kmin != ~0ull;
        const float gmin = ok ? unord_f32((uint32_t)(kmin >> 32)) : __int_as_float(0x7f800000);
        const bool better = ok && gmin < gf_old;  // strict improvement (R-5)
        if (better) {
            ctl->gf = gmin;
            ctl->gidx = (long long)(uint32_t)(kmin & 0xffffffffu);
        }
        ctl->hist[t_new] = gmin;
        ctl->fin_sel = better ? w : -1;
        __threadfence();
        st_release_gpu_u32(&ctl->fin_epoch, (unsigned int)flag);
    }
    // 4. every CTA: the decision, then its slice of the winner's staged row -> G
    if (threadIdx.x == 0) {
        t0 = globaltimer_ns();
        while (ld_acquire_gpu_u32(&ctl->fin_epoch) != (unsigned int)flag) {
            if (globaltimer_ns() - t0 > 2 * a.peer_timeout_ns) { ctl->err = 1; break; }
            __nanosleep(64);
        }
        sh_sel = *(volatile int*)&ctl->fin_sel;
    }
    __syncthreads();
    if (sh_sel >= 0)
        grid_copy4(reinterpret_cast<float4*>(a.G),
                   reinterpret_cast<const float4*>(a.mbox[sh_sel] +
                                                   ((long long)par * a.world + sh_sel) * a.mb_slot + 16),
                   NQ);
}

#ifndef EVOX_PSO_SHORT_U
#define EVOX_PSO_SHORT_U U  // chunks in flight of the generation kernel for short rows (<= 256)
#endif
// The persistent generation kernel's geometry: the row geometry of ld with its own chunk
// count for short rows (a lane's quad order, hence every reduction order, is unchanged).
#define EVOX_PSO_GEOM(G_) Geom<G_::LPR, G_::WPR, G_::LPR <= 8 ? EVOX_PSO_SHORT_U : G_::NU, G_::EFL>

// The cooperative kernel's partial last round ("tail"): rows [rw, rows) are fewer than the
// grid's row slots, so instead of a few warps walking one more whole row each while the rest of
// the grid waits at the barrier, every CTA takes <= TR of them as one flat tile (the phases of
// k_pso_gen_flat: all 256 threads move the tile's quads and stage their fitness pre-terms, then
// the geometry's lane groups fold each row in the geometry's order -- bitwise the row walk).
// Called by every thread of the CTA (CTA-local barriers); returns this thread's argmin key.
template <int P, class G, bool UNI>
__device__ __forceinline__ unsigned long long pso_tail_tile(const PsoArgs& a, long long row0,
                                                            int nrow, unsigned long long t,
                                                            float4* st, const float* htab,
                                                            Fit<P>* sh_acc, float* sh_head,
                                                            unsigned char* sh_pend) {
    const int NQ = (int)(a.ld >> 2);
    const int tq = nrow * NQ;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    const int lr = wid * G::RPW + lane / G::LPR;  // this lane group's row in the tile
    const bool ok = lr < nrow;
    const bool lead = ok && (lane & (G::LPR - 1)) == 0;
    if ((int)threadIdx.x < nrow) sh_pend[threadIdx.x] = a.imp[row0 + threadIdx.x];
    float pf_old = 0.0f;
    if (lead) pf_old = a.pf[row0 + lr];
    __syncthreads();
    const uint32_t magic = (uint32_t)(0xffffffffu / (uint32_t)NQ) + 1u;  // i / NQ exactly
    const float4* Xt = reinterpret_cast<const float4*>(a.X) + row0 * NQ;
    const float4* Vt = reinterpret_cast<const float4*>(a.V) + row0 * NQ;
    const float4* Pt = reinterpret_cast<const float4*>(a.P) + row0 * NQ;
    for (int i = threadIdx.x; i < tq; i += 256) {
        const int r = (int)__umulhi((uint32_t)i, magic);
        const int q = i - r * NQ;
        const bool pend = sh_pend[r] != 0;
        const int o = i - q;  // r * NQ
        MoverPso<UNI, true> mv(a, const_cast<float4*>(Xt) + o, const_cast<float4*>(Vt) + o,
                               const_cast<float4*>(Pt) + o, (uint32_t)(a.row0 + row0) + (uint32_t)r,
                               (uint32_t)t, pend);
        mv.x[0] = ld_stream<G::EFL>(Xt + i);
        mv.v[0] = ld_stream<G::EFL>(Vt + i);
        if (!pend) mv.p[0] = ld_stream<G::EFL>(Pt + i);
        stage_quad<P>(st, tq, i, q, mv.step(0, q), htab);
    }
    __syncthreads();
    unsigned long long best = ~0ull;
    if (wid * G::RPW < nrow) {  // warp-uniform: warps without rows skip the fold
        const float f = fold_staged_row<P, G>(st, tq, ok ? lr : 0, NQ, a.D, ok, htab, sh_acc,
                                              sh_head);
        if (lead) {
            const long long row = row0 + lr;
            const bool imp = f < pf_old;  // per-row tell (A11): strict, NaN never improves
            a.f[row] = f;
            a.imp[row] = imp ? 1 : 0;
            if (imp) a.pf[row] = f;
            best = make_key(f, a.row0 + row);
        }
    }
    __syncthreads();  // staging and sh_pend are reused next generation
    return best;
}

#ifndef EVOX_MID_SPIN_NS
#define EVOX_MID_SPIN_NS 32  // back-off of the arrival spin (measurement knob)
#endif
#ifndef EVOX_MID_ALL_FENCE
#define EVOX_MID_ALL_FENCE 0  // every thread fences before the arrival (measurement knob)
#endif
#ifndef EVOX_MID_LOCAL_G
#define EVOX_MID_LOCAL_G 1  // warp-row geometries: replicated gbest decision + CTA-local G copy
#endif

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// The cooperative kernel's generations for warp-row geometries, without a "last CTA" on the
// critical path: every CTA folds its minimum key into mkey[t % 3], arrives at a monotonic
// counter and, once all have arrived, takes the SAME gbest decision from the same key and its
// register copy of gf (strict improvement, R-5), and refreshes its own shared-memory copy of G
// from the winner row (read through L2).  CTA 0 alone writes the host-visible state (G, gf,
// gidx, hist, t) and resets the key slot of generation t + 2 (every CTA has read it: they all
// passed this generation's barrier after reading it at the previous one).  Invariant between
// launches: mkey[(t+1) % 3] and mkey[(t+2) % 3] are ~0.  Same decisions as pso_finalize: the
// trajectory is bitwise the stepwise one.
template <int P, class G, bool UNI>
__device__ __forceinline__ void k_pso_run_mid_local(const PsoArgs& a, long long n, long long rw,
                                                    int tr) {
    __shared__ Fit<P> sh_acc[1];
    __shared__ float sh_head[1];
    __shared__ __align__(16) HStore<P, G> sh_h;
    __shared__ unsigned char sh_pend[G::RPC];
    __shared__ unsigned long long sh_k[WARPS];
    __shared__ unsigned long long sh_key;
    __shared__ int sh_abort;
    extern __shared__ __align__(128) unsigned char mid_tail_smem[];  // [G copy][tail staging]
    float* sG = reinterpret_cast<float*>(mid_tail_smem);
    float4* tail_st = reinterpret_cast<float4*>(mid_tail_smem + ((a.ld * 4 + 127) / 128) * 128);
    const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
    const RowMap<G> m(a.ld >> 2);
    Ctl* ctl = a.ctl;
    for (long long j = threadIdx.x; j < a.ld; j += blockDim.x) sG[j] = a.G[j];
    float gf = *(volatile float*)&ctl->gf;
    // nobody arrives before every CTA has read the base: a whole generation comes first
    const unsigned int base = *(volatile unsigned int*)&ctl->arrive;
    unsigned long long t = *(volatile unsigned long long*)&ctl->t;
    __syncthreads();
    PsoArgs aw = a;  // rows [0, rw): the warps' whole rounds, G from shared memory
    aw.rows = rw;
    aw.G = sG;
    PsoArgs at = a;  // rows [rw, rows): the tail tiles
    at.G = sG;
    const long long NQ = a.ld >> 2;
    for (long long g = 0; g < n; ++g, ++t) {
        unsigned long long best = pso_gen_rows<P, G, UNI, true>(aw, m, t, htab, sh_acc, sh_head);
        if (tr > 0) {
            const long long row0 = rw + (long long)blockIdx.x * tr;
            const long long left = a.rows - row0;
            const int nrow = left < tr ? (left > 0 ? (int)left : 0) : tr;
            if (nrow > 0) {  // CTA-uniform
                const unsigned long long k =
                    pso_tail_tile<P, G, UNI>(at, row0, nrow, t, tail_st, htab, sh_acc, sh_head, sh_pend);
                best = k < best ? k : best;
            }
        }
#if EVOX_MID_PF
        if (g + 1 < n && lane_id() == 0 && m.wfirst < a.rows) {
            const long long nr = a.rows - m.wfirst < G::RPW ? a.rows - m.wfirst : G::RPW;
            const long long o = m.wfirst * a.ld * 4;
            long long bytes = nr * a.ld * 4;
            if (bytes > 64 * 1024) bytes = 64 * 1024;
            prefetch_l2(reinterpret_cast<const char*>(a.X) + o, bytes);
            prefetch_l2(reinterpret_cast<const char*>(a.V) + o, bytes);
            prefetch_l2(reinterpret_cast<const char*>(a.P) + o, bytes);
        }
#endif
        // arrival: this CTA's rows visible device-wide (bar.sync, then thread 0's cumulative
        // fence -- the grid-sync pattern), its minimum in the generation's slot
        best = warp_min_u64(best);
        if (lane_id() == 0) sh_k[threadIdx.x >> 5] = best;
#if EVOX_MID_ALL_FENCE
        __threadfence();
#endif
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long k = sh_k[0];
#pragma unroll
            for (int i = 1; i < WARPS; ++i) k = sh_k[i] < k ? sh_k[i] : k;
            unsigned long long* slot = &ctl->mkey[t % 3];
            if (k != ~0ull) atomicMin(slot, k);
            __threadfence();
            atomicAdd(&ctl->arrive, 1u);
            const unsigned int target = base + (unsigned int)(g + 1) * gridDim.x;
            int abort = 0;
            const unsigned long long t0 = globaltimer_ns();
            while ((int)(ld_acquire_gpu_u32(&ctl->arrive) - target) < 0) {
                if (globaltimer_ns() - t0 > 10000000000ull) {  // 10 s: not co-resident
                    ctl->err = 1;
                    abort = 1;
                    break;
                }
                if (EVOX_MID_SPIN_NS > 0) __nanosleep(EVOX_MID_SPIN_NS);
            }
            sh_key = ld_acquire_gpu_u64(slot);
            sh_abort = abort;
        }
        __syncthreads();
        if (sh_abort) return;
        // the replicated decision (pso_finalize's): strict improvement over gf
        const unsigned long long key = sh_key;
        const bool any = key != ~0ull;
        const long long grow = (long long)(uint32_t)(key & 0xffffffffu);
        const float fmin = any ? unord_f32((uint32_t)(key >> 32)) : __int_as_float(0x7f800000);
        const bool better = any && fmin < gf;
        if (better) {
            const float4* src = reinterpret_cast<const float4*>(a.X + (grow - a.row0) * a.ld);
            float4* dst = reinterpret_cast<float4*>(sG);
            float4* Gg = reinterpret_cast<float4*>(a.G);
            for (long long q = threadIdx.x; q < NQ; q += blockDim.x) {
                const float4 v = __ldcg(src + q);
                dst[q] = v;
                if (blockIdx.x == 0) Gg[q] = v;
            }
            gf = fmin;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->mkey[(t + 2) % 3] = ~0ull;
            if (better) {
                ctl->gf = fmin;
                ctl->gidx = grow;
            }
            ctl->hist[t + 1] = fmin;
            ctl->t = t + 1;
        }
        __syncthreads();  // the shared G copy is complete
    }
}

#ifndef EVOX_MID_U
#define EVOX_MID_U 4     // chunks in flight of the cooperative kernel, warp-per-row geometry
#endif
#ifndef EVOX_MID_MINB
#define EVOX_MID_MINB EVOX_MINB  // its CTAs/SM (register cap), warp-per-row geometry
#endif
#ifndef EVOX_MID_TAIL
#define EVOX_MID_TAIL 32768  // max staging bytes per CTA of the tail split (0: off)
#endif
#ifndef EVOX_MID_PF
#define EVOX_MID_PF 1  // k_pso_run_mid: L2 prefetch of the next generation's first rows
#endif

// Persistent PSO for mid-size populations (e.g. C2: 1e4 x 1000,
// where a ~7 us per-launch fixed cost plus the launch gap is 20 % of a generation,
// profiles/r01_c2_pop_sweep.txt): all n generations in ONE cooperative launch of
// the resident grid, a grid-wide release/acquire barrier on ctl->bar between
// generations instead of a kernel boundary.  Rows, reduction order and decisions
// are those of k_pso_gen (same geometry, same per-row code), so the trajectory is
// bitwise the stepwise one.  The barrier spin is bounded (ctl->err, no hang).
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, G::LPR == 4 ? EVOX_PSO_SHORT_MINB
                                                   : (G::WPR == 1 ? EVOX_MID_MINB : EVOX_MINB))
    k_pso_run_mid(PsoArgs a, long long n, long long rw, int tr) {
    if constexpr (G::WPR == 1 && EVOX_MID_LOCAL_G) {
        k_pso_run_mid_local<P, G, UNI>(a, n, rw, tr);
    } else {
        __shared__ Fit<P> sh_acc[G::WPR];
        __shared__ float sh_head[G::WPR];
        __shared__ __align__(16) HStore<P, G> sh_h;
        __shared__ int sh_abort;
        __shared__ unsigned char sh_pend[G::WPR == 1 ? G::RPC : 1];
        extern __shared__ __align__(128) unsigned char mid_tail_smem[];  // tail staging (tr > 0)
        const float* htab = HTable<P, G>::fill(sh_h.v, a.ld);
        const RowMap<G> m(a.ld >> 2);
        Ctl* ctl = a.ctl;
        // nobody writes ctl->bar before every CTA has arrived at the first grid_argmin,
        // so every CTA reads the same base
        const unsigned int base = *(volatile unsigned int*)&ctl->bar;
        unsigned long long t = *(volatile unsigned long long*)&ctl->t;
        // rows [0, rw) are walked by the warps' whole rounds; with tr > 0, rows [rw, rows) are the
        // tail tiles, tr rows per CTA (pso_tail_tile)
        PsoArgs aw = a;
        aw.rows = rw;
        for (long long g = 0; g < n; ++g, ++t) {
            unsigned long long best = pso_gen_rows<P, G, UNI, true>(aw, m, t, htab, sh_acc, sh_head);
            if constexpr (G::WPR == 1) {
                if (tr > 0) {
                    const long long row0 = rw + (long long)blockIdx.x * tr;
                    const long long left = a.rows - row0;
                    const int nrow = left < tr ? (left > 0 ? (int)left : 0) : tr;
                    if (nrow > 0) {  // CTA-uniform
                        const unsigned long long k = pso_tail_tile<P, G, UNI>(
                            a, row0, nrow, t, reinterpret_cast<float4*>(mid_tail_smem), htab, sh_acc,
                            sh_head, sh_pend);
                        best = k < best ? k : best;
                    }
                }
            }
    #if EVOX_MID_PF
            // the warp's first rows of the next generation (its own, already final) go to L2
            // while the grid drains the tail of this one (the pbest row only if not pending)
            if (g + 1 < n && lane_id() == 0 && m.wfirst < a.rows) {
                const long long nr = a.rows - m.wfirst < G::RPW ? a.rows - m.wfirst : G::RPW;
                const long long o = m.wfirst * a.ld * 4 + m.qb * 16;
                long long bytes = G::WPR == 1 ? nr * a.ld * 4 : (m.qe - m.qb) * 16;
                if (bytes > 64 * 1024) bytes = 64 * 1024;
                prefetch_l2(reinterpret_cast<const char*>(a.X) + o, bytes);
                prefetch_l2(reinterpret_cast<const char*>(a.V) + o, bytes);
                prefetch_l2(reinterpret_cast<const char*>(a.P) + o, bytes);
            }
    #endif
            unsigned long long key;
            const unsigned int target = base + (unsigned int)g + 1u;
            if (grid_argmin(ctl, best, &key)) {
                pso_finalize(a, key, t + 1);  // G, gf, gidx, hist; gen_key/ticket reset; t
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    st_release_gpu_u32(&ctl->bar, target);
                }
            } else if (g + 1 < n) {
                if (threadIdx.x == 0) {
                    int abort = 0;
                    const unsigned long long t0 = globaltimer_ns();
                    while (ld_acquire_gpu_u32(&ctl->bar) != target) {
                        if (globaltimer_ns() - t0 > 10000000000ull) {  // 10 s: not co-resident
                            ctl->err = 1;
                            abort = 1;
                            break;
                        }
                        __nanosleep(64);
                    }
                    sh_abort = abort;
                }
                __syncthreads();
                if (sh_abort) return;
            }
        }
    }
}


// Persistent single-CTA PSO for tiny populations (latency-bound, e.g. C1:
// 100 x 10): all n generations in one launch, a CTA barrier instead of the
// grid-wide argmin.  Per-row arithmetic, reduction order and decisions are
// those of k_pso_gen, so the trajectory is bitwise identical.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256) k_pso_run_small(PsoArgs a, long long n_gens) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P, G> sh_h;
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
    __shared__ __align__(16) HStore<P, G> sh_h;
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
    if (grid_argmin(a.ctl, best, &key) && !a.fin_kernel) pso_finalize(a, key, t + 1);
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
    if (grid_argmin(a.ctl, best, &key) && !a.fin_kernel) pso_finalize(a, key, t);
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


}  // namespace

cudaError_t launch_pso_init(const PsoArgs& a, cudaStream_t st) {
    const long long total = a.rows * (a.ld >> 2);
    long long g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    k_pso_init<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Populations beyond the persistent cooperative kernel's range (> 2^25 elements).
constexpr long long BIG = 1LL << 25;

// Warp-per-row rows of a big population: no next-row L2 prefetch (it re-read 2.9 % of the
// bytes and cost 4 points at H: 0.863 -> 0.900 without it) and 4 waves of resident CTAs
// (+0.6 points); short rows (4 / 8 lanes per row) and L2-sized populations keep the
// prefetch (C4g 0.764 vs 0.706 without; C2 0.678 vs 0.637), profiles/r02_pf.txt.
#ifndef EVOX_PF_NEXT
#define EVOX_PF_NEXT -1  // measurement builds: 0 / 1 force the mode-A prefetch off / on
#endif
bool pso_prefetch_next(long long ld, long long rows) {
    if (EVOX_PF_NEXT >= 0) return EVOX_PF_NEXT != 0;
    return !(geom_id(ld) == 1 && rows * ld > BIG);
}

#ifndef EVOX_WAVE_MIN_WAVES
#define EVOX_WAVE_MIN_WAVES 3  // minimum waves of CTAs for the warp-per-row wave grid
#endif
#ifndef EVOX_WAVE_GRIEWANK
#define EVOX_WAVE_GRIEWANK 0  // measurement builds: Griewank's warp-per-row rows on the wave grid
#endif
#ifndef EVOX_WAVE
// which big populations take the wave grid (bit k: geometry id k; measurement builds may
// change it).  Measured same box (profiles/r02_ab_wave_h.txt): warp-per-row rows with 2 chunks
// in flight and 4 CTAs/SM: H (Ackley) 0.894 -> 0.924, Sphere 0.913 -> 0.971, Rastrigin
// 0.903 -> 0.939, Rosenbrock 0.898 -> 0.915 of the HBM peak; CTA-per-row (C5) 0.895 -> 0.923;
// short rows (4 / 8 lanes per row) run k_pso_gen_flat on the same grid (C4g 0.767 -> 0.842,
// C4r 0.781 -> 0.911).
#define EVOX_WAVE ((1 << 0) | (1 << 1) | (1 << 2) | (1 << 3))
#endif
bool pso_wave(int problem, long long ld, long long rows, int device) {
    const int g = geom_id(ld);
    if (rows * ld <= BIG || !((EVOX_WAVE >> g) & 1)) return false;
    // warp-per-row rows: the wave grid pays off only over enough waves of CTAs -- with few
    // (pop 1e4 x dim 4096: 1,250 CTAs of 8 rows on 592 slots = 2.1 waves: 0.72 vs 0.79; dim 3000
    // at 2.5 waves 0.74 vs 0.76; dim 2048 at 4.2 waves 0.83 vs 0.80) its last partial wave idles
    // most of the GPU, where the persistent walk spreads the rows over its warps.  The flat and
    // CTA-per-row grids win from 4.5 waves down (profiles/r02_wave_threshold.txt).
    if (g == 1) {
        const long long units = (rows + 7) / 8;
        const long long slots = (long long)sm_count(device) * EVOX_WAVE_MINB;
        if (units < (long long)EVOX_WAVE_MIN_WAVES * slots) return false;
    }
    if (g == 0 || g == 3) return true;  // short rows: k_pso_gen_flat
    // Griewank's warp-row kernels keep a 16 KB shared-memory column table per CTA: at 4 CTAs/SM
    // that takes the L1 the streaming loads need (0.874 -> 0.801): persistent grid
    return !(problem == GRIEWANK && g == 1 && !EVOX_WAVE_GRIEWANK);
}

int pso_gen_grid(int problem, long long ld, long long rows, int device, bool wave) {
    int g = 1;
    if (wave) {
        EVOX_DISPATCH_GEOM(ld, { g = (int)row_units<G_>(rows); });
        return g;
    }
    const int waves = geom_id(ld) == 1 && rows * ld > BIG ? 4 : 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        using GP_ = EVOX_PSO_GEOM(G_);
        g = grid_for((const void*)k_pso_gen<P_, GP_, true>, row_units<GP_>(rows), device, waves);
    }));
    return g;  // the TMA variant uses the same grid (2 CTAs/SM: 2 x 96 KB of staging)
}

// The TMA-staged kernel is an opt-in variant (EVOX_FLAG_TMA) of the warp-per-row
// geometry: measured 4-5 points BELOW the LDG kernel at H and C2.
static bool use_tma(long long ld, bool tma) { return tma && geom_id(ld) == 1 && U == 4; }

template <class K>
static void tma_attr(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM);
}

cudaError_t launch_pso_gen(int problem, const PsoArgs& a, int grid, cudaStream_t st, bool tma,
                           bool wave) {
    cudaError_t e = cudaSuccess;
    if (wave && !use_tma(a.ld, tma)) {
        // the wave kernel keeps fewer chunks in flight (registers for 3 CTAs/SM); the chunk
        // count never changes a lane's quad order, so the reduction order is the geometry's
        EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
            if constexpr (G_::WPR == 1 && (G_::LPR <= 8 || EVOX_FLAT_G32)) {
                // short rows: flat tile walk + the geometry's fitness fold (bitwise k_pso_gen)
                const size_t smem = flat_stage_bytes<P_>(G_::RPC, a.ld);
                if (smem > 48 * 1024)
                    cudaFuncSetAttribute(k_pso_gen_flat<P_, G_, U_>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                e = launch_pdl(k_pso_gen_flat<P_, G_, U_>, grid, a, st, smem);
            } else if (G_::WPR == 1 && EVOX_WAVE_PF && a.ld <= EVOX_WAVE_PF_MAX_LD) {
                // tile prefetch; default-policy loads and stores (the prefetched lines stay in L2)
                using GWP_ = Geom<G_::LPR, 1, EVOX_WAVE_U, (EVOX_WAVE_PF_EF != 0)>;
                e = launch_pdl(k_pso_gen_wave<P_, GWP_, U_, true>, grid, a, st);
            } else {
                using GW_ = Geom<G_::LPR, G_::WPR, G_::WPR == 1 ? EVOX_WAVE_U : EVOX_ROW_U, G_::EFL>;
                e = launch_pdl(k_pso_gen_wave<P_, GW_, U_, false>, grid, a, st);
            }
        })));
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    if (use_tma(a.ld, tma)) {
        EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, {
            tma_attr(k_pso_gen_tma<P_, U_>);
            e = launch_pdl(k_pso_gen_tma<P_, U_>, grid, a, st, TMA_SMEM);
        }));
    } else {
        EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
            using GP_ = EVOX_PSO_GEOM(G_);
            e = launch_pdl(k_pso_gen<P_, GP_, U_>, grid, a, st);
        })));
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

// One CTA walking the whole population beats the resident cooperative grid (~11 us per
// generation at any small size) only below ~2^14 elements: pop 100 x dim 128 8.9 us, x 512
// 29 us per generation in one CTA (profiles/r02_sweeps.txt); C1 (100 x 10) stays here.
bool pso_small(long long rows, long long ld) { return rows * ld <= 16384; }

// Mid-size populations run n generations in one cooperative launch (k_pso_run_mid);
// beyond 2^25 elements a generation is long enough that the launch cost is noise.
bool pso_mid(long long rows, long long ld) { return rows * ld <= BIG; }

cudaError_t launch_pso_run_mid(int problem, const PsoArgs& a, long long n, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaSuccess;
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
        using GM_ = Geom<G_::LPR, G_::WPR, G_::LPR == 32 && G_::WPR == 1 ? EVOX_MID_U : G_::NU,
                         G_::EFL>;
        const void* fn = (const void*)k_pso_run_mid<P_, GM_, U_>;
        // the tail split: the rows beyond the grid's whole rounds as flat tiles of <= tr rows
        // per CTA, when their staging fits EVOX_MID_TAIL bytes (warp-row geometries)
        const size_t gcopy = (GM_::WPR == 1 && EVOX_MID_LOCAL_G) ? (size_t)((a.ld * 4 + 127) / 128) * 128 : 0;
        size_t smem = gcopy;
        long long rw = a.rows;
        int tr = 0;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + 32768));
        int grid = 1;
        {
            int per_sm = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
            if (per_sm < 1) per_sm = 1;
            long long g = (long long)sm_count(dev) * per_sm;  // resident grid only
            const long long units = row_units<G_>(a.rows);
            grid = (int)(units < g ? units : g);
        }
        if (GM_::WPR == 1 && EVOX_MID_TAIL > 0) {
            const long long slots = (long long)grid * GM_::RPC;  // rows per round of the grid
            const long long full = a.rows / slots * slots;
            const long long tail = a.rows - full;
            const long long t_r = (tail + grid - 1) / grid;
            const size_t bytes = (size_t)t_r * (size_t)a.ld * 4 * stage_comps<P_>();
            if (tail > 0 && t_r <= GM_::RPC && bytes <= (size_t)EVOX_MID_TAIL) {
                int per_sm = 1;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, gcopy + bytes);
                if ((long long)per_sm * sm_count(dev) >= grid) {  // still co-resident
                    rw = full;
                    tr = (int)t_r;
                    smem = gcopy + bytes;
                }
            }
        }
        PsoArgs aa = a;
        long long nn = n;
        void* args[] = {&aa, &nn, &rw, &tr};
        e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(256), args, smem, st);
    })));
    return e != cudaSuccess ? e : cudaGetLastError();
}

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
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && a.fin_kernel) e = launch_pso_fin(a, (long long)t, st);
    return e;
}

// One CTA per 16 KB of the row (at most 64): the staged / pulled rows are copied by a few
// SMs, so even a 400 KB row (C5) moves in a few microseconds.
cudaError_t launch_pso_fin(const PsoArgs& a, long long t_new, cudaStream_t st) {
    long long g = (a.ld * 4 + 16383) / 16384;
    if (g > 64) g = 64;
    if (g < 1) g = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = EVOX_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_pso_fin, a, t_new);
    return e != cudaSuccess ? e : cudaGetLastError();
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


}  // namespace evox
