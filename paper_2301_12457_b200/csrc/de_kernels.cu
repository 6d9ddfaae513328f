// de_kernels.cu -- DE/rand/1/bin (R-14): double-buffered population, rejection-
// sampled donors (optionally across shards through peer memory).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "evox_device.cuh"
#include "evox_internal.h"
#include "row_engine.cuh"

namespace evox {

namespace {

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
    __device__ __forceinline__ void load(int u, int q) {
        x[u] = ld_stream<EF>(Xi + q);
        xa[u] = __ldcg(Xa + q);  // donors: random rows, may be re-read by other targets
        xb[u] = __ldcg(Xb + q);
        xc[u] = __ldcg(Xc + q);
    }
    template <bool EF>
    __device__ __forceinline__ void load_late(int, int) {}
    __device__ __forceinline__ static float trial(float xi, float va, float vb, float vc, float U,
                                                  float CR, float F, bool forced, float lo,
                                                  float hi) {
        const float v = __fmaf_rn(F, __fsub_rn(vb, vc), va);
        const float y = (U < CR || forced) ? v : xi;
        return clipf(y, lo, hi);
    }
    __device__ __forceinline__ float4 step(int u, int q) {
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

#ifndef EVOX_DE_FIN
#define EVOX_DE_FIN 0
#endif

// One DE generation: trial of every target from the population at parity p,
// evaluation, greedy "<=" replacement by flipping the buffer-select flag.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, G::LPR == 4 ? EVOX_DE_SHORT_MINB : EVOX_MINB) k_de_gen(DeArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P, G> sh_h;
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
#if EVOX_DE_FIN
    // the CTA's minimum key: one relaxed atomicMin, no fence / ticket (k_de_fin publishes
    // after the kernel boundary)
    __shared__ unsigned long long sh_k[WARPS];
    best = warp_min_u64(best);
    if (lane_id() == 0) sh_k[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = sh_k[0];
#pragma unroll
        for (int i = 1; i < WARPS; ++i) k = sh_k[i] < k ? sh_k[i] : k;
        if (k != ~0ull) atomicMin(&a.ctl->gen_key, k);
    }
#else
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key, a.peer != 0)) de_finalize(a, key, t + 1);
#endif
}

#ifndef EVOX_DE_FLAT_MINB
#define EVOX_DE_FLAT_MINB 5  // CTAs/SM of k_de_gen_flat (register cap; 3/4/6: 0.818/0.816/0.857, D1)
#endif
#ifndef EVOX_DE_FLAT_FIN
#define EVOX_DE_FLAT_FIN 1  // CTA minimum by relaxed atomicMin; k_de_fin publishes
#endif
#ifndef EVOX_DE_FLAT_PF
#define EVOX_DE_FLAT_PF 0  // L2 prefetch: bit 0 the (local) donor rows, bit 1 the target rows
                           // (measured: both on 0.643 vs 0.814 of the HBM peak at D1, off)
#endif

// DE generation for short rows (4 / 8 lanes per row geometries, ld <= 256) on a grid of one
// CTA per G::RPC targets, in three phases (the structure of k_pso_gen_flat):
//  0. one thread per target resolves its donors (de_indices), the buffer flags of the four
//     rows, j_rand and f(x), and issues the L2 bulk prefetch of the target and donor rows
//     (400 B each at D1): the scattered-row DRAM stream starts at once, not behind registers;
//  1. flat: the tile's RPC x NQ trial quads, thread i: quads i, i + 256, ... -- each trial quad
//     is exactly MoverDe::step's (same Philox counter (q, global row, t, 10), op order, clip,
//     zero padding), written to the other buffer and staged in shared memory;
//  2. the geometry's row engine folds f(u) from the staged rows in the geometry's order
//     (bitwise k_de_gen's), then the greedy "<=" replacement and the grid argmin.
template <int P, class G, bool UNI>
__global__ void __launch_bounds__(256, EVOX_DE_FLAT_MINB) k_de_gen_flat(DeArgs a) {
    static_assert(G::WPR == 1, "flat phase: warp-row geometries only");
    extern __shared__ __align__(128) unsigned char de_flat_smem[];
    float4* st = reinterpret_cast<float4*>(de_flat_smem);  // staged tile (+ [ld] htab)
    __shared__ Fit<P> sh_acc[1];
    __shared__ float sh_head[1];
    __shared__ const float4* sh_src[G::RPC][4];  // target, donors r1, r2, r3
    __shared__ int sh_jr[G::RPC];
    __shared__ float sh_fx[G::RPC];
    __shared__ unsigned char sh_si[G::RPC];
    __shared__ float4* sh_out[G::RPC];  // the trial row (the other buffer)
    const int NQ = (int)(a.ld >> 2);
    const int tq = G::RPC * NQ;  // staged quads per component
    const float* htab =
        HTable<P, G>::fill(reinterpret_cast<float*>(st + tq * stage_comps<P>()), a.ld);
    const RowMap<G> m(NQ);
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    const int p = (int)(t & 1);
    const long long row0 = (long long)blockIdx.x * G::RPC;
    const int nrow = a.rows - row0 < G::RPC ? (int)(a.rows - row0) : G::RPC;
    // phase 0: per-target resolution + prefetch
    if ((int)threadIdx.x < nrow) {
        const long long rw = row0 + threadIdx.x;
        long long r[3];
        de_indices(a, a.row0 + rw, (uint32_t)t, r);
        const int si = a.sel[p][rw];
        const float4* src[4];
        src[0] = reinterpret_cast<const float4*>(a.buf[si] + rw * a.ld);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int w = de_owner(a, r[k]);
            const long long lr = r[k] - a.prow0[w];
            const int fl = a.psel[w][p][lr];
            src[k + 1] = reinterpret_cast<const float4*>(a.pbuf[w][fl] + lr * a.ld);
#if EVOX_DE_FLAT_PF & 1
            if (w == a.rank) prefetch_l2(src[k + 1], a.ld * 4);
#endif
        }
#if EVOX_DE_FLAT_PF & 2
        prefetch_l2(src[0], a.ld * 4);
#endif
#pragma unroll
        for (int k = 0; k < 4; ++k) sh_src[threadIdx.x][k] = src[k];
        const uint4 jw = Philox::run(make_uint4(0u, (uint32_t)(a.row0 + rw), (uint32_t)t, 9u), a.rk);
        sh_jr[threadIdx.x] = (int)(((unsigned long long)jw.x * (unsigned long long)a.D) >> 32);
        sh_fx[threadIdx.x] = a.f[p][rw];
        sh_si[threadIdx.x] = (unsigned char)si;
        sh_out[threadIdx.x] = reinterpret_cast<float4*>(a.buf[si ^ 1] + rw * a.ld);
    }
    __syncthreads();
    // phase 1: flat walk of the tile's trial quads (r = i / NQ exactly: i < 2^11, NQ <= 64)
    const int n = nrow * NQ;
    const uint32_t magic = (1u << 20) / (uint32_t)NQ + 1u;
    for (int i = threadIdx.x; i < n; i += 256) {
        const int r = (int)(((uint32_t)i * magic) >> 20);
        const int q = i - r * NQ;
        MoverDe<UNI> mv(a);
        mv.Xi = sh_src[r][0];
        mv.Xa = sh_src[r][1];
        mv.Xb = sh_src[r][2];
        mv.Xc = sh_src[r][3];
        mv.Out = sh_out[r];
        mv.jrand = sh_jr[r];
        mv.row_g = (uint32_t)(a.row0 + row0) + (uint32_t)r;
        mv.t = (uint32_t)t;
        mv.template load<G::EFL>(0, q);
        stage_quad<P>(st, tq, i, q, mv.step(0, q), htab);
    }
    __syncthreads();
    // phase 2: f(u) in the geometry's order, greedy replacement, argmin key
    unsigned long long best = ~0ull;
    {
        const long long row = m.first;
        const bool ok = row < a.rows;
        const float fu = fold_staged_row<P, G>(st, tq, ok ? (int)(row - row0) : 0, NQ, a.D, ok,
                                               htab, sh_acc, sh_head);
        if (m.leader && ok) {
            const int lr = (int)(row - row0);
            const float fx = sh_fx[lr];
            const int si = sh_si[lr];
            const bool accept = nan_inf(fu) <= nan_inf(fx);  // S:325, NaN as +inf
            const float fn = accept ? fu : fx;
            a.sel[p ^ 1][row] = (unsigned char)(accept ? (si ^ 1) : si);
            a.f[p ^ 1][row] = fn;
            best = make_key(fn, a.row0 + row);
        }
    }
#if EVOX_DE_FLAT_FIN
    // the CTA's minimum key: one relaxed atomicMin, no fence / ticket (k_de_fin publishes
    // after the kernel boundary)
    __shared__ unsigned long long sh_k[WARPS];
    best = warp_min_u64(best);
    if (lane_id() == 0) sh_k[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = sh_k[0];
#pragma unroll
        for (int i = 1; i < WARPS; ++i) k = sh_k[i] < k ? sh_k[i] : k;
        if (k != ~0ull) atomicMin(&a.ctl->gen_key, k);
    }
#else
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key, a.peer != 0)) de_finalize(a, key, t + 1);
#endif
}

// End of a DE generation launched without the in-kernel grid argmin (EVOX_DE_FIN): the
// generation's minimum, hist, and (peers) the end-of-generation barrier + global minimum.
// The kernel boundary orders every row the generation wrote before the peer publication.
__global__ void __launch_bounds__(32) k_de_fin(DeArgs a) {
    if (a.peer) __threadfence_system();
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    de_finalize(a, *(volatile unsigned long long*)&a.ctl->gen_key, t + 1);
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

// Gather the current population into `dst` WITHOUT touching buf/sel: with peers
// connected, other ranks read this shard's rows through sel[p] in their generation
// kernels, so the state must not change in place.
__global__ void __launch_bounds__(256) k_de_gather(DeArgs a, float* __restrict__ dst) {
    const int p = (int)(a.ctl->t & 1);
    const long long NQ = a.ld >> 2;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    for (long long row = (long long)blockIdx.x * WARPS + wid; row < a.rows;
         row += (long long)gridDim.x * WARPS) {
        const float* src = a.buf[a.sel[p][row] ? 1 : 0];
        const float4* s = reinterpret_cast<const float4*>(src + row * a.ld);
        float4* d = reinterpret_cast<float4*>(dst + row * a.ld);
        for (long long q = lane; q < NQ; q += 32) d[q] = s[q];
    }
}


}  // namespace

cudaError_t launch_de_gather(const DeArgs& a, float* dst, cudaStream_t st) {
    long long g = (a.rows + WARPS - 1) / WARPS;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_de_gather<<<(int)g, 256, 0, st>>>(a, dst);
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

#ifndef EVOX_DE_U
#define EVOX_DE_U 2  // chunks in flight per lane group in the DE generation (short rows)
#endif
#ifndef EVOX_DE_WAVES
#define EVOX_DE_WAVES 16
#endif
// The DE generation's geometry: the row geometry of ld with its own chunk count for short
// rows (never a change of any lane's quad order, so the reduction order is the geometry's).
#define EVOX_DE_GEOM(G_) Geom<G_::LPR, G_::WPR, G_::LPR == 4 ? EVOX_DE_U : G_::NU, G_::EFL>

// Short rows (4 / 8 lanes per row) take the flat-tile kernel unless `no_flat`.
static bool de_flat(long long ld, bool no_flat) { return !no_flat && geom_id(ld) != 1 && geom_id(ld) != 2; }

int de_gen_grid(int problem, long long ld, long long rows, int device, bool no_flat) {
    int g = 1;
    if (de_flat(ld, no_flat)) {
        EVOX_DISPATCH_GEOM(ld, { g = (int)row_units<G_>(rows); });
        return g;
    }
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        using GD_ = EVOX_DE_GEOM(G_);
        g = grid_for((const void*)k_de_gen<P_, GD_, true>, row_units<GD_>(rows), device,
                     EVOX_DE_WAVES);
    }));
    return g;
}

cudaError_t launch_de_gen(int problem, const DeArgs& a, int grid, cudaStream_t st, bool no_flat) {
    if (de_flat(a.ld, no_flat)) {
        EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
            if constexpr (G_::WPR == 1 && G_::LPR <= 8) {
                const size_t smem = flat_stage_bytes<P_>(G_::RPC, a.ld);
                if (smem > 48 * 1024)
                    cudaFuncSetAttribute(k_de_gen_flat<P_, G_, U_>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_de_gen_flat<P_, G_, U_><<<grid, 256, smem, st>>>(a);
            }
        })));
        if (EVOX_DE_FLAT_FIN) k_de_fin<<<1, 32, 0, st>>>(a);
        return cudaGetLastError();
    }
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(a.ld, {
        using GD_ = EVOX_DE_GEOM(G_);
        k_de_gen<P_, GD_, U_><<<grid, 256, 0, st>>>(a);
    })));
    if (EVOX_DE_FIN) k_de_fin<<<1, 32, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_de_materialize(const DeArgs& a, cudaStream_t st) {
    long long g = (a.rows + WARPS - 1) / WARPS;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_de_materialize<<<(int)g, 256, 0, st>>>(a);
    return cudaGetLastError();
}


}  // namespace evox
