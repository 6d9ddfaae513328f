// evox_kernels.cu -- sm_100a kernels of the PSO/CSO generation.
//
// Hot path: one fused kernel per PSO generation reads
// X, V and (unless the row's pbest copy is pending) P once, draws r1/r2 with
// Philox in registers, moves + clips, writes X', V' (and the pending P copy),
// evaluates f(X') from registers, applies the per-row tell and reduces the
// generation's argmin (warp -> CTA -> one atomicMin per CTA); the last CTA to
// finish publishes gbest.  20 B/element of HBM traffic per generation.
//
// Row mapping: WPR warps per row (a function of dim only).  Each warp owns a
// contiguous segment of the row's float4 quads and walks it in chunks of 32
// quads (one LDG.128/STG.128 per lane per array per chunk, 512 B per warp
// instruction), U chunks in flight.
#include <cuda_runtime.h>

#include <cstdint>

#include "evox_device.cuh"
#include "evox_internal.h"

namespace evox {

namespace {

constexpr int U = 4;  // chunks (of 32 quads) in flight per warp

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Row segment of warp `wr` (of WPR) over NQ quads.
__device__ __forceinline__ void row_segment(long long NQ, int wpr, int wr, long long& qb,
                                            long long& qe) {
    const long long seg = (NQ + wpr - 1) / wpr;
    qb = (long long)wr * seg;
    qe = qb + seg < NQ ? qb + seg : NQ;
    if (qb > NQ) qb = NQ;
}

__device__ __forceinline__ float4 bound4(const float* b, float b0, int uniform, long long q) {
    if (uniform) return make_float4(b0, b0, b0, b0);
    return __ldg(reinterpret_cast<const float4*>(b) + q);
}

__device__ __forceinline__ float clipf(float x, float lo, float hi) {
    return fminf(fmaxf(x, lo), hi);
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

// ---------------------------------------------------------------------------
// Row engine: walks one row segment chunk by chunk; `mv` loads/moves a quad
// and returns the value to evaluate; folds the fitness (with the Rosenbrock
// cross-quad halo).  All lanes of the warp execute every chunk iteration.
template <int P, class Mover>
__device__ __forceinline__ void walk_segment(Mover& mv, long long qb, long long qe, long long D,
                                             Fit<P>& acc, float& head_x, float& tail_x,
                                             bool& tail_valid) {
    const int lane = lane_id();
    float pend_x = 0.0f;
    bool pend = false;  // lane 31: x_{4q+3} waiting for x_{4q+4} of the next chunk
    head_x = 0.0f;
    tail_valid = false;
    tail_x = 0.0f;
    for (long long base = qb; base < qe; base += 32 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long q = base + 32 * u + lane;
            if (q < qe) mv.load(u, q);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long cb = base + 32 * u;  // first quad of this chunk
            if (cb >= qe) break;                 // warp-uniform
            const long long q = cb + lane;
            const bool valid = q < qe;
            float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid) xn = mv.step(u, q);
            if (valid) fit_quad<P>(acc, xn, 4 * q, D);
            if constexpr (P == ROSENBROCK) {
                const float nb = __shfl_down_sync(0xffffffffu, xn.x, 1);
                const float f0 = __shfl_sync(0xffffffffu, xn.x, 0);
                if (cb == qb) head_x = f0;
                if (lane == 31 && pend) {
                    acc.pair(pend_x, f0);
                    pend = false;
                }
                if (valid) {
                    const bool has_next = 4 * q + 4 < D;
                    if (q + 1 < qe) {
                        if (lane < 31) {
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

// Reduce a row's fitness over the warp (xor tree) and, for WPR > 1, over the
// row's warps in fixed order through shared memory.  Returns f in lane 0 of
// warp 0 of the row group (other threads: unspecified).
template <int P, int WPR>
__device__ __forceinline__ float reduce_row(Fit<P> acc, long long D, float head_x, float tail_x,
                                            bool tail_valid, Fit<P>* sh_acc, float* sh_head) {
    const int lane = lane_id();
    if constexpr (WPR > 1 && P == ROSENBROCK) {
        const int wr = threadIdx.x >> 5;
        if (lane == 0) sh_head[wr] = head_x;
        __syncthreads();
        if (tail_valid && wr + 1 < WPR) acc.pair(tail_x, sh_head[wr + 1]);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        Fit<P> o = acc;
        o.shfl_xor(m);
        acc.combine(o);
    }
    if constexpr (WPR == 1) return acc.finish(D);
    const int wr = threadIdx.x >> 5;
    if (lane == 0) sh_acc[wr] = acc;
    __syncthreads();
    float f = 0.0f;
    if (threadIdx.x == 0) {
        Fit<P> t = sh_acc[0];
#pragma unroll 1
        for (int k = 1; k < WPR; ++k) t.combine(sh_acc[k]);
        f = t.finish(D);
    }
    __syncthreads();  // sh_acc / sh_head reusable for the next row
    return f;
}

// ---------------------------------------------------------------------------
// Movers
struct MoverEval {
    const float4* Xr;
    float4 x[U];
    __device__ __forceinline__ void load(int u, long long q) { x[u] = ld_stream(Xr + q); }
    __device__ __forceinline__ float4 step(int u, long long) { return x[u]; }
};

// PSO move of one row (A1, A3, A4, lazy A5).  Holds a reference to the kernel
// parameter block (resolved to constant-bank operands once inlined: the
// Philox round keys, w, phi*2^-24 and the bounds feed instructions directly).
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
    __device__ __forceinline__ void load(int u, long long q) {
        x[u] = ld_stream(Xr + q);
        v[u] = ld_stream(Vr + q);
        if (!pend) p[u] = ld_stream(Pr + q);
    }
    __device__ __forceinline__ float4 step(int u, long long q) {
        const float4 xo = x[u];
        const float4 pb = pend ? xo : p[u];
        if (pend) st_stream(Pr + q, xo);
        const float4 g = __ldg(reinterpret_cast<const float4*>(a.G) + q);
        float4 lo, hi;
        if (a.uniform_bounds) {
            lo = make_float4(a.lb0, a.lb0, a.lb0, a.lb0);
            hi = make_float4(a.ub0, a.ub0, a.ub0, a.ub0);
        } else {
            lo = __ldg(reinterpret_cast<const float4*>(a.lb) + q);
            hi = __ldg(reinterpret_cast<const float4*>(a.ub) + q);
        }
        const uint4 b1 = Philox::run(make_uint4((uint32_t)q, row_g, t, 2u), a.rk);
        const uint4 b2 = Philox::run(make_uint4((uint32_t)q, row_g, t, 3u), a.rk);
        float4 xn = xo, vn = v[u];
        const float w = a.w, cp = a.cp, cg = a.cg;
        pso_elem(xn.x, vn.x, pb.x, g.x, scaled_u24(b1.x, cp), scaled_u24(b2.x, cg), w, lo.x, hi.x);
        pso_elem(xn.y, vn.y, pb.y, g.y, scaled_u24(b1.y, cp), scaled_u24(b2.y, cg), w, lo.y, hi.y);
        pso_elem(xn.z, vn.z, pb.z, g.z, scaled_u24(b1.z, cp), scaled_u24(b2.z, cg), w, lo.z, hi.z);
        pso_elem(xn.w, vn.w, pb.w, g.w, scaled_u24(b1.w, cp), scaled_u24(b2.w, cg), w, lo.w, hi.w);
        if (4 * q + 3 >= a.D) {  // padding columns stay 0
            const long long j0 = 4 * q;
            if (j0 + 1 >= a.D) { xn.y = 0.f; vn.y = 0.f; }
            if (j0 + 2 >= a.D) { xn.z = 0.f; vn.z = 0.f; }
            if (j0 + 3 >= a.D) { xn.w = 0.f; vn.w = 0.f; }
        }
        st_stream(Xr + q, xn);
        st_stream(Vr + q, vn);
        return xn;
    }
};

// Bulk L2 prefetch (Hopper+ cp.async.bulk.prefetch): pulls a whole row segment
// from HBM into L2 with one instruction, so the next row's LDGs hit L2.
__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
    if (bytes > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)bytes)
                     : "memory");
}

// ---------------------------------------------------------------------------
// Grid-level argmin + finalize (A12/A13).  Every thread calls it after its
// last row; `my_key` is meaningful in any thread (~0 = none).
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long k) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, m);
        k = o < k ? o : k;
    }
    return k;
}

// Returns true in the (whole) last CTA to finish; key in *out_key.
__device__ __forceinline__ bool grid_argmin(Ctl* ctl, unsigned long long my_key,
                                            unsigned long long* out_key) {
    __shared__ unsigned long long sh_k[32];
    __shared__ int sh_last;
    const int lane = lane_id(), wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    my_key = warp_min_u64(my_key);
    if (lane == 0) sh_k[wid] = my_key;
    __threadfence();  // this thread's population stores visible device-wide
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

// In the last CTA: gbest update (strict, R-5), hist, record for world > 1.
// `t_new` is the index of the population just evaluated.
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

// ---------------------------------------------------------------------------
// Kernels

// A2: X0 = fmaf(u, ub-lb, lb) (Philox tag 0, t = 0), V0 = 0, P0 = X0.
__global__ void k_pso_init(PsoArgs a) {
    const long long NQ = a.ld >> 2;
    const long long total = a.rows * NQ;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / NQ, q = i - r * NQ;
        const uint4 b = Philox::run(make_uint4((uint32_t)q, (uint32_t)(a.row0 + r), 0u, 0u), a.k0,
                                    a.k1);
        const float4 lo = bound4(a.lb, a.lb0, a.uniform_bounds, q);
        const float4 hi = bound4(a.ub, a.ub0, a.uniform_bounds, q);
        float4 x;
        x.x = __fmaf_rn(u24(b.x), __fsub_rn(hi.x, lo.x), lo.x);
        x.y = __fmaf_rn(u24(b.y), __fsub_rn(hi.y, lo.y), lo.y);
        x.z = __fmaf_rn(u24(b.z), __fsub_rn(hi.z, lo.z), lo.z);
        x.w = __fmaf_rn(u24(b.w), __fsub_rn(hi.w, lo.w), lo.w);
        const long long j0 = 4 * q;
        if (j0 + 1 >= a.D) x.y = 0.f;
        if (j0 + 2 >= a.D) x.z = 0.f;
        if (j0 + 3 >= a.D) x.w = 0.f;
        reinterpret_cast<float4*>(a.X)[i] = x;
        reinterpret_cast<float4*>(a.P)[i] = x;
        reinterpret_cast<float4*>(a.V)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        a.pf[r] = __int_as_float(0x7f800000);
        a.f[r] = __int_as_float(0x7f800000);
        a.imp[r] = 0;
    }
}

// evox_eval: fit[r] = f(X[r]).
template <int P, int WPR>
__global__ void __launch_bounds__(WPR == 1 ? 256 : WPR * 32) k_eval(const float* __restrict__ X, long long rows,
                                              long long D, long long ld, float* __restrict__ fit) {
    __shared__ Fit<P> sh_acc[WPR > 1 ? WPR : 1];
    __shared__ float sh_head[WPR > 1 ? WPR : 1];
    constexpr int RPC = (WPR == 1) ? 8 : 1;  // rows per CTA pass
    const int wid = threadIdx.x >> 5;
    const int wr = (WPR == 1) ? 0 : wid;
    const int slot = (WPR == 1) ? wid : 0;
    long long qb, qe;
    row_segment(ld >> 2, WPR, wr, qb, qe);
    for (long long row = (long long)blockIdx.x * RPC + slot; row < rows;
         row += (long long)gridDim.x * RPC) {
        MoverEval mv;
        mv.Xr = reinterpret_cast<const float4*>(X + row * ld);
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P>(mv, qb, qe, D, acc, hx, tx, tv);
        const float f = reduce_row<P, WPR>(acc, D, hx, tx, tv, sh_acc, sh_head);
        if ((WPR == 1) ? (threadIdx.x & 31) == 0 : threadIdx.x == 0) fit[row] = f;
    }
}

// Fused PSO generation: lazy pbest + move + clip + evaluate + tell + argmin.
template <int P, int WPR>
__global__ void __launch_bounds__(WPR == 1 ? 256 : WPR * 32) k_pso_gen(PsoArgs a) {
    __shared__ Fit<P> sh_acc[WPR > 1 ? WPR : 1];
    __shared__ float sh_head[WPR > 1 ? WPR : 1];
    constexpr int RPC = (WPR == 1) ? 8 : 1;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    const int wr = (WPR == 1) ? 0 : wid;
    const int slot = (WPR == 1) ? wid : 0;
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    long long qb, qe;
    row_segment(a.ld >> 2, WPR, wr, qb, qe);
    unsigned long long best = ~0ull;
    const long long stride = (long long)gridDim.x * RPC;
    const long long seg_off = qb * 16, seg_bytes = (qe - qb) * 16;
    long long row = (long long)blockIdx.x * RPC + slot;
    // pbest-pending flags one and two rows ahead (imp[r] is rewritten only by
    // the warp(s) that own row r, later in this kernel, so these reads see the
    // previous generation's decisions).
    bool pend_cur = row < a.rows ? a.imp[row] != 0 : false;
    bool pend_nxt = row + stride < a.rows ? a.imp[row + stride] != 0 : true;
    for (; row < a.rows; row += stride) {
        const long long nxt = row + stride, nn = nxt + stride;
        if (lane == 0 && nxt < a.rows) {  // next row of this warp: HBM -> L2 now
            const long long o = nxt * a.ld * 4 + seg_off;
            prefetch_l2(reinterpret_cast<const char*>(a.X) + o, seg_bytes);
            prefetch_l2(reinterpret_cast<const char*>(a.V) + o, seg_bytes);
            if (!pend_nxt) prefetch_l2(reinterpret_cast<const char*>(a.P) + o, seg_bytes);
        }
        const bool pend_nn = nn < a.rows ? a.imp[nn] != 0 : true;
        float pf_old = 0.0f;
        if (lane == 0) pf_old = a.pf[row];
        MoverPso mv(a, row, (uint32_t)t, pend_cur);
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P>(mv, qb, qe, a.D, acc, hx, tx, tv);
        const float f = reduce_row<P, WPR>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
        if (lane == 0 && (WPR == 1 || wid == 0)) {
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
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key)) pso_finalize(a, key, t + 1);
}

// Unfused ask: move X_t -> X_{t+1} (no evaluation).
template <int WPR>
__global__ void __launch_bounds__(WPR == 1 ? 256 : WPR * 32) k_pso_move(PsoArgs a,
                                                                        unsigned long long t) {
    constexpr int RPC = (WPR == 1) ? 8 : 1;
    const int wid = threadIdx.x >> 5;
    const int wr = (WPR == 1) ? 0 : wid;
    const int slot = (WPR == 1) ? wid : 0;
    long long qb, qe;
    row_segment(a.ld >> 2, WPR, wr, qb, qe);
    for (long long row = (long long)blockIdx.x * RPC + slot; row < a.rows;
         row += (long long)gridDim.x * RPC) {
        MoverPso mv(a, row, (uint32_t)t, a.imp[row] != 0);
        Fit<SPHERE> acc;  // unused
        float hx, tx;
        bool tv;
        walk_segment<SPHERE>(mv, qb, qe, a.D, acc, hx, tx, tv);
        __syncwarp();
        if (WPR > 1) __syncthreads();
        if (lane_id() == 0 && (WPR == 1 || wid == 0)) a.imp[row] = 0;
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
    for (long long row = (long long)blockIdx.x * 8 + wid; row < a.rows;
         row += (long long)gridDim.x * 8) {
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
    __device__ __forceinline__ void init(uint32_t blk, uint32_t t, uint32_t Bb_, uint32_t k0,
                                         uint32_t k1) {
        const uint4 rk = Philox::run(make_uint4(blk, 0u, t, 4u), k0, k1);
        k[0] = rk.x; k[1] = rk.y; k[2] = rk.z; k[3] = rk.w;
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
struct MoverCso {
    float4* Xl;
    float4* Vl;
    const float4* Xw;
    const float4* lb;
    const float4* ub;
    const float4* xbar;
    float lb0, ub0, phi;
    const PhiloxKey* rk;
    uint32_t row_g, t;
    bool uni;
    long long D;
    float4 x[U], v[U], xw[U];
    __device__ __forceinline__ void load(int u, long long q) {
        x[u] = ld_stream(Xl + q);
        v[u] = ld_stream(Vl + q);
        xw[u] = ld_stream(Xw + q);
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
        const uint4 b1 = Philox::run(make_uint4((uint32_t)q, row_g, t, 5u), *rk);
        const uint4 b2 = Philox::run(make_uint4((uint32_t)q, row_g, t, 6u), *rk);
        const bool use3 = phi != 0.0f;
        float4 c3 = make_float4(0.f, 0.f, 0.f, 0.f), xb = c3;
        if (use3) {
            const uint4 b3 = Philox::run(make_uint4((uint32_t)q, row_g, t, 7u), *rk);
            c3 = make_float4(__fmul_rn(phi, u24(b3.x)), __fmul_rn(phi, u24(b3.y)),
                             __fmul_rn(phi, u24(b3.z)), __fmul_rn(phi, u24(b3.w)));
            xb = __ldg(xbar + q);
        }
        const float4 lo = uni ? make_float4(lb0, lb0, lb0, lb0) : __ldg(lb + q);
        const float4 hi = uni ? make_float4(ub0, ub0, ub0, ub0) : __ldg(ub + q);
        float4 xn, vn;
        xn.x = upd(x[u].x, v[u].x, xw[u].x, u24(b1.x), u24(b2.x), c3.x, xb.x, use3, lo.x, hi.x, vn.x);
        xn.y = upd(x[u].y, v[u].y, xw[u].y, u24(b1.y), u24(b2.y), c3.y, xb.y, use3, lo.y, hi.y, vn.y);
        xn.z = upd(x[u].z, v[u].z, xw[u].z, u24(b1.z), u24(b2.z), c3.z, xb.z, use3, lo.z, hi.z, vn.z);
        xn.w = upd(x[u].w, v[u].w, xw[u].w, u24(b1.w), u24(b2.w), c3.w, xb.w, use3, lo.w, hi.w, vn.w);
        if (4 * q + 3 >= D) {
            const long long j0 = 4 * q;
            if (j0 + 1 >= D) { xn.y = 0.f; vn.y = 0.f; }
            if (j0 + 2 >= D) { xn.z = 0.f; vn.z = 0.f; }
            if (j0 + 3 >= D) { xn.w = 0.f; vn.w = 0.f; }
        }
        st_stream(Xl + q, xn);
        st_stream(Vl + q, vn);
        return xn;
    }
};

__device__ void cso_finalize(const CsoArgs& a, unsigned long long key, unsigned long long t_new) {
    if (threadIdx.x == 0) {
        Ctl* ctl = a.ctl;
        if (a.exchange) {
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

// One CSO generation over this shard's whole blocks.  One work item per pair
// (plus one for the unpaired member of an odd block); WPR warps per item.
template <int P, int WPR>
__global__ void __launch_bounds__(WPR == 1 ? 256 : WPR * 32) k_cso_gen(CsoArgs a) {
    __shared__ Fit<P> sh_acc[WPR > 1 ? WPR : 1];
    __shared__ float sh_head[WPR > 1 ? WPR : 1];
    constexpr int RPC = (WPR == 1) ? 8 : 1;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    const int wr = (WPR == 1) ? 0 : wid;
    const int slot = (WPR == 1) ? wid : 0;
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    long long qb, qe;
    row_segment(a.ld >> 2, WPR, wr, qb, qe);
    const long long blk0 = a.row0 / a.B;
    const long long nblk = (a.row0 + a.rows + a.B - 1) / a.B - blk0;
    const long long ipb = (a.B + 1) / 2;
    const long long items = nblk * ipb;
    unsigned long long best = ~0ull;
    for (long long it = (long long)blockIdx.x * RPC + slot; it < items;
         it += (long long)gridDim.x * RPC) {
        const long long bl = it / ipb, p = it - bl * ipb;
        const long long blk = blk0 + bl;
        const long long base = blk * a.B;
        const long long Bb = (base + a.B <= a.pop) ? a.B : a.pop - base;
        if (p >= (Bb + 1) / 2) continue;  // uniform across the item's warps
        CsoPerm perm;
        perm.init((uint32_t)blk, (uint32_t)t, (uint32_t)Bb, a.k0, a.k1);
        if (2 * p + 1 >= Bb) {  // odd block: unpaired member passes unchanged
            const long long gi = base + perm((uint32_t)(Bb - 1));
            if (lane == 0 && (WPR == 1 || wid == 0)) {
                const unsigned long long k = make_key(a.f[gi - a.row0], gi);
                best = k < best ? k : best;
            }
            continue;
        }
        const long long gi = base + perm((uint32_t)(2 * p));
        const long long gk = base + perm((uint32_t)(2 * p + 1));
        float fi = a.f[gi - a.row0], fk = a.f[gk - a.row0];
        const float oi = fi != fi ? __int_as_float(0x7f800000) : fi;
        const float ok = fk != fk ? __int_as_float(0x7f800000) : fk;
        const bool i_wins = oi < ok || (oi == ok && gi < gk);
        const long long gw = i_wins ? gi : gk, gl = i_wins ? gk : gi;
        const float fw = i_wins ? fi : fk;
        MoverCso mv;
        mv.Xl = reinterpret_cast<float4*>(a.X + (gl - a.row0) * a.ld);
        mv.Vl = reinterpret_cast<float4*>(a.V + (gl - a.row0) * a.ld);
        mv.Xw = reinterpret_cast<const float4*>(a.X + (gw - a.row0) * a.ld);
        mv.lb = reinterpret_cast<const float4*>(a.lb);
        mv.ub = reinterpret_cast<const float4*>(a.ub);
        mv.xbar = reinterpret_cast<const float4*>(a.xbar);
        mv.lb0 = a.lb0; mv.ub0 = a.ub0; mv.phi = a.phi;
        mv.rk = &a.rk;
        mv.row_g = (uint32_t)gl;
        mv.t = (uint32_t)t;
        mv.uni = a.uniform_bounds != 0;
        mv.D = a.D;
        Fit<P> acc;
        float hx, tx;
        bool tv;
        walk_segment<P>(mv, qb, qe, a.D, acc, hx, tx, tv);
        const float fl = reduce_row<P, WPR>(acc, a.D, hx, tx, tv, sh_acc, sh_head);
        if (lane == 0 && (WPR == 1 || wid == 0)) {
            a.f[gl - a.row0] = fl;
            const unsigned long long kw = make_key(fw, gw), kl = make_key(fl, gl);
            const unsigned long long k = kw < kl ? kw : kl;
            best = k < best ? k : best;
        }
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key)) cso_finalize(a, key, t + 1);
}

// Generation 0 (after the evaluation of X0): population minimum -> hist[0].
__global__ void __launch_bounds__(256) k_cso_tell0(CsoArgs a) {
    unsigned long long best = ~0ull;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
         r += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = make_key(a.f[r], a.row0 + r);
        best = k < best ? k : best;
    }
    unsigned long long key;
    if (grid_argmin(a.ctl, best, &key)) cso_finalize(a, key, 0);
}

// CSO init: X0 = fmaf(u, ub-lb, lb) (tag 0, t = 0), V0 = 0 -- same stream as PSO init.
__global__ void k_cso_init(CsoArgs a) {
    const long long NQ = a.ld >> 2;
    const long long total = a.rows * NQ;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / NQ, q = i - r * NQ;
        const uint4 b = Philox::run(make_uint4((uint32_t)q, (uint32_t)(a.row0 + r), 0u, 0u), a.k0,
                                    a.k1);
        const float4 lo = bound4(a.lb, a.lb0, a.uniform_bounds, q);
        const float4 hi = bound4(a.ub, a.ub0, a.uniform_bounds, q);
        float4 x;
        x.x = __fmaf_rn(u24(b.x), __fsub_rn(hi.x, lo.x), lo.x);
        x.y = __fmaf_rn(u24(b.y), __fsub_rn(hi.y, lo.y), lo.y);
        x.z = __fmaf_rn(u24(b.z), __fsub_rn(hi.z, lo.z), lo.z);
        x.w = __fmaf_rn(u24(b.w), __fsub_rn(hi.w, lo.w), lo.w);
        const long long j0 = 4 * q;
        if (j0 + 1 >= a.D) x.y = 0.f;
        if (j0 + 2 >= a.D) x.z = 0.f;
        if (j0 + 3 >= a.D) x.w = 0.f;
        reinterpret_cast<float4*>(a.X)[i] = x;
        reinterpret_cast<float4*>(a.V)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
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

__global__ void k_debug_philox(const uint4* ctr, uint32_t k0, uint32_t k1, uint4* out,
                               long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = Philox::run(ctr[i], k0, k1);
}

// ----------------------------------------------------------------- dispatch
int sm_count(int device) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

}  // namespace

int wpr_for_dim(long long ld) {
    const long long NQ = ld >> 2;
    if (NQ <= 1024) return 1;
    if (NQ <= 8192) return 8;
    return 32;
}

#define EVOX_DISPATCH_WPR(wpr, ...)          \
    do {                                      \
        if ((wpr) == 1) {                     \
            constexpr int W_ = 1;             \
            __VA_ARGS__;                             \
        } else if ((wpr) == 8) {              \
            constexpr int W_ = 8;             \
            __VA_ARGS__;                             \
        } else {                              \
            constexpr int W_ = 32;            \
            __VA_ARGS__;                             \
        }                                     \
    } while (0)

#define EVOX_DISPATCH_PROB(p, ...)            \
    do {                                       \
        switch (p) {                           \
            case SPHERE: {                     \
                constexpr int P_ = SPHERE;     \
                __VA_ARGS__;                          \
            } break;                           \
            case ACKLEY: {                     \
                constexpr int P_ = ACKLEY;     \
                __VA_ARGS__;                          \
            } break;                           \
            case RASTRIGIN: {                  \
                constexpr int P_ = RASTRIGIN;  \
                __VA_ARGS__;                          \
            } break;                           \
            case GRIEWANK: {                   \
                constexpr int P_ = GRIEWANK;   \
                __VA_ARGS__;                          \
            } break;                           \
            default: {                         \
                constexpr int P_ = ROSENBROCK; \
                __VA_ARGS__;                          \
            } break;                           \
        }                                      \
    } while (0)

static int grid_for(const void* fn, int threads, long long units, int device) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)sm_count(device) * per_sm;
    if (units < g) g = units;
    return (int)(g < 1 ? 1 : g);
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
    const int wpr = wpr_for_dim(ld);
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_WPR(wpr, {
        const int threads = W_ == 1 ? 256 : W_ * 32;
        const long long units = W_ == 1 ? (rows + 7) / 8 : rows;
        const int g = grid_for((const void*)k_eval<P_, W_>, threads, units, dev);
        k_eval<P_, W_><<<g, threads, 0, st>>>(X, rows, D, ld, fit);
    }));
    return cudaGetLastError();
}

int pso_gen_grid(int problem, long long ld, long long rows, int device) {
    const int wpr = wpr_for_dim(ld);
    int g = 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_WPR(wpr, {
        const int threads = W_ == 1 ? 256 : W_ * 32;
        const long long units = W_ == 1 ? (rows + 7) / 8 : rows;
        g = grid_for((const void*)k_pso_gen<P_, W_>, threads, units, device);
    }));
    return g;
}

cudaError_t launch_pso_gen(int problem, const PsoArgs& a, int grid, cudaStream_t st) {
    const int wpr = wpr_for_dim(a.ld);
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_WPR(wpr, {
        const int threads = W_ == 1 ? 256 : W_ * 32;
        k_pso_gen<P_, W_><<<grid, threads, 0, st>>>(a);
    }));
    return cudaGetLastError();
}

cudaError_t launch_pso_move(const PsoArgs& a, unsigned long long t, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int wpr = wpr_for_dim(a.ld);
    EVOX_DISPATCH_WPR(wpr, {
        const int threads = W_ == 1 ? 256 : W_ * 32;
        const long long units = W_ == 1 ? (a.rows + 7) / 8 : a.rows;
        const int g = grid_for((const void*)k_pso_move<W_>, threads, units, dev);
        k_pso_move<W_><<<g, threads, 0, st>>>(a, t);
    });
    return cudaGetLastError();
}

cudaError_t launch_pso_tell(const PsoArgs& a, const float* fit, unsigned long long t,
                            cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int g = grid_for((const void*)k_pso_tell, 256, (a.rows + 255) / 256, dev);
    k_pso_tell<<<g, 256, 0, st>>>(a, fit, t);
    return cudaGetLastError();
}

cudaError_t launch_gbest_select(const PsoArgs& a, cudaStream_t st) {
    k_gbest_select<<<1, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pso_materialize(const PsoArgs& a, cudaStream_t st) {
    long long g = (a.rows + 7) / 8;
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
    const int g = grid_for((const void*)k_cso_tell0, 256, (a.rows + 255) / 256, dev);
    k_cso_tell0<<<g, 256, 0, st>>>(a);
    return cudaGetLastError();
}

static long long cso_items(const CsoArgs& a) {
    const long long blk0 = a.row0 / a.B;
    const long long nblk = (a.row0 + a.rows + a.B - 1) / a.B - blk0;
    return nblk * ((a.B + 1) / 2);
}

int cso_gen_grid(int problem, const CsoArgs& a, int device) {
    const int wpr = wpr_for_dim(a.ld);
    const long long items = cso_items(a);
    int g = 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_WPR(wpr, {
        const int threads = W_ == 1 ? 256 : W_ * 32;
        const long long units = W_ == 1 ? (items + 7) / 8 : items;
        g = grid_for((const void*)k_cso_gen<P_, W_>, threads, units, device);
    }));
    return g;
}

cudaError_t launch_cso_gen(int problem, const CsoArgs& a, int grid, cudaStream_t st) {
    const int wpr = wpr_for_dim(a.ld);
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_WPR(wpr, {
        const int threads = W_ == 1 ? 256 : W_ * 32;
        k_cso_gen<P_, W_><<<grid, threads, 0, st>>>(a);
    }));
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

cudaError_t launch_debug_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                                long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long g = (n + 255) / 256;
    if (g > 4096) g = 4096;
    k_debug_philox<<<(int)g, 256, 0, st>>>(reinterpret_cast<const uint4*>(ctr), k0, k1,
                                           reinterpret_cast<uint4*>(out), n);
    return cudaGetLastError();
}

}  // namespace evox
