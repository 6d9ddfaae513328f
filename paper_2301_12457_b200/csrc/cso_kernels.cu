// cso_kernels.cu -- CSO (Table II; R-8): keyed block pairing, loser update,
// global pairing across shards.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "evox_device.cuh"
#include "evox_internal.h"
#include "row_engine.cuh"

#ifndef EVOX_CSO_U
#define EVOX_CSO_U U        // chunks in flight per lane group (warp-row geometries)
#endif
#ifndef EVOX_CSO_MINB
#define EVOX_CSO_MINB EVOX_MINB
#endif
#ifndef EVOX_CSO_WAVES
#define EVOX_CSO_WAVES 1
#endif

namespace evox {

namespace {

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
    __device__ __forceinline__ void load(int u, int q) {
        x[u] = ld_stream<EF>(Xl + q);
        v[u] = ld_stream<EF>(Vl + q);
        xw[u] = ld_stream<EF>(Xw + q);
    }
    template <bool EF>
    __device__ __forceinline__ void load_late(int, int) {}
    __device__ __forceinline__ static float upd(float xl, float vl, float xwv, float r1, float r2,
                                                float c3, float xb, bool use3, float lo, float hi,
                                                float& vout) {
        float v = __fmaf_rn(r2, __fsub_rn(xwv, xl), __fmul_rn(r1, vl));
        if (use3) v = __fmaf_rn(c3, __fsub_rn(xb, xl), v);
        vout = v;
        return clipf(__fadd_rn(xl, v), lo, hi);
    }
    __device__ __forceinline__ float4 step(int u, int q) {
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
__global__ void __launch_bounds__(256, EVOX_CSO_MINB) k_cso_gen(CsoArgs a) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P, G> sh_h;
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

// Column means for the phi != 0 term (R-15).  x is quantised to the fixed-point
// grid 2^-qs (qs = 54 - ceil(log2 max|bound|), so |q| <= 2^54) and summed as exact
// integers: int64 per 256-row chunk (|sum| < 2^62), folded into two carry-free
// 64-bit limbs (the chunk sum's low 32 bits, unsigned, and its high part,
// signed).  Integer addition is associative, so every partition of the rows --
// CTAs, shards, NCCL or peer reduction order -- gives the same limbs and hence a
// bitwise identical x-bar for every world size.
constexpr long long COL_CH = 256;
__global__ void k_colsum(const float* __restrict__ X, long long rows, long long ld, double scale,
                         unsigned long long* __restrict__ limb) {
    const long long NQ = ld >> 2;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= NQ) return;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    const long long nch = (rows + COL_CH - 1) / COL_CH;
    for (long long c = blockIdx.y; c < nch; c += gridDim.y) {
        const long long r0 = c * COL_CH, r1 = r0 + COL_CH < rows ? r0 + COL_CH : rows;
        long long cs[4] = {0, 0, 0, 0};
#pragma unroll 4
        for (long long r = r0; r < r1; ++r) {
            const float4 x = __ldcs(X4 + r * NQ + q);
            cs[0] += __double2ll_rn((double)x.x * scale);
            cs[1] += __double2ll_rn((double)x.y * scale);
            cs[2] += __double2ll_rn((double)x.z * scale);
            cs[3] += __double2ll_rn((double)x.w * scale);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            atomicAdd(&limb[4 * q + k], (unsigned long long)cs[k] & 0xffffffffull);
            atomicAdd(&limb[ld + 4 * q + k], (unsigned long long)(cs[k] >> 32));
        }
    }
}

// x-bar[j] = (sum_w limbs_w[j]) 2^-qs / pop.  With peers (evox_cso_connect) every
// CTA first publishes "my limbs are final for generation t" into every rank's
// flag slot and waits for all W flags (st.release.sys / ld.acquire.sys); the
// limbs are single-buffered because no rank zeroes them for t+1 before the
// end-of-generation barrier of t.  Without peers the limbs are already global
// (W = 1, or NCCL-summed).
__global__ void k_colmean(CsoArgs a, double inv_scale) {
    const unsigned long long t = *(volatile unsigned long long*)&a.ctl->t;
    if (a.peer) {
        __shared__ int ok;
        if (threadIdx.x == 0) {
            const unsigned long long flag = t + 1;
            __threadfence_system();
            for (int w = 0; w < a.world; ++w) st_release_sys(a.pcflag[w] + a.rank, flag);
            const unsigned long long t0 = globaltimer_ns();
            ok = 1;
            for (int w = 0; w < a.world && ok; ++w) {
                while (ld_acquire_sys(a.pcflag[a.rank] + w) < flag) {
                    if (globaltimer_ns() - t0 > a.peer_timeout_ns) {
                        a.ctl->err = 1;
                        ok = 0;
                        break;
                    }
                    __nanosleep(128);
                }
            }
        }
        __syncthreads();
        if (!ok) return;
    }
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.ld) return;
    unsigned long long lo = 0, hi = 0;
    const int n = a.peer ? a.world : 1;
    for (int w = 0; w < n; ++w) {
        const unsigned long long* l = a.peer ? a.plimb[w] : a.limb;
        lo += __ldcg(l + j);
        hi += __ldcg(l + a.ld + j);
    }
    const long long h = (long long)hi + (long long)(lo >> 32);  // S = h 2^32 + (lo mod 2^32)
    const double S = __fma_rn((double)h, 4294967296.0, (double)(lo & 0xffffffffull));
    a.xbar[j] = (float)(S * inv_scale / (double)a.pop);
}

// world > 1: hist[t] from the all-reduced (min) keys.
__global__ void k_keys_to_hist(Ctl* ctl, unsigned long long t0, long long n) {
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long k = ctl->hkeys[t0 + i];
        ctl->hist[t0 + i] =
            k != ~0ull ? unord_f32((uint32_t)(k >> 32)) : __int_as_float(0x7f800000);
    }
}


}  // namespace

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

// The CSO generation's geometry: the row geometry of ld with its own chunk count (never a
// change of any lane's quad order, so the reduction order is the geometry's).
#define EVOX_CSO_GEOM(G_) Geom<G_::LPR, G_::WPR, G_::WPR == 1 ? EVOX_CSO_U : G_::NU, G_::EFL>

int cso_gen_grid(int problem, const CsoArgs& a, int device) {
    int g = 1;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM_ID(cso_geom_id(a.ld), {
        using GC_ = EVOX_CSO_GEOM(G_);
        g = grid_for((const void*)k_cso_gen<P_, GC_, true>, row_units<GC_>(cso_items(a)), device,
                     EVOX_CSO_WAVES);
    }));
    return g;
}

cudaError_t launch_cso_gen(int problem, const CsoArgs& a, int grid, cudaStream_t st) {
    EVOX_DISPATCH_UNI(a.uniform_bounds, EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM_ID(cso_geom_id(a.ld), {
        using GC_ = EVOX_CSO_GEOM(G_);
        k_cso_gen<P_, GC_, U_><<<grid, 256, 0, st>>>(a);
    })));
    return cudaGetLastError();
}

cudaError_t launch_cso_colsum(const CsoArgs& a, double scale, cudaStream_t st) {
    const long long NQ = a.ld >> 2, nch = (a.rows + COL_CH - 1) / COL_CH;
    dim3 g((unsigned)((NQ + 127) / 128), (unsigned)(nch < 65535 ? nch : 65535));
    k_colsum<<<g, 128, 0, st>>>(a.X, a.rows, a.ld, scale, a.limb);
    return cudaGetLastError();
}

cudaError_t launch_cso_colmean(const CsoArgs& a, double inv_scale, cudaStream_t st) {
    k_colmean<<<(unsigned)((a.ld + 255) / 256), 256, 0, st>>>(a, inv_scale);
    return cudaGetLastError();
}

cudaError_t launch_cso_hist_from_keys(const CsoArgs& a, unsigned long long t0, long long n,
                                      cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_keys_to_hist<<<1, 256, 0, st>>>(a.ctl, t0, n);
    return cudaGetLastError();
}


}  // namespace evox
