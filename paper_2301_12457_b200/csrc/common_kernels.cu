// common_kernels.cu -- Problem.evaluate (evox_eval), the argmin query kernel and the
// Philox test hook.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "evox_device.cuh"
#include "evox_internal.h"
#include "row_engine.cuh"

namespace evox {

namespace {

#ifndef EVOX_EVAL_WAVES
// waves of resident CTAs by geometry (0: one CTA per row unit).  Measured same box
// (profiles/r02_ab_eval.txt): warp-per-row 4 waves (EH-ackley 0.916 -> 0.967, rastrigin
// 0.906 -> 0.959, rosenbrock 0.896 -> 0.950, griewank 0.792 -> 0.857 of the HBM peak);
// CTA-per-row one CTA per row (E5-griewank 0.782 -> 0.843); short rows unchanged (1).
#define EVOX_EVAL_WAVES(G_) (G_::WPR > 1 ? 0 : (G_::LPR == 32 ? 4 : 1))
#endif
#ifndef EVOX_EVAL_MINB
#define EVOX_EVAL_MINB 1
#endif
#ifndef EVOX_EVAL_U
#define EVOX_EVAL_U U      // chunks in flight (warp-row geometries)
#endif
#define EVOX_EVAL_GEOM(G_) Geom<G_::LPR, G_::WPR, G_::WPR == 1 ? EVOX_EVAL_U : G_::NU, G_::EFL>

// evox_eval: fit[r] = f(X[r]).
template <int P, class G>
__global__ void __launch_bounds__(256, EVOX_EVAL_MINB) k_eval(const float* __restrict__ X, long long rows,
                                              long long D, long long ld,
                                              float* __restrict__ fit,
                                              const float* __restrict__ hg) {
    __shared__ Fit<P> sh_acc[G::WPR];
    __shared__ float sh_head[G::WPR];
    __shared__ __align__(16) HStore<P, G> sh_h;
    const float* htab;
    if constexpr (P == GRIEWANK && G::WPR > 1) htab = hg;  // global table or nullptr
    else htab = HTable<P, G>::fill(sh_h.v, ld);
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

// Griewank column constants for the CTA-per-row geometry (ld > HTAB): h[j] is
// griewank_h(j) itself, so a kernel reading the table and one computing h_j per
// element (the fused generations, or evox_eval under stream capture) produce the
// same bits.  Saves the conversion + MUFU.RSQ + Newton step (~7 instructions of
// ~30) per element for one L2-resident LDG.128 per quad.
__global__ void k_griewank_table(float* __restrict__ h, long long n) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (long long)gridDim.x * blockDim.x)
        h[j] = griewank_h(j);
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

// best() of one rank's CSO / DE population: the row of the current generation's minimum key
// (ctl->min_key, written by the generation kernel's finalize), from the buffer its selection
// flag names (DE: sel[t & 1]; CSO: one buffer), into out [ld].  Nothing if there is no key.
__global__ void __launch_bounds__(256) k_best_row(const Ctl* ctl, const float* X0, const float* X1,
                                                  const unsigned char* sel0,
                                                  const unsigned char* sel1, long long row0,
                                                  long long rows, long long ld, float* out) {
    const unsigned long long key = ctl->min_key;
    if (key == ~0ull) return;
    const long long r = (long long)(uint32_t)(key & 0xffffffffu) - row0;
    if (r < 0 || r >= rows) return;
    const unsigned char* sel = (ctl->t & 1) ? sel1 : sel0;
    const float* src = (sel != nullptr && sel[r]) ? X1 : X0;
    const float4* s4 = reinterpret_cast<const float4*>(src + r * ld);
    float4* o4 = reinterpret_cast<float4*>(out);
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (ld >> 2);
         q += (long long)gridDim.x * blockDim.x)
        o4[q] = s4[q];
}

__global__ void k_debug_philox(const uint4* ctr, PhiloxKey rk, uint4* out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = Philox::run(ctr[i], rk);
}


// Per-device global table of griewank_h(j), j < cap, grown on demand (evox_eval
// only).  Under stream capture (no allocation allowed) or on any allocation
// failure, nullptr: the kernel then computes h_j per element, with the same bits.
const float* griewank_table(long long ld, int dev, cudaStream_t st, bool no_htab) {
    static std::mutex mu;
    static float* tab[64] = {};
    static long long cap[64] = {};
    if (dev < 0 || dev >= 64 || no_htab) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (cap[dev] < ld) {
        if (tab[dev]) cudaFree(tab[dev]);  // synchronises the device: no reader in flight
        tab[dev] = nullptr;
        cap[dev] = 0;
        float* p = nullptr;
        if (cudaMalloc(&p, (size_t)ld * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        k_griewank_table<<<148, 256, 0, st>>>(p, ld);
        if (cudaGetLastError() != cudaSuccess) {
            cudaFree(p);
            return nullptr;
        }
        // other streams may use the table next: make the fill complete first
        if (cudaStreamSynchronize(st) != cudaSuccess) return nullptr;
        tab[dev] = p;
        cap[dev] = ld;
    }
    return tab[dev];
}

}  // namespace

cudaError_t launch_eval(int problem, const float* X, long long rows, long long D, long long ld,
                        float* fit, cudaStream_t st, bool no_htab) {
    if (rows <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const float* hg = problem == GRIEWANK && geom_id(ld) == 2 ? griewank_table(ld, dev, st, no_htab)
                                                               : nullptr;
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        using GE_ = EVOX_EVAL_GEOM(G_);
        const int g = EVOX_EVAL_WAVES(GE_) > 0
                          ? grid_for((const void*)k_eval<P_, GE_>, row_units<GE_>(rows), dev,
                                     EVOX_EVAL_WAVES(GE_))
                          : (int)row_units<GE_>(rows);
        k_eval<P_, GE_><<<g, 256, 0, st>>>(X, rows, D, ld, fit, hg);
    }));
    return cudaGetLastError();
}

cudaError_t launch_argmin_rows(const float* f, long long rows, long long row0,
                               unsigned long long* key_out, cudaStream_t st) {
    k_argmin_rows<<<1, 1024, 0, st>>>(f, rows, row0, key_out);
    return cudaGetLastError();
}

cudaError_t launch_best_row(const Ctl* ctl, const float* X0, const float* X1,
                            const unsigned char* sel0, const unsigned char* sel1, long long row0,
                            long long rows, long long ld, float* out, cudaStream_t st) {
    long long g = ((ld >> 2) + 255) / 256;
    if (g > 32) g = 32;
    k_best_row<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(ctl, X0, X1, sel0, sel1, row0, rows, ld, out);
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
