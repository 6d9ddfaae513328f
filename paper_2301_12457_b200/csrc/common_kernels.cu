// common_kernels.cu -- Problem.evaluate (evox_eval), the argmin query kernel and the
// Philox test hook.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "evox_device.cuh"
#include "evox_internal.h"
#include "row_engine.cuh"

namespace evox {

namespace {

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

__global__ void k_debug_philox(const uint4* ctr, PhiloxKey rk, uint4* out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = Philox::run(ctr[i], rk);
}


}  // namespace

cudaError_t launch_eval(int problem, const float* X, long long rows, long long D, long long ld,
                        float* fit, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    EVOX_DISPATCH_PROB(problem, EVOX_DISPATCH_GEOM(ld, {
        const int g = grid_for((const void*)k_eval<P_, G_>, row_units<G_>(rows), dev);
        carveout((const void*)k_eval<P_, G_>);
        k_eval<P_, G_><<<g, 256, 0, st>>>(X, rows, D, ld, fit);
    }));
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
    const PhiloxKey rk = Philox::schedule(((uint64_t)k1 << 32) | k0);
    k_debug_philox<<<(int)g, 256, 0, st>>>(reinterpret_cast<const uint4*>(ctr), rk,
                                           reinterpret_cast<uint4*>(out), n);
    return cudaGetLastError();
}


}  // namespace evox
