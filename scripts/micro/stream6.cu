// Microbenchmark: the fused PSO kernel's memory pattern without its arithmetic.
// Each warp streams rows of ld floats: reads X, V, P (float4, evict-first) and writes
// X', V', P (evict-first), with the same next-row L2 bulk prefetch.  Reports GB/s.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void pf(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <bool PREF>
__global__ void __launch_bounds__(256, 2) k(float4* X, float4* V, float4* P, long long rows, long long nq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long stride = (long long)gridDim.x * 8;
    for (long long row = (long long)blockIdx.x * 8 + wid; row < rows; row += stride) {
        if (PREF && lane == 0 && row + stride < rows) {
            pf(X + (row + stride) * nq, nq * 16);
            pf(V + (row + stride) * nq, nq * 16);
            pf(P + (row + stride) * nq, nq * 16);
        }
        for (long long b = 0; b < nq; b += 128) {
            float4 x[4], v[4], p[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                long long q = b + 32 * u + lane;
                if (q < nq) {
                    const long long o = row * nq + q;
                    x[u] = __ldcs(X + o); v[u] = __ldcs(V + o); p[u] = __ldcs(P + o);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                long long q = b + 32 * u + lane;
                if (q < nq) {
                    const long long o = row * nq + q;
                    float4 a = x[u], c = v[u], d = p[u];
                    a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
                    __stcs(X + o, a); __stcs(V + o, c); __stcs(P + o, d);
                }
            }
        }
    }
}

int main() {
    const long long rows = 1000000, nq = 250;  // the headline: 1e6 x 1000
    const size_t bytes = rows * nq * 16;
    float4 *X, *V, *P;
    cudaMalloc(&X, bytes); cudaMalloc(&V, bytes); cudaMalloc(&P, bytes);
    cudaMemset(X, 0, bytes); cudaMemset(V, 0, bytes); cudaMemset(P, 0, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int pref = 0; pref < 2; ++pref) {
        for (int it = 0; it < 3; ++it) pref ? k<true><<<296, 256>>>(X, V, P, rows, nq) : k<false><<<296, 256>>>(X, V, P, rows, nq);
        cudaEventRecord(a);
        const int n = 10;
        for (int it = 0; it < n; ++it) pref ? k<true><<<296, 256>>>(X, V, P, rows, nq) : k<false><<<296, 256>>>(X, V, P, rows, nq);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = 6.0 * bytes / (ms / n * 1e-3) / 1e9;
        printf("{\"prefetch\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", pref, ms / n, gbs);
    }
    return 0;
}
