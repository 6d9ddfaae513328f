// Microbenchmark: HBM throughput of the fused PSO generation's access pattern under
// different state layouts (no arithmetic beyond an add).  One warp per row, 4 float4
// chunks in flight per lane, 2 CTAs/SM x 148 SMs, evict-first loads/stores (as the kernel).
//   sep   : X, V, P are three separate [rows x ld] arrays (the current layout)
//   ileav : one [rows x 3 x ld] array (row r of X, V, P adjacent)
// Patterns (arrays read / written per element): copy 1R1W (a -> b), inplace 1R1W,
// 3R3W, 3R2W (X V P read, X V written), 2R3W (X V read, X V P written).
// Reports algorithmic GB/s (bytes the pattern moves / time).
#include <cstdio>
#include <cuda_runtime.h>

template <int NR, int NW, bool EF>
__global__ void __launch_bounds__(256, 2)
k(float4* base, long long rows, long long nq, long long rstride, long long astride, float4* out,
  int copy) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long stride = (long long)gridDim.x * 8;
    for (long long row = (long long)blockIdx.x * 8 + wid; row < rows; row += stride) {
        float4* rb = base + row * rstride;
        for (long long b = 0; b < nq; b += 128) {
            float4 r[NR][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                long long q = b + 32 * u + lane;
                if (q < nq) {
#pragma unroll
                    for (int a = 0; a < NR; ++a) r[a][u] = EF ? __ldcs(rb + a * astride + q) : rb[a * astride + q];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                long long q = b + 32 * u + lane;
                if (q < nq) {
                    float4 s = r[0][u];
#pragma unroll
                    for (int a = 1; a < NR; ++a) { s.x += r[a][u].x; s.y += r[a][u].y; }
#pragma unroll
                    for (int a = 0; a < NW; ++a) {
                        float4* d = copy ? out + row * nq + q : rb + a * astride + q;
                        if (EF) __stcs(d, s); else *d = s;
                        s.z += 1.f;
                    }
                }
            }
        }
    }
}

template <int NR, int NW, bool EF>
void run(const char* name, float4* base, long long rows, long long nq, long long rstride,
         long long astride, float4* out, int copy) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) k<NR, NW, EF><<<296, 256>>>(base, rows, nq, rstride, astride, out, copy);
    cudaEventRecord(a);
    const int n = 10;
    for (int it = 0; it < n; ++it) k<NR, NW, EF><<<296, 256>>>(base, rows, nq, rstride, astride, out, copy);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)(NR + NW) * rows * nq * 16;
    printf("{\"case\": \"%s\", \"ef\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", name, (int)EF, ms / n,
           bytes / (ms / n * 1e-3) / 1e9);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}

int main() {
    const long long rows = 1000000, nq = 250;  // the headline: 1e6 x 1000
    const size_t abytes = rows * nq * 16;
    float4 *S, *O;
    if (cudaMalloc(&S, 3 * abytes) != cudaSuccess || cudaMalloc(&O, abytes) != cudaSuccess) return 1;
    cudaMemset(S, 0, 3 * abytes);
    cudaMemset(O, 0, abytes);
    const long long A = rows * nq;  // separate: array stride
#define BOTH(NR, NW, nm)                                                        \
    run<NR, NW, true>("sep_" nm, S, rows, nq, nq, A, O, 0);                     \
    run<NR, NW, true>("ileav_" nm, S, rows, nq, 3 * nq, nq, O, 0);              \
    run<NR, NW, false>("sep_" nm, S, rows, nq, nq, A, O, 0);                    \
    run<NR, NW, false>("ileav_" nm, S, rows, nq, 3 * nq, nq, O, 0);
    run<1, 1, true>("copy", S, rows, nq, nq, A, O, 1);
    run<1, 1, false>("copy", S, rows, nq, nq, A, O, 1);
    run<1, 1, true>("inplace1", S, rows, nq, nq, A, O, 0);
    BOTH(3, 3, "3R3W")
    BOTH(3, 2, "3R2W")
    BOTH(2, 3, "2R3W")
    BOTH(2, 2, "2R2W")
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
