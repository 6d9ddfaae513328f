// Microbenchmark: row-to-warp mapping and occupancy (capped with dynamic smem) for the fused generation's access
// pattern (3R2W: X V P read, X V written; 2R3W: X V read, X V P written), 1e6 x 1000 fp32,
// warp per row, U = 4 float4 chunks in flight per lane, evict-first.  Occupancy is capped with
// dynamic shared memory (the generation kernel runs 2 CTAs/SM at 128 registers).
//   pers : persistent grid (CTAs/SM x 148), static grid-stride rows (current kernel)
//   tick : persistent grid, each warp takes its next row from a global atomic counter
//   np   : non-persistent, one CTA per RPW*8 consecutive rows (block scheduler order)
#include <cstdio>
#include <cuda_runtime.h>

struct St { float4 *X, *V, *P; long long rows, nq; unsigned long long* ctr; };

template <int NR, int NW>
__device__ __forceinline__ void do_row(const St& s, long long row) {
    const int lane = threadIdx.x & 31;
    float4* arr[3] = {s.X + row * s.nq, s.V + row * s.nq, s.P + row * s.nq};
    for (long long b = 0; b < s.nq; b += 128) {
        float4 r[NR][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            long long q = b + 32 * u + lane;
            if (q < s.nq) {
#pragma unroll
                for (int a = 0; a < NR; ++a) r[a][u] = __ldcs(arr[a] + q);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            long long q = b + 32 * u + lane;
            if (q < s.nq) {
                float4 v = r[0][u];
#pragma unroll
                for (int a = 1; a < NR; ++a) { v.x += r[a][u].x; v.y += r[a][u].y; }
#pragma unroll
                for (int a = 0; a < NW; ++a) { __stcs(arr[a] + q, v); v.z += 1.f; }
            }
        }
    }
}

template <int NR, int NW>
__global__ void __launch_bounds__(256) k_pers(St s) {
    const long long stride = (long long)gridDim.x * 8;
    for (long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); row < s.rows; row += stride)
        do_row<NR, NW>(s, row);
}
template <int NR, int NW>
__global__ void __launch_bounds__(256) k_tick(St s) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long row = 0;
        if (lane == 0) row = atomicAdd(s.ctr, 1ull);
        row = __shfl_sync(0xffffffffu, row, 0);
        if ((long long)row >= s.rows) break;
        do_row<NR, NW>(s, (long long)row);
    }
}
template <int NR, int NW, int RPW>
__global__ void __launch_bounds__(256) k_np(St s) {
    const long long r0 = (long long)blockIdx.x * 8 * RPW + (threadIdx.x >> 5);
#pragma unroll 1
    for (int k = 0; k < RPW; ++k) {
        const long long row = r0 + 8 * k;
        if (row < s.rows) do_row<NR, NW>(s, row);
    }
}

template <class K>
void timeit(const char* name, int occ, K kern, int grid, St s, double bytes) {
    // cap residency at `occ` CTAs/SM with dynamic shared memory (228 KB per SM)
    const int smem = occ >= 8 ? 0 : (220 * 1024) / occ - 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int n = 10;
    for (int i = 0; i < 3 + n; ++i) {
        cudaMemsetAsync(s.ctr, 0, 8);
        if (i == 3) cudaEventRecord(a);
        kern<<<grid, 256, smem>>>(s);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&tot, a, b);
    printf("{\"case\": \"%s\", \"occ\": %d, \"grid\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", name, occ, grid,
           tot / n, bytes / (tot / n * 1e-3) / 1e9);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}

int main() {
    St s;
    s.rows = 1000000;
    s.nq = 250;
    const size_t ab = s.rows * s.nq * 16;
    cudaMalloc(&s.X, ab);
    cudaMalloc(&s.V, ab);
    cudaMalloc(&s.P, ab);
    cudaMalloc(&s.ctr, 8);
    cudaMemset(s.X, 0, ab);
    cudaMemset(s.V, 0, ab);
    cudaMemset(s.P, 0, ab);
    const double b5 = 5.0 * ab;
    const int npg1 = (int)((s.rows + 7) / 8), npg4 = (int)((s.rows + 31) / 32);
    for (int occ : {2, 3, 4}) {
        timeit("pers_3R2W", occ, k_pers<3, 2>, 148 * occ, s, b5);
        timeit("tick_3R2W", occ, k_tick<3, 2>, 148 * occ, s, b5);
        timeit("pers_2R3W", occ, k_pers<2, 3>, 148 * occ, s, b5);
        timeit("tick_2R3W", occ, k_tick<2, 3>, 148 * occ, s, b5);
    }
    for (int occ : {2, 4}) {
        timeit("np1_3R2W", occ, k_np<3, 2, 1>, npg1, s, b5);
        timeit("np1_2R3W", occ, k_np<2, 3, 1>, npg1, s, b5);
    }
    timeit("pers_3R2W", 8, k_pers<3, 2>, 148 * 8, s, b5);
    timeit("np1_3R2W", 8, k_np<3, 2, 1>, npg1, s, b5);
    timeit("np4_3R2W", 8, k_np<3, 2, 4>, npg4, s, b5);
    timeit("np1_2R3W", 8, k_np<2, 3, 1>, npg1, s, b5);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
