// Microbenchmark: which access order reaches the measured copy peak?  1R1W copy of
// 1e9 floats (a -> b) in several thread-to-data mappings; reports GB/s (read + write).
#include <cstdio>
#include <cuda_runtime.h>

// 1: one float4 per thread, non-persistent grid (elementwise-kernel style)
__global__ void k_flat1(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}
// 2: U float4 per thread, block-strided, non-persistent
template <int U>
__global__ void k_flatU(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
    long long i0 = (long long)blockIdx.x * blockDim.x * U + threadIdx.x;
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * blockDim.x < n) r[u] = a[i0 + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * blockDim.x < n) b[i0 + u * blockDim.x] = r[u];
}
// 3: persistent, grid-stride over the flat array, U in flight
template <int U>
__global__ void __launch_bounds__(256, 2) k_pers(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
    const long long T = (long long)gridDim.x * blockDim.x;
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += T * U) {
        float4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i0 + u * T < n) r[u] = a[i0 + u * T];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i0 + u * T < n) b[i0 + u * T] = r[u];
    }
}
// 4: persistent, each CTA owns a contiguous slab; within it block-strided, U in flight
template <int U>
__global__ void __launch_bounds__(256, 2) k_slab(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    const long long s = blockIdx.x * per, e = s + per < n ? s + per : n;
    for (long long i0 = s + threadIdx.x; i0 < e; i0 += 256 * U) {
        float4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i0 + u * 256 < e) r[u] = a[i0 + u * 256];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i0 + u * 256 < e) b[i0 + u * 256] = r[u];
    }
}
// 5: warp per row of nq float4 (the generation kernel's mapping), grid-stride over rows
template <int U>
__global__ void __launch_bounds__(256, 2) k_rows(const float4* __restrict__ a, float4* __restrict__ b, long long rows, long long nq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long stride = (long long)gridDim.x * 8;
    for (long long row = (long long)blockIdx.x * 8 + wid; row < rows; row += stride) {
        for (long long q0 = lane; q0 < nq; q0 += 32 * U) {
            float4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) if (q0 + 32 * u < nq) r[u] = a[row * nq + q0 + 32 * u];
#pragma unroll
            for (int u = 0; u < U; ++u) if (q0 + 32 * u < nq) b[row * nq + q0 + 32 * u] = r[u];
        }
    }
}
// 6: warp per row, rows assigned in contiguous per-warp blocks (warp w owns rows [w*k, (w+1)*k))
template <int U>
__global__ void __launch_bounds__(256, 2) k_rowsblk(const float4* __restrict__ a, float4* __restrict__ b, long long rows, long long nq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long W = (long long)gridDim.x * 8, gw = (long long)blockIdx.x * 8 + wid;
    const long long per = (rows + W - 1) / W;
    const long long r0 = gw * per, r1 = r0 + per < rows ? r0 + per : rows;
    for (long long row = r0; row < r1; ++row) {
        for (long long q0 = lane; q0 < nq; q0 += 32 * U) {
            float4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) if (q0 + 32 * u < nq) r[u] = a[row * nq + q0 + 32 * u];
#pragma unroll
            for (int u = 0; u < U; ++u) if (q0 + 32 * u < nq) b[row * nq + q0 + 32 * u] = r[u];
        }
    }
}

// 3: persistent, grid-stride over the flat array, U in flight
template <int U>
__global__ void __launch_bounds__(256, 8) k_pers8(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
    const long long T = (long long)gridDim.x * blockDim.x;
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += T * U) {
        float4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i0 + u * T < n) r[u] = a[i0 + u * T];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i0 + u * T < n) b[i0 + u * T] = r[u];
    }
}
// 5: warp per row of nq float4 (the generation kernel's mapping), grid-stride over rows
template <int U>
__global__ void __launch_bounds__(256, 8) k_rows8(const float4* __restrict__ a, float4* __restrict__ b, long long rows, long long nq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long stride = (long long)gridDim.x * 8;
    for (long long row = (long long)blockIdx.x * 8 + wid; row < rows; row += stride) {
        for (long long q0 = lane; q0 < nq; q0 += 32 * U) {
            float4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) if (q0 + 32 * u < nq) r[u] = a[row * nq + q0 + 32 * u];
#pragma unroll
            for (int u = 0; u < U; ++u) if (q0 + 32 * u < nq) b[row * nq + q0 + 32 * u] = r[u];
        }
    }
}
template <class F>
void timeit(const char* name, F f, double bytes) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    const int n = 10;
    for (int i = 0; i < n; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"case\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, ms / n, bytes / (ms / n * 1e-3) / 1e9);
}

int main() {
    const long long rows = 1000000, nq = 250, n = rows * nq;
    float4 *A, *B;
    cudaMalloc(&A, n * 16);
    cudaMalloc(&B, n * 16);
    cudaMemset(A, 0, n * 16);
    cudaMemset(B, 0, n * 16);
    const double bytes = 2.0 * n * 16;
    timeit("cudaMemcpy", [&] { cudaMemcpyAsync(B, A, n * 16, cudaMemcpyDeviceToDevice); }, bytes);
    timeit("flat1", [&] { k_flat1<<<(n + 255) / 256, 256>>>(A, B, n); }, bytes);
    timeit("flat4", [&] { k_flatU<4><<<(n + 1023) / 1024, 256>>>(A, B, n); }, bytes);
    timeit("flat8", [&] { k_flatU<8><<<(n + 2047) / 2048, 256>>>(A, B, n); }, bytes);
    timeit("pers4_296", [&] { k_pers<4><<<296, 256>>>(A, B, n); }, bytes);
    timeit("pers8_296", [&] { k_pers<8><<<296, 256>>>(A, B, n); }, bytes);
    timeit("slab4_296", [&] { k_slab<4><<<296, 256>>>(A, B, n); }, bytes);
    timeit("slab8_296", [&] { k_slab<8><<<296, 256>>>(A, B, n); }, bytes);
    timeit("rows4_296", [&] { k_rows<4><<<296, 256>>>(A, B, rows, nq); }, bytes);
    timeit("rows8_296", [&] { k_rows<8><<<296, 256>>>(A, B, rows, nq); }, bytes);
    timeit("rowsblk4_296", [&] { k_rowsblk<4><<<296, 256>>>(A, B, rows, nq); }, bytes);
    timeit("rowsblk8_296", [&] { k_rowsblk<8><<<296, 256>>>(A, B, rows, nq); }, bytes);

    // occupancy: flat1 limited to 2 CTAs/SM through dynamic shared memory
    cudaFuncSetAttribute(k_flat1, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    timeit("flat1_2ctas", [&] { k_flat1<<<(n + 255) / 256, 256, 100 * 1024>>>(A, B, n); }, bytes);
    cudaFuncSetAttribute(k_flatU<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    timeit("flat4_2ctas", [&] { k_flatU<4><<<(n + 1023) / 1024, 256, 100 * 1024>>>(A, B, n); }, bytes);
    timeit("rows4_1184", [&] { k_rows8<4><<<1184, 256>>>(A, B, rows, nq); }, bytes);
    timeit("rows4_np", [&] { k_rows8<4><<<(rows + 7) / 8, 256>>>(A, B, rows, nq); }, bytes);
    timeit("rows1_1184", [&] { k_rows8<1><<<1184, 256>>>(A, B, rows, nq); }, bytes);
    timeit("rows2_1184", [&] { k_rows8<2><<<1184, 256>>>(A, B, rows, nq); }, bytes);
    timeit("pers4_1184", [&] { k_pers8<4><<<1184, 256>>>(A, B, n); }, bytes);
    timeit("pers1_1184", [&] { k_pers8<1><<<1184, 256>>>(A, B, n); }, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
