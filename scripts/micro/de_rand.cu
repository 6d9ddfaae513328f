// Microbenchmark: the DE generation's access pattern at D1 (1e6 x 100 fp32): per target row
// read the row itself + 3 donor rows and write one trial row (20 B/element).  Donors are
// random rows (as DE/rand/1 draws them) or the next rows (i+1..i+3, streaming), to separate
// the cost of scattered 400-byte row reads from the kernel's own overheads.
//   LPR lanes per row (4: the kernel's geometry for dim <= 128), U float4 chunks per lane.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct St { const float4* X; float4* T; long long rows, nq; };

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int RAND, int LPR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_de(St s) {
    const int RPW = 32 / LPR;
    const long long row = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * RPW + (threadIdx.x & 31) / LPR;
    const int sl = threadIdx.x & (LPR - 1);
    if (row >= s.rows) return;
    long long r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        r[k] = RAND ? (long long)(((uint64_t)hash32((uint32_t)(row * 3 + k + 1)) * (uint64_t)s.rows) >> 32)
                    : (row + k + 1) % s.rows;
    const float4* xi = s.X + row * s.nq;
    const float4* xa = s.X + r[0] * s.nq;
    const float4* xb = s.X + r[1] * s.nq;
    const float4* xc = s.X + r[2] * s.nq;
    float4* out = s.T + row * s.nq;
    for (int q = sl; q < s.nq; q += LPR) {
        const float4 a = __ldcs(xi + q), b = __ldcg(xa + q), c = __ldcg(xb + q), d = __ldcg(xc + q);
        float4 o;
        o.x = fmaf(0.5f, c.x - d.x, b.x) + 0.f * a.x;
        o.y = fmaf(0.5f, c.y - d.y, b.y) + 0.f * a.y;
        o.z = fmaf(0.5f, c.z - d.z, b.z) + 0.f * a.z;
        o.w = fmaf(0.5f, c.w - d.w, b.w) + 0.f * a.w;
        __stcs(out + q, o);
    }
}

template <class K>
void timeit(const char* name, K kern, St s, double bytes, int lpr) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    const long long rpc = 8LL * (32 / lpr);
    const int grid = (int)((s.rows + rpc - 1) / rpc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int n = 20;
    for (int i = 0; i < 3 + n; ++i) {
        if (i == 3) cudaEventRecord(a);
        kern<<<grid, 256>>>(s);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&tot, a, b);
    printf("{\"case\": \"%s\", \"occ\": %d, \"us\": %.1f, \"GBps\": %.1f, \"err\": \"%s\"}\n", name, occ,
           tot / n * 1e3, bytes / (tot / n * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
}

int main() {
    St s;
    s.rows = 1000000;
    s.nq = 25;
    const size_t ab = s.rows * s.nq * 16;
    float4 *X, *T;
    cudaMalloc(&X, ab);
    cudaMalloc(&T, ab);
    cudaMemset(X, 0x3f, ab);
    s.X = X;
    s.T = T;
    const double bytes = 5.0 * ab;
    timeit("seq_lpr4", k_de<0, 4, 2>, s, bytes, 4);
    timeit("rand_lpr4", k_de<1, 4, 2>, s, bytes, 4);
    timeit("rand_lpr4_m4", k_de<1, 4, 4>, s, bytes, 4);
    timeit("rand_lpr8", k_de<1, 8, 2>, s, bytes, 8);
    timeit("rand_lpr2", k_de<1, 2, 2>, s, bytes, 2);
    timeit("rand_lpr1", k_de<1, 1, 2>, s, bytes, 1);
    timeit("seq_lpr1", k_de<0, 1, 2>, s, bytes, 1);
    // copy reference: 1R1W of the same array size
    return 0;
}
