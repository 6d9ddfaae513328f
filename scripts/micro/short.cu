// Microbenchmark: the fused PSO generation's access pattern at short rows (C4: 1e6 x 100 fp32,
// ld = 100 = 25 float4 quads per row).  3R2W per element (X, V, P read; X, V written) +
// f written per row; optional Philox4x32-10 x2 per quad (PH=1) as the kernel draws r1/r2.
//   lane4 : 4 lanes per row, U chunks in flight per lane (the library's geometry for
//           ld <= 128), persistent grid (MINB CTAs/SM) or wave grid (one CTA per 64 rows)
//   flat  : one CTA per tile of R rows, threads walk the tile's R*25 quads flat (every
//           warp instruction reads 512 contiguous bytes), x' staged in shared memory,
//           then the row sums from shared memory in the lane4 order (RED=1) or no
//           reduction (RED=0, the pure stream)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct St { float4 *X, *V, *P; float* f; long long rows; int nq; };

__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t h0 = __umulhi(0xD2511F53u, c.x), l0 = 0xD2511F53u * c.x;
        const uint32_t h1 = __umulhi(0xCD9E8D57u, c.z), l1 = 0xCD9E8D57u * c.z;
        c = make_uint4(h1 ^ c.y ^ k.x, l1, h0 ^ c.w ^ k.y, l0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

template <int PH>
__device__ __forceinline__ float4 upd(float4 x, float4& v, float4 p, int q, uint32_t row) {
    float c1 = 0.3f, c2 = 0.7f;
    uint4 a = make_uint4(0, 0, 0, 0), b = a;
    if (PH) {
        a = philox(make_uint4(q, row, 5u, 2u), make_uint2(1u, 2u));
        b = philox(make_uint4(q, row, 5u, 3u), make_uint2(1u, 2u));
    }
    float4 o;
#define E(c)                                                                                    \
    {                                                                                           \
        const float r1 = PH ? (a.c >> 8) * (2.5f / 16777216.f) : c1;                            \
        const float r2 = PH ? (b.c >> 8) * (0.8f / 16777216.f) : c2;                            \
        const float vn = fmaf(r2, 0.5f - x.c, fmaf(r1, p.c - x.c, 0.6f * v.c));                 \
        v.c = vn;                                                                               \
        o.c = fminf(fmaxf(x.c + vn, -32.f), 32.f);                                              \
    }
    E(x) E(y) E(z) E(w)
#undef E
    return o;
}

template <int U, int PH, int MINB, int WAVE>
__global__ void __launch_bounds__(256, MINB) k_lane4(St s) {
    const int sl = threadIdx.x & 3;
    const long long r0 = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * 8 + ((threadIdx.x & 31) >> 2);
    const long long stride = WAVE ? s.rows + 64 : (long long)gridDim.x * 64;
    for (long long row = r0; row < s.rows + 7; row += stride) {
        const bool ok = row < s.rows;
        float acc = 0.f;
        float4* X = s.X + row * s.nq;
        float4* V = s.V + row * s.nq;
        float4* P = s.P + row * s.nq;
        for (int base = 0; base < s.nq; base += 4 * U) {
            float4 x[U], v[U], p[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = base + 4 * u + sl;
                if (ok && q < s.nq) { x[u] = __ldcs(X + q); v[u] = __ldcs(V + q); p[u] = __ldcs(P + q); }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = base + 4 * u + sl;
                if (ok && q < s.nq) {
                    float4 vv = v[u];
                    const float4 o = upd<PH>(x[u], vv, p[u], q, (uint32_t)row);
                    __stcs(X + q, o);
                    __stcs(V + q, vv);
                    acc += o.x * o.x; acc += o.y * o.y; acc += o.z * o.z; acc += o.w * o.w;
                }
            }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 2, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1, 4);
        if (ok && sl == 0) s.f[row] = acc;
        if (WAVE) break;
    }
}

// R rows per CTA; the tile's quads are walked flat with K quads per thread in flight.
template <int R, int K, int PH, int RED, int MINB>
__global__ void __launch_bounds__(256, MINB) k_flat(St s) {
    extern __shared__ float4 xs[];  // [R][nq]
    const long long row0 = (long long)blockIdx.x * R;
    const int nrow = s.rows - row0 < R ? (int)(s.rows - row0) : R;
    const int nq = s.nq, n = nrow * nq;
    float4* X = s.X + row0 * nq;
    float4* V = s.V + row0 * nq;
    float4* P = s.P + row0 * nq;
    for (int b = 0; b < n; b += 256 * K) {
        float4 x[K], v[K], p[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = b + 256 * k + threadIdx.x;
            if (i < n) { x[k] = __ldcs(X + i); v[k] = __ldcs(V + i); p[k] = __ldcs(P + i); }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = b + 256 * k + threadIdx.x;
            if (i < n) {
                const int r = i / nq, q = i - r * nq;
                float4 vv = v[k];
                const float4 o = upd<PH>(x[k], vv, p[k], q, (uint32_t)(row0 + r));
                __stcs(X + i, o);
                __stcs(V + i, vv);
                if (RED) xs[i] = o;
                else if (o.x == 12345.f) s.f[0] = o.y;  // keep the value live
            }
        }
    }
    if (!RED) return;
    __syncthreads();
    // lane4 order: row = threadIdx/4, sub-lane sl walks quads sl, sl+4, ...
    for (int t = threadIdx.x; t < R * 4; t += 256) {
        const int r = t >> 2, sl = t & 3;
        float acc = 0.f;
        if (r < nrow)
            for (int q = sl; q < nq; q += 4) {
                const float4 o = xs[r * nq + q];
                acc += o.x * o.x; acc += o.y * o.y; acc += o.z * o.z; acc += o.w * o.w;
            }
        acc += __shfl_xor_sync(0xffffffffu, acc, 2, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1, 4);
        if (r < nrow && sl == 0) s.f[row0 + r] = acc;
    }
}

template <class K>
void timeit(const char* name, K kern, St s, int grid, size_t smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    if (grid <= 0) grid = 148 * occ;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int n = 20;
    for (int i = 0; i < 3 + n; ++i) {
        if (i == 3) cudaEventRecord(a);
        kern<<<grid, 256, smem>>>(s);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= n;
    const double bytes = 20.0 * s.rows * s.nq * 4 + 4.0 * s.rows;
    printf("{\"case\": \"%s\", \"occ\": %d, \"grid\": %d, \"smem\": %zu, \"us\": %.1f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           name, occ, grid, smem, ms * 1e3, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    St s;
    s.rows = 1000000;
    s.nq = 25;
    const size_t nb = (size_t)s.rows * s.nq * 16;
    cudaMalloc(&s.X, nb);
    cudaMalloc(&s.V, nb);
    cudaMalloc(&s.P, nb);
    cudaMalloc(&s.f, s.rows * 4);
    cudaMemset(s.X, 0, nb);
    cudaMemset(s.V, 0, nb);
    cudaMemset(s.P, 0, nb);
    const int wave64 = (int)((s.rows + 63) / 64);
    for (int ph = 0; ph < 2; ++ph) {
#define L4(U, M, W) timeit("lane4_U" #U "_m" #M "_w" #W, ph ? (void (*)(St))k_lane4<U, 1, M, W> : k_lane4<U, 0, M, W>, s, W ? wave64 : 0, 0)
        printf("# PH=%d\n", ph);
        L4(4, 2, 0); L4(2, 3, 0); L4(2, 4, 0); L4(4, 2, 1); L4(2, 4, 1); L4(1, 6, 1);
#define FL(R, K, RED, M) timeit("flat_R" #R "_K" #K "_red" #RED "_m" #M, ph ? (void (*)(St))k_flat<R, K, 1, RED, M> : k_flat<R, K, 0, RED, M>, s, (int)((s.rows + R - 1) / R), RED ? (size_t)R * 25 * 16 : 0)
        FL(32, 1, 1, 6); FL(32, 2, 1, 4); FL(32, 4, 1, 2); FL(64, 2, 1, 4); FL(64, 4, 1, 2); FL(64, 4, 1, 3);
        FL(128, 4, 1, 2); FL(64, 2, 0, 4); FL(64, 4, 0, 2); FL(32, 1, 0, 6); FL(256, 1, 0, 8);
    }
    return 0;
}
