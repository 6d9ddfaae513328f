// Microbenchmark: CTA-wide bulk-copy ring for the fused generation's 3R2W access pattern
// (X V P read, X V written; 1e6 x 1000 fp32 rows), against the LDG streams of mapping.cu.
//   ring<NC,NS,ST,PH>: one producer warp (lane 0) fills an NS-stage shared-memory ring, one row
//   (X, V, P: 3 x 4000 B) per stage, with cp.async.bulk + mbarrier complete_tx; NC consumer
//   warps each take a whole stage (row), read it with LDS.128, and write X', V' back either with
//   STG.128 (ST = 0) or into the stage + cp.async.bulk shared->global (ST = 1).
//   PH = 1 adds two Philox4x32-10 per quad (the kernel's RNG cost) to the compute.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct St { float4 *X, *V, *P; long long rows, nq; };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t h0 = __umulhi(0xD2511F53u, c.x), l0 = 0xD2511F53u * c.x;
        const uint32_t h1 = __umulhi(0xCD9E8D57u, c.z), l1 = 0xCD9E8D57u * c.z;
        c = make_uint4(h1 ^ c.y ^ k0, l1, h0 ^ c.w ^ k1, l0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

template <int PH>
__device__ __forceinline__ void compute(float4& x, float4& v, const float4 p, int q, uint32_t row) {
    float4 c1 = make_float4(0.25f, 0.25f, 0.25f, 0.25f), c2 = c1;
    if (PH) {
        const uint4 b1 = philox(make_uint4(q, row, 7u, 2u), 11u, 13u);
        const uint4 b2 = philox(make_uint4(q, row, 7u, 3u), 11u, 13u);
        c1 = make_float4((b1.x >> 8) * 0x1p-24f, (b1.y >> 8) * 0x1p-24f, (b1.z >> 8) * 0x1p-24f,
                         (b1.w >> 8) * 0x1p-24f);
        c2 = make_float4((b2.x >> 8) * 0x1p-24f, (b2.y >> 8) * 0x1p-24f, (b2.z >> 8) * 0x1p-24f,
                         (b2.w >> 8) * 0x1p-24f);
    }
    v.x = fmaf(c1.x, p.x - x.x, fmaf(c2.x, -x.x, 0.6f * v.x)); x.x += v.x;
    v.y = fmaf(c1.y, p.y - x.y, fmaf(c2.y, -x.y, 0.6f * v.y)); x.y += v.y;
    v.z = fmaf(c1.z, p.z - x.z, fmaf(c2.z, -x.z, 0.6f * v.z)); x.z += v.z;
    v.w = fmaf(c1.w, p.w - x.w, fmaf(c2.w, -x.w, 0.6f * v.w)); x.w += v.w;
}

template <int NC, int NS, int ST, int PH>
__global__ void __launch_bounds__(32 * (NC + 1)) k_ring(St s) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + NS;
    const int nq = (int)s.nq;
    const uint32_t abytes = nq * 16;
    float4* ring = reinterpret_cast<float4*>(sm + 1024);  // stage k: [3][nq] float4
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long nk = (s.rows - blockIdx.x + gridDim.x - 1) / gridDim.x;  // rows of this CTA
    if (wid == NC) {  // producer
        if (lane == 0) {
            for (long long k = 0; k < nk; ++k) {
                const int st = (int)(k % NS);
                const uint32_t ph = (uint32_t)((k / NS) & 1);
                mbar_wait(&empty[st], ph ^ 1);
                const long long row = blockIdx.x + k * gridDim.x;
                float4* dst = ring + (long long)st * 3 * nq;
                mbar_expect_tx(&full[st], 3 * abytes);
                bulk_g2s(dst, s.X + row * nq, abytes, &full[st]);
                bulk_g2s(dst + nq, s.V + row * nq, abytes, &full[st]);
                bulk_g2s(dst + 2 * nq, s.P + row * nq, abytes, &full[st]);
            }
        }
        return;
    }
    for (long long k = wid; k < nk; k += NC) {
        const int st = (int)(k % NS);
        const uint32_t ph = (uint32_t)((k / NS) & 1);
        mbar_wait(&full[st], ph);
        const long long row = blockIdx.x + k * gridDim.x;
        float4* xs = ring + (long long)st * 3 * nq;
        float4* vs = xs + nq;
        const float4* ps = xs + 2 * nq;
        for (int q = lane; q < nq; q += 32) {
            float4 x = xs[q], v = vs[q];
            compute<PH>(x, v, ps[q], q, (uint32_t)row);
            if (ST) {
                xs[q] = x;
                vs[q] = v;
            } else {
                __stcs(s.X + row * nq + q, x);
                __stcs(s.V + row * nq + q, v);
            }
        }
        if (ST) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                bulk_s2g(s.X + row * nq, xs, abytes);
                bulk_s2g(s.V + row * nq, vs, abytes);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mbar_arrive(&empty[st]);
            }
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
    }
    if (ST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// LDG baseline (mapping.cu np1): one CTA per 8 rows, warp per row, 4 float4 chunks in flight.
template <int PH>
__global__ void __launch_bounds__(256) k_np(St s) {
    const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= s.rows) return;
    float4* X = s.X + row * s.nq;
    float4* V = s.V + row * s.nq;
    const float4* P = s.P + row * s.nq;
    for (int b = 0; b < s.nq; b += 128) {
        float4 x[4], v[4], p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = b + 32 * u + lane;
            if (q < s.nq) { x[u] = __ldcs(X + q); v[u] = __ldcs(V + q); p[u] = __ldcs(P + q); }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = b + 32 * u + lane;
            if (q < s.nq) {
                compute<PH>(x[u], v[u], p[u], q, (uint32_t)row);
                __stcs(X + q, x[u]);
                __stcs(V + q, v[u]);
            }
        }
    }
}

// persistent grid-stride over rows (warp per row), the LDG pattern of the real kernel
template <int PH>
__global__ void __launch_bounds__(256) k_pers(St s) {
    const int lane = threadIdx.x & 31;
    for (long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); row < s.rows;
         row += (long long)gridDim.x * 8) {
        float4* X = s.X + row * s.nq;
        float4* V = s.V + row * s.nq;
        const float4* P = s.P + row * s.nq;
        for (int b = 0; b < s.nq; b += 128) {
            float4 x[4], v[4], p[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = b + 32 * u + lane;
                if (q < s.nq) { x[u] = __ldcs(X + q); v[u] = __ldcs(V + q); p[u] = __ldcs(P + q); }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = b + 32 * u + lane;
                if (q < s.nq) {
                    compute<PH>(x[u], v[u], p[u], q, (uint32_t)row);
                    __stcs(X + q, x[u]);
                    __stcs(V + q, v[u]);
                }
            }
        }
    }
}


// np1 with the real kernel's extra work switched on feature by feature (bits of F):
// 1 gbest row read per quad (__ldg, L1-resident 4 KB); 2 Ackley terms + row reduction +
// f store; 4 per-row imp/pf read + write; 8 lazy pbest: rows flagged pending do not read
// P but write P := X (45 % of rows, as at H).
struct St2 { float4 *X, *V, *P; long long rows, nq; const float4* G; float* f; float* pf;
             unsigned char* imp; };
__device__ __forceinline__ float sinpi_red(float x) {
    const float r = x - rintf(x);
    const float z = r * r;
    float p = fmaf(z, 0.0821458f, -0.5992645f);
    p = fmaf(z, p, 2.5501640f);
    p = fmaf(z, p, -5.1677128f);
    p = fmaf(z, p, 3.1415927f);
    return r * p;
}
template <int F, int MINB, int ORD = 0>
__global__ void __launch_bounds__(256, MINB) k_np2(St2 s) {
    const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= s.rows) return;
    float4* X = s.X + row * s.nq;
    float4* V = s.V + row * s.nq;
    float4* P = s.P + row * s.nq;
    bool pend = false;
    float pf_old = 0.f;
    if (F & 8) pend = s.imp[row] != 0;
    if ((F & 4) && lane == 0) pf_old = s.pf[row];
    float s2 = 0.f, ss = 0.f;
    for (int b = 0; b < s.nq; b += 128) {
        float4 x[4], v[4], p[4];
        if (ORD) {  // X, V of the whole group first: pend is needed only for P
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = b + 32 * u + lane;
                if (q < s.nq) { x[u] = __ldcs(X + q); v[u] = __ldcs(V + q); }
            }
            if (!pend) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = b + 32 * u + lane;
                    if (q < s.nq) p[u] = __ldcs(P + q);
                }
            }
        } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = b + 32 * u + lane;
            if (q < s.nq) {
                x[u] = __ldcs(X + q); v[u] = __ldcs(V + q);
                if (!pend) p[u] = __ldcs(P + q);
            }
        }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = b + 32 * u + lane;
            if (q < s.nq) {
                float4 pb = pend ? x[u] : p[u];
                if (pend) __stcs(P + q, x[u]);
                if (F & 1) {
                    const float4 g = __ldg(s.G + q);
                    pb.x += g.x; pb.y += g.y; pb.z += g.z; pb.w += g.w;
                }
                compute<1>(x[u], v[u], pb, q, (uint32_t)row);
                __stcs(X + q, x[u]);
                __stcs(V + q, v[u]);
                if (F & 2) {
                    const float a[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        s2 = fmaf(a[l], a[l], s2);
                        const float sn = sinpi_red(a[l]);
                        ss = fmaf(sn, sn, ss);
                    }
                }
            }
        }
    }
    if (F & 2) {
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            s2 += __shfl_xor_sync(0xffffffffu, s2, m);
            ss += __shfl_xor_sync(0xffffffffu, ss, m);
        }
        if (lane == 0) s.f[row] = -20.f * expm1f(-0.2f * sqrtf(s2 / 1000.f)) - 2.718f * expm1f(-2.f * ss / 1000.f);
    }
    if ((F & 4) && lane == 0) {
        const float fv = (F & 2) ? s.f[row] : s2;
        const bool imp = fv < pf_old;
        s.imp[row] = imp;
        if (imp) s.pf[row] = fv;
    }
}

template <class K, class S>
void timeit2(const char* name, K kern, int grid, S s, double bytes) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int n = 10;
    for (int i = 0; i < 3 + n; ++i) {
        if (i == 3) cudaEventRecord(a);
        kern<<<grid, 256>>>(s);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&tot, a, b);
    printf("{\"case\": \"%s\", \"occ\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n", name, occ,
           tot / n, bytes / (tot / n * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
}

template <class K>
void timeit(const char* name, K kern, int grid, int block, int smem, St s, double bytes) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
    if (grid == 0) grid = 148 * (occ > 0 ? occ : 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int n = 10;
    for (int i = 0; i < 3 + n; ++i) {
        if (i == 3) cudaEventRecord(a);
        kern<<<grid, block, smem>>>(s);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&tot, a, b);
    cudaError_t e = cudaGetLastError();
    printf("{\"case\": \"%s\", \"occ\": %d, \"grid\": %d, \"smem\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           name, occ, grid, smem, tot / n, bytes / (tot / n * 1e-3) / 1e9, cudaGetErrorString(e));
    fflush(stdout);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}

#define RING(NC, NS, ST, PH, CTAS)                                                              \
    timeit("ring_nc" #NC "_ns" #NS "_st" #ST "_ph" #PH "_x" #CTAS, k_ring<NC, NS, ST, PH>,      \
           148 * CTAS, 32 * (NC + 1), 1024 + NS * 3 * (int)(s.nq * 16), s, b5)

int main() {
    St s;
    s.rows = 1000000;
    s.nq = 250;
    const size_t ab = s.rows * s.nq * 16;
    cudaMalloc(&s.X, ab);
    cudaMalloc(&s.V, ab);
    cudaMalloc(&s.P, ab);
    const double b5 = 5.0 * ab;
    const int npg = (int)((s.rows + 7) / 8);
    cudaMemset(s.X, 0x3f, ab);
    cudaMemset(s.V, 0, ab);
    cudaMemset(s.P, 0x3f, ab);
    timeit("np1_ph1", k_np<1>, npg, 256, 0, s, b5);
    RING(4, 8, 0, 1, 2);
    RING(4, 8, 1, 1, 2);
    RING(4, 4, 0, 1, 3);
    RING(4, 4, 1, 1, 3);
    RING(8, 8, 0, 1, 2);
    RING(8, 8, 1, 1, 2);
    RING(6, 6, 0, 1, 3);
    RING(6, 6, 1, 1, 3);
    RING(8, 16, 0, 1, 1);
    RING(16, 16, 0, 1, 1);
    RING(12, 12, 0, 1, 1);
    RING(2, 4, 0, 1, 4);
    RING(3, 3, 0, 1, 4);
    const double b4 = 4.0 * ab;
    (void)b4;
    return 0;
}
