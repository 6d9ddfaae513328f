// evox_device.cuh -- device building blocks of the B200 PSO/CSO generation.
//
// Written independently of oracle/ (no shared code); both follow PAPER.md /
// SPEC.md and the readings R-1..R-13 of DESIGN.md §3.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace evox {

enum Problem : int { SPHERE = 0, ACKLEY = 1, RASTRIGIN = 2, GRIEWANK = 3, ROSENBROCK = 4 };

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11): R-6.  The multiplies compile to
// IMAD.WIDE.U32 (hi and lo in one instruction); the three-input XORs to LOP3.
// The key schedule k + r*W is uniform across the grid.
// Precomputed key schedule (k + r*W, r = 0..9), passed in the kernel parameter
// block so every round XOR reads its key straight from the constant bank.
struct PhiloxKey {
    uint32_t k0[10];
    uint32_t k1[10];
};

struct Philox {
    static constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    static constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    __host__ __device__ static PhiloxKey schedule(uint64_t seed) {
        PhiloxKey k;
        for (int r = 0; r < 10; ++r) {
            k.k0[r] = (uint32_t)(seed & 0xffffffffu) + (uint32_t)r * W0;
            k.k1[r] = (uint32_t)(seed >> 32) + (uint32_t)r * W1;
        }
        return k;
    }
    __device__ __forceinline__ static uint4 run(uint4 c, const PhiloxKey& k) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint64_t p0 = (uint64_t)M0 * c.x;
            const uint64_t p1 = (uint64_t)M1 * c.z;
            uint4 n;
            n.x = (uint32_t)(p1 >> 32) ^ c.y ^ k.k0[r];
            n.y = (uint32_t)p1;
            n.z = (uint32_t)(p0 >> 32) ^ c.w ^ k.k1[r];
            n.w = (uint32_t)p0;
            c = n;
        }
        return c;
    }
    __device__ __forceinline__ static uint4 run(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint64_t p0 = (uint64_t)M0 * c.x;
            const uint64_t p1 = (uint64_t)M1 * c.z;
            const uint32_t rk0 = k0 + (uint32_t)r * W0, rk1 = k1 + (uint32_t)r * W1;
            uint4 n;
            n.x = (uint32_t)(p1 >> 32) ^ c.y ^ rk0;
            n.y = (uint32_t)p1;
            n.z = (uint32_t)(p0 >> 32) ^ c.w ^ rk1;
            n.w = (uint32_t)p0;
            c = n;
        }
        return c;
    }
};

// 24-bit uniform in [0,1): (b >> 8) * 2^-24 (exact).  R-6.
__device__ __forceinline__ float u24(uint32_t b) {
    return __fmul_rn(__uint2float_rn(b >> 8), 0x1p-24f);
}
// phi * u24(b) in ONE rounding: (b >> 8) * (phi * 2^-24), where phi * 2^-24 is
// exact (the host checks it is a normal float or 0), so the product is the
// same correctly rounded value as phi * ((b >> 8) * 2^-24).
__device__ __forceinline__ float scaled_u24(uint32_t b, float phi_s) {
    return __fmul_rn(__uint2float_rn(b >> 8), phi_s);
}

// -------------------------------------------------------- argmin keys (R-5)
// Order-preserving f32 -> u32 (NaN -> +inf, -0 -> +0); key = ord << 32 | row.
__device__ __forceinline__ uint32_t ord_f32(float f) {
    if (f != f) f = __int_as_float(0x7f800000);
    if (f == 0.0f) f = 0.0f;
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
    const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(b);
}
__device__ __forceinline__ unsigned long long make_key(float f, long long global_row) {
    return ((unsigned long long)ord_f32(f) << 32) | (unsigned long long)(uint32_t)global_row;
}

// ------------------------------------------------------------ memory hints
// Streaming (evict-first) loads/stores for the population: each element is
// touched once per generation and the state (12 GB at the headline config)
// is far larger than L2, so keep L2 for G, bounds, f/pf/imp.
#ifndef EVOX_EF
#define EVOX_EF 3  // bit 0: evict-first loads, bit 1: evict-first stores
#endif
template <bool EF = true>
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    if constexpr ((EVOX_EF & 1) != 0 && EF) return __ldcs(p);
    else return *p;
}
template <bool EF = true>
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
    if constexpr ((EVOX_EF & 2) != 0 && EF) __stcs(p, v);
    else *p = v;
}

// --------------------------------------------------------- fitness (R-7)
// fp32 forms that are algebraically identical to the textbook definitions
// but free of cancellation near the optimum:
//   Ackley:    -20 expm1(-0.2 sqrt(S2/D)) - e expm1(-2 SS/D), SS = sum sin^2(pi x)
//              (sum cos(2 pi x) = D - 2 SS)
//   Rastrigin: sum (x^2 + 20 sin^2(pi x))           (10 - 10 cos 2 pi x = 20 sin^2 pi x)
//   Griewank:  S2/4000 + q, q = 1 - prod cos(x_j h_j) accumulated as the complement
//              product q <- q + a - q a, a_j = 2 sin^2(x_j h_j / 2), h_j = 1/sqrt(j+1)
//   Rosenbrock: sum 100 d^2 + (1-x_j)^2, d = fmaf(-x_j, x_j, x_{j+1})
// Per-lane sequential accumulation, then a fixed xor-shuffle tree and a fixed
// cross-warp order: the reduction order depends on dim only, never on the
// shard, grid or population size (=> bitwise identical across W, R-11).
template <int P> struct Fit;

// sin^2(pi x): sin^2 has period 1, so reduce exactly to r = x - rint(x) in
// [-1/2, 1/2] (Sterbenz) and evaluate sin(pi r) = r P(r^2) with a degree-4
// minimax-style polynomial (fitted on [0, 1/4] in r^2; max relative error of
// the fp32 result ~4e-7).  9 instructions instead of sinpif's ~20.
__device__ __forceinline__ float sinpi_red(float x) {  // sin(pi (x - rint x)), sign irrelevant
    const float r = __fsub_rn(x, rintf(x));
    const float z = __fmul_rn(r, r);
    float p = 0x1.3db042p-4f;
    p = __fmaf_rn(p, z, -0x1.324cd0p-1f);
    p = __fmaf_rn(p, z, 0x1.4668b0p+1f);
    p = __fmaf_rn(p, z, -0x1.4abbc2p+2f);
    p = __fmaf_rn(p, z, 0x1.921fb6p+1f);
    return __fmul_rn(r, p);
}
__device__ __forceinline__ float sin2pi(float x) {
    const float s = sinpi_red(x);
    return __fmul_rn(s, s);
}

template <> struct Fit<SPHERE> {
    float s = 0.0f;
    __device__ __forceinline__ void elem(float x, int64_t) { s = __fmaf_rn(x, x, s); }
    __device__ __forceinline__ void combine(const Fit& o) { s = __fadd_rn(s, o.s); }
    __device__ __forceinline__ void shfl_xor(int m, int w) { s = __shfl_xor_sync(0xffffffffu, s, m, w); }
    __device__ __forceinline__ float finish(int64_t) const { return s; }
};

template <> struct Fit<ACKLEY> {
    float s2 = 0.0f, ss = 0.0f;
    __device__ __forceinline__ void elem(float x, int64_t) {
        s2 = __fmaf_rn(x, x, s2);
        const float sn = sinpi_red(x);
        ss = __fmaf_rn(sn, sn, ss);
    }
    __device__ __forceinline__ void combine(const Fit& o) {
        s2 = __fadd_rn(s2, o.s2);
        ss = __fadd_rn(ss, o.ss);
    }
    __device__ __forceinline__ void shfl_xor(int m, int w) {
        s2 = __shfl_xor_sync(0xffffffffu, s2, m, w);
        ss = __shfl_xor_sync(0xffffffffu, ss, m, w);
    }
    __device__ __forceinline__ float finish(int64_t D) const {
        const float invD = __frcp_rn((float)D);
        const float a = -20.0f * expm1f(-0.2f * sqrtf(__fmul_rn(s2, invD)));
        const float b = -2.718281828459045f * expm1f(-2.0f * __fmul_rn(ss, invD));
        return __fadd_rn(a, b);
    }
};

template <> struct Fit<RASTRIGIN> {
    float s = 0.0f;
    __device__ __forceinline__ void elem(float x, int64_t) {
        const float sn = sinpi_red(x);
        s = __fadd_rn(s, __fmaf_rn(__fmul_rn(20.0f, sn), sn, __fmul_rn(x, x)));
    }
    __device__ __forceinline__ void combine(const Fit& o) { s = __fadd_rn(s, o.s); }
    __device__ __forceinline__ void shfl_xor(int m, int w) { s = __shfl_xor_sync(0xffffffffu, s, m, w); }
    __device__ __forceinline__ float finish(int64_t) const { return s; }
};

// Griewank: a_j = 1 - cos(x_j / sqrt(j+1)) = 2 sin^2(pi z), z = x_j h_j with
// h_j = 1 / (2 pi sqrt(j+1)) (per-column constant: from the CTA's shared-memory
// table when one exists (ld <= 4096), else computed per element: MUFU.RSQ plus one
// Newton step, ~1 ulp -- the correctly rounded __frsqrt_rn cost 2.7x the kernel
// time of evox_eval at dim 1e5; an h_j error of a few ulp moves f far below the
// 1e-5 tolerance, and every kernel uses this same function, so fused and
// standalone fitness stay bitwise equal).
__device__ __forceinline__ float griewank_h(int64_t j) {
    const float x = (float)(j + 1);
    const float y = rsqrtf(x);
    const float r = __fmaf_rn(__fmul_rn(-0.5f * x, y), y, 1.5f);  // 1.5 - x y^2 / 2
    return __fmul_rn(0.15915494309189535f, __fmul_rn(y, r));
}

template <> struct Fit<GRIEWANK> {
    float s2 = 0.0f, q = 0.0f;
    __device__ __forceinline__ void term(float x, float h) {
        s2 = __fmaf_rn(x, x, s2);
        const float sn = sinpi_red(__fmul_rn(x, h));
        const float a = __fmul_rn(2.0f, __fmul_rn(sn, sn));  // 1 - cos(x/sqrt(j+1))
        q = __fmaf_rn(-q, a, __fadd_rn(q, a));               // complement product
    }
    __device__ __forceinline__ void elem(float x, int64_t j) { term(x, griewank_h(j)); }
    __device__ __forceinline__ void combine(const Fit& o) {
        s2 = __fadd_rn(s2, o.s2);
        q = __fmaf_rn(-q, o.q, __fadd_rn(q, o.q));
    }
    __device__ __forceinline__ void shfl_xor(int m, int w) {
        s2 = __shfl_xor_sync(0xffffffffu, s2, m, w);
        q = __shfl_xor_sync(0xffffffffu, q, m, w);
    }
    __device__ __forceinline__ float finish(int64_t) const {
        return __fadd_rn(__fmul_rn(s2, 1.0f / 4000.0f), q);
    }
};

template <> struct Fit<ROSENBROCK> {
    float s = 0.0f;
    __device__ __forceinline__ void elem(float, int64_t) {}
    __device__ __forceinline__ void pair(float x, float xn) {  // term j with x_j, x_{j+1}
        const float d = __fmaf_rn(-x, x, xn);
        const float e = __fsub_rn(1.0f, x);
        s = __fadd_rn(s, __fmaf_rn(__fmul_rn(100.0f, d), d, __fmul_rn(e, e)));
    }
    __device__ __forceinline__ void combine(const Fit& o) { s = __fadd_rn(s, o.s); }
    __device__ __forceinline__ void shfl_xor(int m, int w) { s = __shfl_xor_sync(0xffffffffu, s, m, w); }
    __device__ __forceinline__ float finish(int64_t) const { return s; }
};

// Sphere/Ackley/Rastrigin/Griewank fold all valid lanes of a quad; Rosenbrock
// folds the three intra-quad pairs (the pair crossing into the next quad is
// handled by the row engine with a shuffle / carried value).
template <int P>
__device__ __forceinline__ void fit_quad(Fit<P>& acc, float4 x, int j0, int D,
                                         const float* = nullptr) {
    if (j0 + 3 < D) {
        acc.elem(x.x, j0); acc.elem(x.y, j0 + 1); acc.elem(x.z, j0 + 2); acc.elem(x.w, j0 + 3);
    } else {
        if (j0 < D) acc.elem(x.x, j0);
        if (j0 + 1 < D) acc.elem(x.y, j0 + 1);
        if (j0 + 2 < D) acc.elem(x.z, j0 + 2);
    }
}
template <>
__device__ __forceinline__ void fit_quad<GRIEWANK>(Fit<GRIEWANK>& acc, float4 x, int j0,
                                                   int D, const float* htab) {
    float4 h;
    if (htab) {
        h = *reinterpret_cast<const float4*>(htab + j0);  // LDS.128 of the column constants
    } else {
        h = make_float4(griewank_h(j0), griewank_h(j0 + 1), griewank_h(j0 + 2),
                        griewank_h(j0 + 3));
    }
    if (j0 + 3 < D) {
        acc.term(x.x, h.x); acc.term(x.y, h.y); acc.term(x.z, h.z); acc.term(x.w, h.w);
    } else {
        if (j0 < D) acc.term(x.x, h.x);
        if (j0 + 1 < D) acc.term(x.y, h.y);
        if (j0 + 2 < D) acc.term(x.z, h.z);
    }
}
template <>
__device__ __forceinline__ void fit_quad<ROSENBROCK>(Fit<ROSENBROCK>& acc, float4 x, int j0,
                                                     int D, const float*) {
    if (j0 + 1 < D) acc.pair(x.x, x.y);
    if (j0 + 2 < D) acc.pair(x.y, x.z);
    if (j0 + 3 < D) acc.pair(x.z, x.w);
}

// ---- split fitness fold (the flat-tile kernels): fit_quad == fold_quad(pre_quad(x)).
// pre_quad computes every per-element quantity that does not depend on the running
// accumulator (the expensive part: sin^2 terms, products) where all lanes of a CTA take part;
// fold_quad then applies exactly fit_quad's accumulator operations, in the same order, to the
// staged values -- so a lane that folds a row from staged pre-terms produces bitwise the value
// it would have folded from x.  One float4 per quad (A) or two (A, B: PRE_COMPS == 2).
// Rosenbrock is not split (its pairs straddle quads; the row engine folds it from x).
template <int P>
__host__ __device__ constexpr int pre_comps() { return (P == ACKLEY || P == GRIEWANK) ? 2 : 1; }

template <int P>
__device__ __forceinline__ void pre_quad(float4 x, int j0, const float* htab, float4& A, float4& B);
template <>
__device__ __forceinline__ void pre_quad<SPHERE>(float4 x, int, const float*, float4& A, float4&) {
    A = x;  // s = fmaf(x, x, s)
}
template <>
__device__ __forceinline__ void pre_quad<ACKLEY>(float4 x, int, const float*, float4& A, float4& B) {
    A = x;  // s2 = fmaf(x, x, s2); ss = fmaf(sn, sn, ss)
    B = make_float4(sinpi_red(x.x), sinpi_red(x.y), sinpi_red(x.z), sinpi_red(x.w));
}
__device__ __forceinline__ float rastrigin_term(float x) {
    const float sn = sinpi_red(x);
    return __fmaf_rn(__fmul_rn(20.0f, sn), sn, __fmul_rn(x, x));
}
template <>
__device__ __forceinline__ void pre_quad<RASTRIGIN>(float4 x, int, const float*, float4& A,
                                                    float4&) {
    A = make_float4(rastrigin_term(x.x), rastrigin_term(x.y), rastrigin_term(x.z),
                    rastrigin_term(x.w));  // s = s + term
}
__device__ __forceinline__ float griewank_a(float x, float h) {
    const float sn = sinpi_red(__fmul_rn(x, h));
    return __fmul_rn(2.0f, __fmul_rn(sn, sn));
}
template <>
__device__ __forceinline__ void pre_quad<GRIEWANK>(float4 x, int j0, const float* htab, float4& A,
                                                   float4& B) {
    float4 h;
    if (htab) {
        h = *reinterpret_cast<const float4*>(htab + j0);
    } else {
        h = make_float4(griewank_h(j0), griewank_h(j0 + 1), griewank_h(j0 + 2),
                        griewank_h(j0 + 3));
    }
    A = x;  // s2 = fmaf(x, x, s2); q = fmaf(-q, a, q + a)
    B = make_float4(griewank_a(x.x, h.x), griewank_a(x.y, h.y), griewank_a(x.z, h.z),
                    griewank_a(x.w, h.w));
}

template <int P>
__device__ __forceinline__ void fold_elem(Fit<P>& acc, float a, float b);
template <>
__device__ __forceinline__ void fold_elem<SPHERE>(Fit<SPHERE>& acc, float a, float) {
    acc.s = __fmaf_rn(a, a, acc.s);
}
template <>
__device__ __forceinline__ void fold_elem<ACKLEY>(Fit<ACKLEY>& acc, float a, float b) {
    acc.s2 = __fmaf_rn(a, a, acc.s2);
    acc.ss = __fmaf_rn(b, b, acc.ss);
}
template <>
__device__ __forceinline__ void fold_elem<RASTRIGIN>(Fit<RASTRIGIN>& acc, float a, float) {
    acc.s = __fadd_rn(acc.s, a);
}
template <>
__device__ __forceinline__ void fold_elem<GRIEWANK>(Fit<GRIEWANK>& acc, float a, float b) {
    acc.s2 = __fmaf_rn(a, a, acc.s2);
    acc.q = __fmaf_rn(-acc.q, b, __fadd_rn(acc.q, b));
}
template <int P>
__device__ __forceinline__ void fold_quad(Fit<P>& acc, float4 A, float4 B, int j0, int D) {
    if (j0 + 3 < D) {
        fold_elem<P>(acc, A.x, B.x); fold_elem<P>(acc, A.y, B.y);
        fold_elem<P>(acc, A.z, B.z); fold_elem<P>(acc, A.w, B.w);
    } else {
        if (j0 < D) fold_elem<P>(acc, A.x, B.x);
        if (j0 + 1 < D) fold_elem<P>(acc, A.y, B.y);
        if (j0 + 2 < D) fold_elem<P>(acc, A.z, B.z);
    }
}

}  // namespace evox
