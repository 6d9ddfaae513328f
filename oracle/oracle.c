/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C99, compiled
 * -O2 -ffp-contract=off (no fast-math), optional OpenMP over independent rows
 * (used only to time the oracle; results do not depend on the thread count
 * because every row is computed independently and every reduction below is a
 * sequential loop in index order).
 *
 * Every function cites the passage it follows.  The paper gives no equations
 * for PSO/CSO or the test functions; where it is silent the reading from
 * DESIGN.md §3 (R-1..R-13) is followed and cited as "R-k".
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ Philox */
/* Random123 Philox4x32 round function (Salmon et al. SC'11, Fig. 2 / Table 2):
 * (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0)),
 * Weyl key schedule k0 += 0x9E3779B9, k1 += 0xBB67AE85 between rounds. */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    int r;
    for (r = 0; r < 10; ++r) {
        uint64_t p0, p1;
        uint32_t n0, n1, n2, n3;
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        n1 = (uint32_t)p1;
        n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R-6: 24-bit uniform in [0,1). */
float oracle_uniform24(uint32_t b) { return (float)(b >> 8) * 0x1p-24f; }

static void key_of(uint64_t seed, uint32_t key[2]) {
    key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
    key[1] = (uint32_t)(seed >> 32);
}

/* R-6 counter layout: ctr = (column quad q = j/4, global row, generation, stream tag). */
static float draw_one(int64_t j, int64_t row, uint64_t t, uint32_t tag, const uint32_t key[2]) {
    uint32_t ctr[4], out[4];
    ctr[0] = (uint32_t)(j / 4);
    ctr[1] = (uint32_t)row;
    ctr[2] = (uint32_t)t;
    ctr[3] = tag;
    oracle_philox4x32_10(ctr, key, out);
    return oracle_uniform24(out[j % 4]);
}

void oracle_draw(int64_t rows, int64_t D, int64_t row0, uint64_t t, uint32_t tag,
                 uint64_t seed, float* R) {
    uint32_t key[2];
    int64_t r, j;
    key_of(seed, key);
    for (r = 0; r < rows; ++r)
        for (j = 0; j < D; ++j) R[r * D + j] = draw_one(j, row0 + r, t, tag, key);
}

/* ------------------------------------------------------------- functions */
/* R-7: textbook definitions, evaluated in fp64 over the fp32 positions.
 * Sphere is the function of the paper's experiment. */
static double f_sphere(int64_t D, const float* x) {
    double s = 0.0;
    int64_t j;
    for (j = 0; j < D; ++j) s += (double)x[j] * (double)x[j];
    return s;
}

/* Ackley, a=20, b=0.2, c=2*pi. */
static double f_ackley(int64_t D, const float* x) {
    const double pi = 3.14159265358979323846;
    double s2 = 0.0, sc = 0.0;
    int64_t j;
    for (j = 0; j < D; ++j) {
        double v = (double)x[j];
        s2 += v * v;
        sc += cos(2.0 * pi * v);
    }
    return -20.0 * exp(-0.2 * sqrt(s2 / (double)D)) - exp(sc / (double)D) + 20.0 + exp(1.0);
}

/* Rastrigin, A=10. */
static double f_rastrigin(int64_t D, const float* x) {
    const double pi = 3.14159265358979323846;
    double s = 10.0 * (double)D;
    int64_t j;
    for (j = 0; j < D; ++j) {
        double v = (double)x[j];
        s += v * v - 10.0 * cos(2.0 * pi * v);
    }
    return s;
}

/* Griewank, 1-based index in the sqrt. */
static double f_griewank(int64_t D, const float* x) {
    double s = 0.0, p = 1.0;
    int64_t j;
    for (j = 0; j < D; ++j) {
        double v = (double)x[j];
        s += v * v;
        p *= cos(v / sqrt((double)(j + 1)));
    }
    return 1.0 + s / 4000.0 - p;
}

/* Rosenbrock, sum over j < D-1 (D = 1 -> 0). */
static double f_rosenbrock(int64_t D, const float* x) {
    double s = 0.0;
    int64_t j;
    for (j = 0; j + 1 < D; ++j) {
        double a = (double)x[j], b = (double)x[j + 1];
        s += 100.0 * (b - a * a) * (b - a * a) + (1.0 - a) * (1.0 - a);
    }
    return s;
}

static double eval_row(int problem, int64_t D, const float* x) {
    switch (problem) {
        case ORC_SPHERE: return f_sphere(D, x);
        case ORC_ACKLEY: return f_ackley(D, x);
        case ORC_RASTRIGIN: return f_rastrigin(D, x);
        case ORC_GRIEWANK: return f_griewank(D, x);
        case ORC_ROSENBROCK: return f_rosenbrock(D, x);
        default: return NAN;
    }
}

static void set_threads(int threads) {
#ifdef _OPENMP
    omp_set_num_threads(threads > 0 ? threads : 1);
#else
    (void)threads;
#endif
}

/* Problem.evaluate (Table I, Eq. (2); S:444 row-wise purity). */
void oracle_eval(int problem, int64_t rows, int64_t D, const float* X, double* F, int threads) {
    int64_t r;
    set_threads(threads);
#pragma omp parallel for schedule(static)
    for (r = 0; r < rows; ++r) F[r] = eval_row(problem, D, X + r * D);
}

/* ------------------------------------------------------------------- PSO */
/* R-3 / S:315: X0 uniform in [lb,ub], V0 = 0. */
void oracle_pso_init(int64_t rows, int64_t D, int64_t row0, const float* lb, const float* ub,
                     uint64_t seed, float* X, float* V) {
    uint32_t key[2];
    int64_t r, j;
    key_of(seed, key);
    for (r = 0; r < rows; ++r) {
        for (j = 0; j < D; ++j) {
            float u = draw_one(j, row0 + r, 0, 0, key);
            float span = ub[j] - lb[j];
            X[r * D + j] = fmaf(u, span, lb[j]);
            V[r * D + j] = 0.0f;
        }
    }
}

/* Canonical gbest PSO with inertia (Kennedy & Eberhart, cited at P:700;
 * v <- w v + c1 r1 (pbest - x) + c2 r2 (gbest - x); x <- x + v),
 * operation order R-1, clip R-4 (positions only, velocity not clamped). */
void oracle_pso_move_with(int64_t rows, int64_t D, float* X, float* V, const float* P,
                          const float* G, const float* R1, const float* R2,
                          float w, float phi_p, float phi_g, const float* lb, const float* ub) {
    int64_t r, j;
    for (r = 0; r < rows; ++r) {
        for (j = 0; j < D; ++j) {
            int64_t k = r * D + j;
            float x = X[k];
            float a = P[k] - x;
            float b = G[j] - x;
            float c1 = phi_p * R1[k];
            float c2 = phi_g * R2[k];
            float wv = w * V[k];
            float v = fmaf(c2, b, fmaf(c1, a, wv));
            float xn = fminf(fmaxf(x + v, lb[j]), ub[j]);
            V[k] = v;
            X[k] = xn;
        }
    }
}

void oracle_pso_move(int64_t rows, int64_t D, int64_t row0, uint64_t t, uint64_t seed,
                     float* X, float* V, const float* P, const float* G,
                     float w, float phi_p, float phi_g, const float* lb, const float* ub,
                     int threads) {
    int64_t r;
    set_threads(threads);
#pragma omp parallel for schedule(static)
    for (r = 0; r < rows; ++r) {
        uint32_t key[2];
        float* r1 = (float*)malloc(sizeof(float) * (size_t)(D > 0 ? D : 1));
        float* r2 = (float*)malloc(sizeof(float) * (size_t)(D > 0 ? D : 1));
        int64_t j;
        key_of(seed, key);
        for (j = 0; j < D; ++j) {
            r1[j] = draw_one(j, row0 + r, t, 2, key);
            r2[j] = draw_one(j, row0 + r, t, 3, key);
        }
        oracle_pso_move_with(1, D, X + r * D, V + r * D, P + r * D, G, r1, r2, w, phi_p, phi_g,
                             lb, ub);
        free(r1);
        free(r2);
    }
}

/* tell, pbest part ("strict improvement; ties keep incumbent"; R-5). */
void oracle_pso_tell_rows(int64_t rows, int64_t D, const float* X, const float* f,
                          float* P, float* pf, uint8_t* imp) {
    int64_t r;
    for (r = 0; r < rows; ++r) {
        int better = f[r] < pf[r]; /* NaN compares false: never improves */
        imp[r] = (uint8_t)better;
        if (better) {
            memcpy(P + r * D, X + r * D, sizeof(float) * (size_t)D);
            pf[r] = f[r];
        }
    }
}

/* gbest argmin (S:285 lowest index on ties; R-5 NaN as +inf). */
int64_t oracle_argmin(int64_t rows, const float* f, float* fmin) {
    int64_t r, best = 0;
    float bv = INFINITY;
    for (r = 0; r < rows; ++r) {
        float v = isnan(f[r]) ? INFINITY : f[r];
        if (r == 0 || v < bv) {
            bv = v;
            best = r;
        }
    }
    if (fmin) *fmin = bv;
    return best;
}

/* Tell of one generation over W simulated shards, given the generation's f32
 * fitness (every node evaluates its shard, the results are
 * all-gathered, and one unified tell follows; R-11 contiguous slices
 * differing by <= 1).  Order (Listing 1, R-2): pbest
 * first (S:316 strict, ties keep the incumbent), then each shard's winner
 * (S:285 lowest index on ties), the shard winners combined by (fitness,
 * global index) (S:349 first encountered on ties), and gbest moves only on a
 * strict improvement over the incumbent (R-5). */
void oracle_pso_tell(int64_t N, int64_t D, int W, const float* X, const float* f, float* P,
                     float* pf, float* G, float* gf, int64_t* gidx, float* hist_t) {
    uint8_t* imp = (uint8_t*)malloc((size_t)(N > 0 ? N : 1));
    float best_f = INFINITY;
    int64_t best_i = -1, r0 = 0;
    int s;
    oracle_pso_tell_rows(N, D, X, f, P, pf, imp);
    for (s = 0; s < W; ++s) {
        int64_t rows = N / W + (s < N % W ? 1 : 0);
        if (rows > 0) {
            float lf;
            int64_t li = oracle_argmin(rows, f + r0, &lf) + r0;
            /* combine shard winners by (fitness, global index) */
            if (best_i < 0 || lf < best_f || (lf == best_f && li < best_i)) {
                best_f = lf;
                best_i = li;
            }
        }
        r0 += rows;
    }
    *hist_t = best_f;
    if (best_f < *gf) { /* strict improvement (R-5) */
        *gf = best_f;
        *gidx = best_i;
        memcpy(G, X + best_i * D, sizeof(float) * (size_t)D);
    }
    free(imp);
}

/* Problem.evaluate (Eq. (2)) in fp64, rounded to f32 for every decision
 * (R-9/R-10), then the unified tell. */
static void eval_and_tell(int problem, int64_t N, int64_t D, int W, float* X, float* P,
                          float* pf, float* f, double* F64, float* G, float* gf,
                          int64_t* gidx, float* hist_t, int threads) {
    int64_t i;
    oracle_eval(problem, N, D, X, F64, threads);
    for (i = 0; i < N; ++i) f[i] = (float)F64[i];
    oracle_pso_tell(N, D, W, X, f, P, pf, G, gf, gidx, hist_t);
}

/* The stateful driver behind oracle_pso_run and oracle_pso_run_with:
 * Workflow.step (Listing 2; Eqs. (1)-(3) P:443-447), order R-2:
 * the state rests after evaluation; a fresh state is evaluated + told at t=0,
 * then every generation is move(t) -> t+1 -> evaluate -> tell.
 * mode 0: continue from generation t0; 1: fresh, X0/V0 from the seed (R-3);
 * 2: fresh from the caller's X, V.  R1/R2 NULL: draw r1/r2 from Philox (tags
 * 2, 3, R-6); else injected, dense [n_gens x N x D] (test hook). */
static void pso_driver(int problem, int64_t N, int64_t D, const float* lb, const float* ub,
                       float w, float phi_p, float phi_g, uint64_t seed, int64_t n_gens, int W,
                       int mode, int64_t t0, float* X, float* V, float* P, float* pf, float* f,
                       double* F64, float* G, float* gf, int64_t* gidx, float* hist,
                       int threads, const float* R1, const float* R2) {
    int64_t g, t = t0, k = 0;
    if (mode != 0) {
        int64_t i;
        if (mode == 1) oracle_pso_init(N, D, 0, lb, ub, seed, X, V);
        memcpy(P, X, sizeof(float) * (size_t)(N * D));
        for (i = 0; i < N; ++i) pf[i] = INFINITY;
        *gf = INFINITY;
        *gidx = -1;
        for (i = 0; i < D; ++i) G[i] = 0.0f;
        t = 0;
        eval_and_tell(problem, N, D, W, X, P, pf, f, F64, G, gf, gidx, &hist[k++], threads);
    }
    for (g = 0; g < n_gens; ++g) {
        if (R1 == NULL)
            oracle_pso_move(N, D, 0, (uint64_t)t, seed, X, V, P, G, w, phi_p, phi_g, lb, ub,
                            threads);
        else
            oracle_pso_move_with(N, D, X, V, P, G, R1 + g * N * D, R2 + g * N * D, w, phi_p,
                                 phi_g, lb, ub);
        t += 1;
        eval_and_tell(problem, N, D, W, X, P, pf, f, F64, G, gf, gidx, &hist[k++], threads);
    }
}

void oracle_pso_run(int problem, int64_t N, int64_t D, const float* lb, const float* ub,
                    float w, float phi_p, float phi_g, uint64_t seed, int64_t n_gens,
                    int W, int fresh, int64_t t0,
                    float* X, float* V, float* P, float* pf, float* f, double* F64,
                    float* G, float* gf, int64_t* gidx, float* hist, int threads) {
    pso_driver(problem, N, D, lb, ub, w, phi_p, phi_g, seed, n_gens, W, fresh ? 1 : 0, t0, X, V,
               P, pf, f, F64, G, gf, gidx, hist, threads, NULL, NULL);
}

void oracle_pso_run_with(int problem, int64_t N, int64_t D, const float* lb, const float* ub,
                         float w, float phi_p, float phi_g, int64_t n_gens, int W,
                         float* X, float* V, float* P, float* pf, float* f, double* F64,
                         float* G, float* gf, int64_t* gidx, float* hist,
                         const float* R1, const float* R2) {
    pso_driver(problem, N, D, lb, ub, w, phi_p, phi_g, 0, n_gens, W, 2, 0, X, V, P, pf, f, F64,
               G, gf, gidx, hist, 1, R1, R2);
}

/* ------------------------------------------------------------------- CSO */
/* R-8: keyed block-local bijection (4-round Feistel + cycle walking). */
static uint32_t feistel(uint32_t x, int h, const uint32_t k[4]) {
    uint32_t mask = (h >= 32) ? 0xFFFFFFFFu : ((1u << h) - 1u);
    uint32_t L = (x >> h) & mask, R = x & mask;
    int r;
    for (r = 0; r < 4; ++r) {
        uint32_t F = (uint32_t)((R ^ k[r]) * 0x9E3779B1u) >> (32 - h);
        uint32_t nL = R, nR = (L ^ F) & mask;
        L = nL;
        R = nR;
    }
    return (L << h) | R;
}

uint32_t oracle_cso_perm(uint32_t x, uint32_t B, uint32_t blk, uint64_t t, uint64_t seed) {
    uint32_t key[2], ctr[4], k[4];
    int b = 0, h;
    uint32_t y;
    while (b < 32 && (1ull << b) < (uint64_t)B) ++b; /* ceil(log2 B) */
    if (b < 2) b = 2;
    if (b & 1) ++b;
    h = b / 2;
    key_of(seed, key);
    ctr[0] = blk;
    ctr[1] = 0;
    ctr[2] = (uint32_t)t;
    ctr[3] = 4;
    oracle_philox4x32_10(ctr, key, k);
    y = feistel(x, h, k);
    while (y >= B) y = feistel(y, h, k);
    return y;
}

/* CSO loser update (Cheng & Jin 2015, Eqs. (6)-(7); R-8):
 * v_l = R1*v_l + R2*(x_w - x_l) [+ phi*R3*(xbar - x_l)], x_l = clip(x_l + v_l),
 * in the fixed order v = fmaf(R2, xw-xl, R1*vl); v = fmaf(phi*R3, xbar-xl, v). */
void oracle_cso_loser_update_with(int64_t D, const float* xw, float* xl, float* vl,
                                  const float* R1, const float* R2, const float* R3, float phi,
                                  const float* xbar, const float* lb, const float* ub) {
    int64_t j;
    for (j = 0; j < D; ++j) {
        float x = xl[j];
        float v = fmaf(R2[j], xw[j] - x, R1[j] * vl[j]);
        if (phi != 0.0f) v = fmaf(phi * R3[j], xbar[j] - x, v);
        vl[j] = v;
        xl[j] = fminf(fmaxf(x + v, lb[j]), ub[j]);
    }
}

/* Competitive swarm optimizer generation (Cheng & Jin 2015, Table II):
 * pairwise competition, winner passes unchanged, loser learns from winner. */
void oracle_cso_generation(int problem, int64_t N, int64_t D, int64_t B, uint64_t t,
                           uint64_t seed, float phi, const float* lb, const float* ub,
                           float* X, float* V, float* f, double* F64, int threads) {
    uint32_t key[2];
    float* xbar = (float*)malloc(sizeof(float) * (size_t)(D > 0 ? D : 1));
    int64_t nblk = (N + B - 1) / B, blk;
    key_of(seed, key);
    if (phi != 0.0f) {
        for (int64_t j = 0; j < D; ++j) {
            double s = 0.0;
            int64_t i;
            for (i = 0; i < N; ++i) s += (double)X[i * D + j];
            xbar[j] = (float)(s / (double)N);
        }
    }
    set_threads(threads);
    for (blk = 0; blk < nblk; ++blk) {
        int64_t base = blk * B;
        int64_t Bb = (base + B <= N) ? B : (N - base);
        int64_t p;
#pragma omp parallel for schedule(static)
        for (p = 0; p < Bb / 2; ++p) {
            int64_t i = base + oracle_cso_perm((uint32_t)(2 * p), (uint32_t)Bb, (uint32_t)blk, t, seed);
            int64_t k = base + oracle_cso_perm((uint32_t)(2 * p + 1), (uint32_t)Bb, (uint32_t)blk, t, seed);
            float fi = isnan(f[i]) ? INFINITY : f[i];
            float fk = isnan(f[k]) ? INFINITY : f[k];
            int64_t w, l;
            if (fi < fk || (fi == fk && i < k)) {
                w = i;
                l = k;
            } else {
                w = k;
                l = i;
            }
            {
                float* R = (float*)malloc(sizeof(float) * (size_t)(3 * (D > 0 ? D : 1)));
                for (int64_t j = 0; j < D; ++j) {
                    R[j] = draw_one(j, l, t, 5, key);
                    R[D + j] = draw_one(j, l, t, 6, key);
                    R[2 * D + j] = (phi != 0.0f) ? draw_one(j, l, t, 7, key) : 0.0f;
                }
                oracle_cso_loser_update_with(D, X + w * D, X + l * D, V + l * D, R, R + D,
                                             R + 2 * D, phi, xbar, lb, ub);
                free(R);
            }
            F64[l] = eval_row(problem, D, X + l * D);
            f[l] = (float)F64[l];
        }
    }
    free(xbar);
}

/* ------------------------------------------------------------------- DE */
/* Donor indices (R-14): rejection sampling on a counter-based word stream. */
void oracle_de_indices(int64_t N, int64_t i, uint64_t t, uint64_t seed, int64_t out[3]) {
    uint32_t key[2], ctr[4], w[4];
    int64_t got = 0;
    uint32_t c = 0;
    key_of(seed, key);
    while (got < 3) {
        int l;
        ctr[0] = c++;
        ctr[1] = (uint32_t)i;
        ctr[2] = (uint32_t)t;
        ctr[3] = 8;
        oracle_philox4x32_10(ctr, key, w);
        for (l = 0; l < 4 && got < 3; ++l) {
            int64_t r = (int64_t)(((uint64_t)w[l] * (uint64_t)N) >> 32);
            int ok = r != i, k;
            for (k = 0; k < got; ++k) ok = ok && r != out[k];
            if (ok) out[got++] = r;
        }
    }
}

int64_t oracle_de_jrand(int64_t D, int64_t i, uint64_t t, uint64_t seed) {
    uint32_t key[2], ctr[4], w[4];
    key_of(seed, key);
    ctr[0] = 0;
    ctr[1] = (uint32_t)i;
    ctr[2] = (uint32_t)t;
    ctr[3] = 9;
    oracle_philox4x32_10(ctr, key, w);
    return (int64_t)(((uint64_t)w[0] * (uint64_t)D) >> 32);
}

/* Mutation v = x_a + F (x_b - x_c) and binomial crossover. */
void oracle_de_trial_with(int64_t D, const float* xi, const float* xa, const float* xb,
                          const float* xc, const float* U, int64_t jrand, float F, float CR,
                          const float* lb, const float* ub, float* u) {
    int64_t j;
    for (j = 0; j < D; ++j) {
        float v = fmaf(F, xb[j] - xc[j], xa[j]);
        float y = (U[j] < CR || j == jrand) ? v : xi[j];
        u[j] = fminf(fmaxf(y, lb[j]), ub[j]);
    }
}

static float nan_as_inf(float v) { return isnan(v) ? INFINITY : v; }

/* One-to-one greedy replacement, "trial replaces target iff trial fitness <=
 * target fitness", synchronous over the population. */
void oracle_de_generation(int problem, int64_t N, int64_t D, float* X, float* f, double* F64,
                          float F, float CR, uint64_t t, uint64_t seed, const float* lb,
                          const float* ub, int threads) {
    float* T = (float*)malloc(sizeof(float) * (size_t)(N * D > 0 ? N * D : 1));
    double* FT = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    int64_t i;
    set_threads(threads);
#pragma omp parallel for schedule(static)
    for (i = 0; i < N; ++i) {
        uint32_t key[2];
        int64_t r[3], j, jr;
        float* U = (float*)malloc(sizeof(float) * (size_t)(D > 0 ? D : 1));
        key_of(seed, key);
        oracle_de_indices(N, i, t, seed, r);
        jr = oracle_de_jrand(D, i, t, seed);
        for (j = 0; j < D; ++j) U[j] = draw_one(j, i, t, 10, key);
        oracle_de_trial_with(D, X + i * D, X + r[0] * D, X + r[1] * D, X + r[2] * D, U, jr, F, CR,
                             lb, ub, T + i * D);
        FT[i] = eval_row(problem, D, T + i * D);
        free(U);
    }
    for (i = 0; i < N; ++i) {
        float fu = (float)FT[i];
        if (nan_as_inf(fu) <= nan_as_inf(f[i])) {
            memcpy(X + i * D, T + i * D, sizeof(float) * (size_t)D);
            f[i] = fu;
            F64[i] = FT[i];
        }
    }
    free(T);
    free(FT);
}
