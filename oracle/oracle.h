/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the EvoX PSO/CSO
 * generation (arXiv 2301.12457).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.  It shares no code with the
 * CUDA path (paper_2301_12457_b200/csrc): no headers, helpers, tables or
 * constants generators.  Both sides are written independently from the same
 * passages (PAPER.md "P:N", SPEC.md "S:N") and from the readings frozen in
 * DESIGN.md §3.
 *
 * Layout: every matrix here is DENSE row-major [rows x D] (no padding); the
 * GPU's padded [rows x ld] views are converted by the tests.  `row0` is the
 * GLOBAL index of the first row passed, so the oracle can recompute any
 * sampled subset of a large population one row at a time.
 *
 * Precision (reading R-10): positions/velocities are fp32 with the
 * exact operation sequence of the paper's update (explicit fmaf, compiled
 * with -ffp-contract=off); fitness is the textbook definition in fp64.
 */
#ifndef EVOX_ORACLE_H
#define EVOX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_SPHERE = 0, ORC_ACKLEY = 1, ORC_RASTRIGIN = 2, ORC_GRIEWANK = 3, ORC_ROSENBROCK = 4 };

/* Philox4x32-10 (Salmon et al., SC'11 "Random123"; the counter-based key of
 * P:253/P:293, generator choice R-6).  out = philox(ctr, key). */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* top 24 bits -> [0,1):  (b >> 8) * 2^-24  (R-6). */
float oracle_uniform24(uint32_t b);

/* R[r][j] = uniform24(philox((j/4, row0+r, t, tag), seed)[j%4]), dense [rows x D]. */
void oracle_draw(int64_t rows, int64_t D, int64_t row0, uint64_t t, uint32_t tag,
                 uint64_t seed, float* R);

/* Fitness, textbook fp64 definitions (R-7), X dense fp32 [rows x D] -> F [rows]. */
void oracle_eval(int problem, int64_t rows, int64_t D, const float* X, double* F, int threads);

/* PSO (gbest PSO with inertia, P:700 / S:313-316, R-1..R-5). */
/* Init (R-3): X0 = fmaf(u, ub-lb, lb) with u from tag 0 at t = 0; V0 = 0. */
void oracle_pso_init(int64_t rows, int64_t D, int64_t row0, const float* lb, const float* ub,
                     uint64_t seed, float* X, float* V);
/* Move with caller-supplied r1, r2 (dense [rows x D]); in place on X, V.
 * G is the gbest row [D].  a=P-X; b=G-X; c1=phi_p*r1; c2=phi_g*r2;
 * v=fmaf(c2,b,fmaf(c1,a,w*V)); x=fminf(fmaxf(X+v,lb),ub). */
void oracle_pso_move_with(int64_t rows, int64_t D, float* X, float* V, const float* P,
                          const float* G, const float* R1, const float* R2,
                          float w, float phi_p, float phi_g, const float* lb, const float* ub);
/* Move drawing r1 (tag 2) and r2 (tag 3) at generation t. */
void oracle_pso_move(int64_t rows, int64_t D, int64_t row0, uint64_t t, uint64_t seed,
                     float* X, float* V, const float* P, const float* G,
                     float w, float phi_p, float phi_g, const float* lb, const float* ub,
                     int threads);
/* Per-row pbest replacement: imp_i = f_i < pf_i (strict; NaN never improves);
 * if imp: P_i = X_i, pf_i = f_i.  Writes imp[rows] (0/1). */
void oracle_pso_tell_rows(int64_t rows, int64_t D, const float* X, const float* f,
                          float* P, float* pf, uint8_t* imp);
/* argmin over f32 with the lowest index on ties, NaN treated as +inf.
 * Returns the local index; *fmin gets f[i*] (NaN mapped to +inf). */
int64_t oracle_argmin(int64_t rows, const float* f, float* fmin);

/* Unified tell of one generation over W simulated shards (R-11),
 * given the f32 fitness f [N] of X: pbest replacement (strict), each
 * shard's argmin (lowest index on ties), shard winners combined by
 * (fitness, global index), then gbest G [D] / *gf / *gidx move only
 * on a strict improvement over the incumbent *gf (R-5).
 * *hist_t = the generation's minimum f32 (NaN as +inf). */
void oracle_pso_tell(int64_t N, int64_t D, int W, const float* X, const float* f, float* P,
                     float* pf, float* G, float* gf, int64_t* gidx, float* hist_t);

/* Whole PSO run, simulated-W mode (R-11): W contiguous row shards (sizes
 * differ by <= 1); every shard finds its local winner, then the winners are
 * combined by (fitness, global index) and gbest moves on strict improvement.
 * Fresh state: evaluate X0 + tell at t=0, then n x (move(t), t+=1, eval, tell).
 * In/out: X, V, P dense [N x D]; pf [N]; G [D]; *gf, *gidx; hist [n+1]
 * (hist[t] = min f32 of generation t); f [N] = last fitness (f32);
 * F64 [N] = last fitness in fp64.  If `fresh` is 0 the state is continued
 * from generation t0 (X already evaluated, pf/P/G/gf valid). */
void oracle_pso_run(int problem, int64_t N, int64_t D, const float* lb, const float* ub,
                    float w, float phi_p, float phi_g, uint64_t seed, int64_t n_gens,
                    int W, int fresh, int64_t t0,
                    float* X, float* V, float* P, float* pf, float* f, double* F64,
                    float* G, float* gf, int64_t* gidx, float* hist, int threads);

/* The same driver as oracle_pso_run, from a caller-supplied initial state X, V
 * (not yet evaluated; P := X, pf = gf = +inf, gidx = -1, G = 0) and with
 * injected r1 = R1, r2 = R2, dense [n_gens x N x D] (the test hook that
 * replays the hand-worked trajectory through this driver).  hist [n_gens+1]. */
void oracle_pso_run_with(int problem, int64_t N, int64_t D, const float* lb, const float* ub,
                         float w, float phi_p, float phi_g, int64_t n_gens, int W,
                         float* X, float* V, float* P, float* pf, float* f, double* F64,
                         float* G, float* gf, int64_t* gidx, float* hist,
                         const float* R1, const float* R2);

/* CSO (Cheng & Jin, IEEE TCYB 2015; listed in Table II), R-8. */
/* pi_{t,blk} on [0,B): 4-round Feistel on b=max(2,ceil(log2 B)) (even) bits,
 * round keys philox((blk,0,t,4),seed), cycle-walked into [0,B). */
uint32_t oracle_cso_perm(uint32_t x, uint32_t B, uint32_t blk, uint64_t t, uint64_t seed);
/* Loser update with caller-supplied R1, R2, R3 [D] (test hook). */
void oracle_cso_loser_update_with(int64_t D, const float* xw, float* xl, float* vl,
                                  const float* R1, const float* R2, const float* R3, float phi,
                                  const float* xbar, const float* lb, const float* ub);
/* One CSO generation at t, in place on X, V, f (f32) and F64.  Blocks of B rows
 * (the last may be shorter); pairs (pi(2p), pi(2p+1)); the lower f (ties: lower
 * global index) wins; the loser: v = fmaf(R2, Xw-Xl, R1*Vl) [+ phi*R3*(xbar-Xl)],
 * x = clip(Xl+v), re-evaluated.  xbar = fp64 column mean of X rounded to fp32. */
void oracle_cso_generation(int problem, int64_t N, int64_t D, int64_t B, uint64_t t,
                           uint64_t seed, float phi, const float* lb, const float* ub,
                           float* X, float* V, float* f, double* F64, int threads);

/* DE/rand/1/bin (Storn & Price 1997, the DE of the paper's experiment P:700,
 * P:748-750), reading R-14 of DESIGN.md. */
/* Donor indices of target i at generation t: the word stream
 * philox((c, i, t, 8), seed)[l], c = 0,1,.. l = 0..3, each mapped to [0,N) by
 * (w * N) >> 32; r1 = first != i, r2 = next not in {i,r1}, r3 = next not in
 * {i,r1,r2}.  N >= 4. */
void oracle_de_indices(int64_t N, int64_t i, uint64_t t, uint64_t seed, int64_t out[3]);
/* Forced crossover dimension: (philox((0, i, t, 9), seed)[0] * D) >> 32. */
int64_t oracle_de_jrand(int64_t D, int64_t i, uint64_t t, uint64_t seed);
/* Trial with caller-supplied crossover uniforms U[D]: v = fmaf(F, xb - xc, xa);
 * u_j = clip(U_j < CR || j == jrand ? v_j : xi_j). */
void oracle_de_trial_with(int64_t D, const float* xi, const float* xa, const float* xb,
                          const float* xc, const float* U, int64_t jrand, float F, float CR,
                          const float* lb, const float* ub, float* u);
/* One synchronous DE generation at t, in place: every trial is built from the
 * population of generation t (U_j = uniform24(philox((j/4, i, t, 10))[j%4])),
 * evaluated (fp64), and replaces its target iff f(u) <= f(x) with NaN ranked
 * as +inf.  f = f32 of F64. */
void oracle_de_generation(int problem, int64_t N, int64_t D, float* X, float* f, double* F64,
                          float F, float CR, uint64_t t, uint64_t seed, const float* lb,
                          const float* ub, int threads);

#ifdef __cplusplus
}
#endif
#endif
