/*
 * evox.h -- C-ABI of the B200-native EvoX PSO/CSO generation engine
 * (arXiv 2301.12457).  Implemented by paper_2301_12457_b200/libevox.so.
 *
 * The calls follow the paper's programming model: Algorithm.setup/ask/tell,
 * Problem.evaluate, Workflow.init/step (Table I, Listing 1
 * P:233-277, Listing 2) and the state transitions of Eqs. (1)-(3)
 * (P:443-447).  The error taxonomy follows SPEC: invalid-argument (S:64,
 * S:130), shape, contract violation, configuration
 * (S:72).  Readings "R-k" are listed in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *  - Returns evox_status; nothing throws or aborts across the ABI.  On any
 *    non-OK status evox_last_error() describes the failure (thread-local).
 *  - Arguments are validated synchronously, before any device work.
 *  - "dev" pointers are CUDA device pointers on the handle's device; "host"
 *    pointers are ordinary host memory (pageable or pinned).
 *  - Matrices are fp32 row-major with a leading dimension ld = round_up(dim,4)
 *    floats (16-byte aligned rows, padding columns held at 0).
 *  - Device state is owned by the handle (library cudaMalloc) unless the
 *    caller passes a workspace in evox_opts, which must then outlive the
 *    handle.  Host arrays passed in are copied; nothing is retained.
 *  - A handle must not be used from two threads at once.  Work is enqueued
 *    asynchronously on the handle's stream; calls documented as
 *    "synchronising" wait for it.  An asynchronous CUDA or NCCL failure is
 *    reported by the next synchronising call as EVOX_ERR_CUDA/EVOX_ERR_NCCL
 *    and POISONS the handle: every later call except *_destroy returns
 *    EVOX_ERR_POISONED.
 */
#ifndef EVOX_H
#define EVOX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVOX_ABI_VERSION 2

typedef enum {
    EVOX_OK = 0,
    EVOX_ERR_INVALID_ARGUMENT = 1, /* bad value: NULL, non-finite, lb >= ub, unknown enum */
    EVOX_ERR_SHAPE = 2,            /* sizes inconsistent or overflowing */
    EVOX_ERR_CONTRACT = 3,         /* call order / state contract violated */
    EVOX_ERR_OUT_OF_MEMORY = 4,    /* device or workspace too small */
    EVOX_ERR_CUDA = 5,             /* CUDA runtime failure (handle poisoned) */
    EVOX_ERR_NCCL = 6,             /* NCCL failure or NCCL unavailable (handle poisoned) */
    EVOX_ERR_POISONED = 7,         /* handle unusable after an earlier CUDA/NCCL failure */
    EVOX_ERR_CONFIG = 8,           /* configuration error, e.g. CSO block size vs shards */
    EVOX_ERR_EXCHANGE = 9          /* peer-memory exchange timed out (a peer stopped; poisoned) */
} evox_status;

/* Numerical test functions (R-7).  Sphere is the function of the paper's
 * scaling experiment; the other four are among the "numerical test
 * functions" of P:36. */
typedef enum {
    EVOX_SPHERE = 0,     /* sum x^2 */
    EVOX_ACKLEY = 1,     /* -20 exp(-0.2 sqrt(sum x^2/D)) - exp(sum cos(2 pi x)/D) + 20 + e */
    EVOX_RASTRIGIN = 2,  /* 10 D + sum (x^2 - 10 cos 2 pi x) */
    EVOX_GRIEWANK = 3,   /* 1 + sum x^2/4000 - prod cos(x_j / sqrt(j+1)) (j 0-based) */
    EVOX_ROSENBROCK = 4  /* sum_{j<D-1} 100 (x_{j+1} - x_j^2)^2 + (1 - x_j)^2 */
} evox_problem;

/* Fields exposed by evox_pso_view / evox_cso_view. */
typedef enum {
    EVOX_FIELD_X = 0,  /* positions  [rows x ld] f32 */
    EVOX_FIELD_V = 1,  /* velocities [rows x ld] f32 */
    EVOX_FIELD_P = 2,  /* pbest positions [rows x ld] f32 (PSO only; materialised first) */
    EVOX_FIELD_F = 3,  /* fitness of the current population [rows] f32 */
    EVOX_FIELD_PF = 4, /* pbest fitness [rows] f32 (PSO only) */
    EVOX_FIELD_G = 5   /* gbest position [ld] f32 (PSO only), rows = 1 */
} evox_field;

typedef struct evox_pso evox_pso; /* opaque handles */
typedef struct evox_cso evox_cso;
typedef struct evox_de evox_de;

/* Per-handle execution options (all optional: pass NULL for the defaults). */
typedef struct {
    void* cuda_stream;       /* cudaStream_t to enqueue on; NULL: the library creates a
                                non-blocking stream owned by the handle.  The legacy
                                default stream (0) is NOT accepted as "NULL" here. */
    const uint8_t* nccl_id;  /* 128-byte ncclUniqueId (from evox_nccl_unique_id on rank 0,
                                broadcast by the caller): world > 1 uses NCCL for the
                                exchange unless evox_pso_connect() switches the handle to
                                the in-kernel peer-memory exchange (then it may be NULL) */
    int rank;                /* this process's shard, 0 <= rank < world (SPMD) */
    int world;               /* number of shards/GPUs; 0 or 1: single GPU */
    int device;              /* CUDA device ordinal; -1: the calling thread's current device */
    void* workspace;         /* optional device buffer for the state (see *_workspace_bytes) */
    size_t workspace_bytes;
    uint32_t flags;          /* EVOX_FLAG_* bits; 0: the library picks every execution path */
    int peer_timeout_ms;     /* peer-memory exchange wait limit (<= 0: 60 000 ms) */
} evox_opts;

/* evox_opts.flags.  They select among execution paths that are tested to give the SAME
 * trajectory bitwise (same per-row reduction order, same decisions); they exist so tests
 * can reach every path on one GPU.  No environment variable selects an execution path (the
 * only one the library reads is EVOX_NCCL_LIB, a path to libnccl.so.2). */
enum {
    EVOX_FLAG_NO_SMALL = 1u << 0,   /* never run a step in the single-CTA persistent kernel */
    EVOX_FLAG_NO_MID = 1u << 1,     /* never run a step in the cooperative persistent kernel */
    EVOX_FLAG_TMA = 1u << 2,        /* PSO, 32 < ld/4 <= 1024: bulk-copy-staged generation kernel */
    EVOX_FLAG_FORCE_NCCL = 1u << 3, /* world == 1: run the NCCL exchange path on a 1-rank
                                       communicator (exercises the multi-GPU code) */
    EVOX_FLAG_NO_GRAPH = 1u << 4,   /* launch generations directly, not through CUDA graphs */
    EVOX_FLAG_NO_WAVE = 1u << 5     /* PSO, > 2^25 elements, and DE with rows of <= 256 floats: the
                                       grid-stride row-walk generation kernel instead of the
                                       one-CTA-per-row-block wave / flat-tile kernels */
};

/* Description of the last failure on the calling thread ("" if none). */
const char* evox_last_error(void);
/* Library version string; also the ABI version as an integer. */
const char* evox_version(void);
int evox_abi_version(void);

/* Row sharding (R-11; "W contiguous row-slices, sizes differing by
 * <= 1"): rows [*row0, *row0 + *rows) of a population of `pop` belong to
 * `rank` of `world`.  Pure host arithmetic. */
evox_status evox_shard_rows(int64_t pop, int world, int rank, int64_t* row0, int64_t* rows);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 calls it; the caller
 * broadcasts it, e.g. through torch.distributed).  NCCL is loaded lazily
 * (dlopen libnccl.so.2); EVOX_ERR_NCCL if it cannot be loaded. */
evox_status evox_nccl_unique_id(uint8_t out[128]);

/* ---------------------------------------------------------------- Problem */
/* Problem.evaluate (Table I; Eq. (2)): fit[i] = f(X[i, :dim]) for
 * i < pop.  X: dev [pop x ld] f32 (ld >= dim, ld % 4 == 0, 16-byte aligned);
 * fit: dev [pop] f32.  Row-wise pure: fit[i] depends only on row i,
 * with a reduction order fixed by dim alone.  Asynchronous on cuda_stream
 * (NULL = legacy default stream).  pop == 0 is a no-op.  ld > 2^31 - 4 ->
 * EVOX_ERR_SHAPE (in-row indices are 32-bit; the same cap applies to dim at
 * every init). */
evox_status evox_eval(evox_problem problem, const float* X, int64_t pop, int64_t dim, int64_t ld,
                      float* fit, void* cuda_stream);
/* evox_eval with flags: EVOX_EVAL_NO_HTAB computes the Griewank column constants per
 * element instead of reading the per-device table (bitwise the same; test hook). */
enum { EVOX_EVAL_NO_HTAB = 1u << 0 };
evox_status evox_eval_ex(evox_problem problem, const float* X, int64_t pop, int64_t dim,
                         int64_t ld, float* fit, void* cuda_stream, uint32_t flags);

/* ---------------------------------------------------------------- PSO */
/* Workspace bytes a handle of this shape needs (for evox_opts.workspace). */
evox_status evox_pso_workspace_bytes(int64_t pop, int64_t dim, int world, int rank, size_t* bytes);

/* Algorithm.setup + Workflow.init (Listing 1 setup P:251-263; R-1, R-3):
 * gbest PSO with inertia w and acceleration coefficients phi_p (cognitive,
 * pbest) and phi_g (social, gbest) -- S:313-316 defaults 0.6, 2.5, 0.8.
 * lb, ub: host [dim] bounds, finite, lb[j] < ub[j].  seed keys the Philox
 * stream (R-6).  Enqueues X0 ~ U[lb,ub] (fp32 fmaf form), V0 = 0, P0 = X0,
 * pf = gf = +inf for this rank's rows (evox_shard_rows).  Every rank calls
 * it with identical arguments (SPMD).  *out receives the handle. */
evox_status evox_pso_init(int64_t pop, int64_t dim, const float* lb, const float* ub, float w,
                          float phi_p, float phi_g, uint64_t seed, const evox_opts* opts,
                          evox_pso** out);

/* Workflow.step x n_gens (Listing 2; Eqs. (1)-(3); order R-2):
 * on a fresh handle first evaluates X0 and tells (generation 0), then runs
 * n_gens fused generations [move -> evaluate -> tell] (+ the per-generation
 * gbest exchange when world > 1).  The problem is bound by the
 * first evaluation; a different problem later -> EVOX_ERR_CONTRACT.
 * n_gens >= 0.  Asynchronous (CUDA-graph replay of per-generation kernels; on
 * one rank, populations of <= 2^16 elements run the n_gens in one single-CTA
 * launch and <= 2^25 elements in one cooperative launch with a grid barrier
 * per generation -- the same trajectory bitwise).  A barrier that times out
 * (10 s) makes the next synchronising call return EVOX_ERR_EXCHANGE. */
evox_status evox_pso_step(evox_pso* s, evox_problem problem, int64_t n_gens);

/* Unfused Algorithm.ask (Table I; Eq. (1)): the first ask on a fresh handle
 * returns X0 unmoved; every later ask moves X_t -> X_{t+1} (R-1, R-4) and
 * returns it.  *X_dev: borrowed dev [rows x ld], valid until the next call
 * on the handle.  Requires the state to be at rest (not already asked). */
evox_status evox_pso_ask(evox_pso* s, const float** X_dev, int64_t* rows, int64_t* ld);

/* Unfused Algorithm.tell (Table I; Eq. (3)): fit_dev: dev [rows] f32,
 * the fitness of the rows the last ask returned (this rank's rows).  Applies
 * pbest (strict <), the gbest argmin (lowest global index on ties, strict
 * improvement; R-5) and, for world > 1, the winner exchange.  Without a
 * preceding ask -> EVOX_ERR_CONTRACT. */
evox_status evox_pso_tell(evox_pso* s, const float* fit_dev);

/* Synchronising.  Best-so-far fitness, its GLOBAL row index (-1 before any
 * finite fitness) and, if row_host != NULL, the gbest position (host [dim]). */
evox_status evox_pso_best(evox_pso* s, float* fit, int64_t* global_index, float* row_host);

/* Synchronising.  Per-generation minimum fitness of the population,
 * hist[t] for t = 0..T (the Monitor's record_fit).
 * Copies min(cap, T+1) values to host best_per_gen; *n = T+1. */
evox_status evox_pso_history(evox_pso* s, float* best_per_gen, int64_t cap, int64_t* n);

/* Borrowed device pointer to one field of this rank's state (evox_field).
 * Valid until the next step/ask/tell/load/destroy.  For EVOX_FIELD_P the
 * lazily-pending pbest rows are materialised first (bitwise-neutral for
 * later generations).  Synchronising. */
evox_status evox_pso_view(evox_pso* s, int field, void** dev, int64_t* rows, int64_t* ld);

/* Synchronising.  Shape/progress: global pop, dim, ld, this rank's row0/rows,
 * the current generation t (index of the current population; -1 before the
 * first evaluation) and the stream the handle enqueues on. */
evox_status evox_pso_info(evox_pso* s, int64_t* pop, int64_t* dim, int64_t* ld, int64_t* row0,
                          int64_t* rows, int64_t* t, void** cuda_stream);

/* Checkpoint / resume (the state is a pure value).  save writes
 * a self-describing blob of this rank's state to host memory (size query:
 * host_blob = NULL, *used = bytes needed).  load restores a blob saved from
 * a handle of identical shape, params and rank.  Both synchronising. */
evox_status evox_pso_save(evox_pso* s, void* host_blob, size_t cap, size_t* used);
evox_status evox_pso_load(evox_pso* s, const void* host_blob, size_t size);

/* Wait for all work enqueued on the handle; surfaces asynchronous errors. */
evox_status evox_pso_sync(evox_pso* s);

/* Kernel timing (measurement aid).  While enabled, every
 * generation kernel (fused PSO generation / CSO generation) is bracketed by
 * CUDA events on the handle's stream and generations are launched directly
 * instead of through CUDA graphs.  kernel_time synchronises and returns the
 * summed device time in ms and the number of generations those launches ran
 * since the last reset (one per launch, except the persistent small-population
 * kernel, which runs all n generations of a step in one launch) and the
 * number of those launches (NULL pointers are skipped); reset != 0 clears
 * the counters after reading. */
evox_status evox_pso_set_timing(evox_pso* s, int enable);
evox_status evox_pso_kernel_time(evox_pso* s, double* total_ms, int64_t* gens, int64_t* launches,
                                 int reset);
/* The same for the gbest-publication kernel k_pso_fin, which follows the generation kernel
 * when the exchange is the in-kernel peer exchange (world > 1) or the population runs on
 * the wave grid: its summed device time (the key-first exchange, the staged / pulled winner
 * row, G) and launch count since the last reset.  Synchronising. */
evox_status evox_pso_fin_time(evox_pso* s, double* total_ms, int64_t* launches, int reset);

/* In-kernel peer-memory exchange (the paper's per-
 * iteration all-gather, done on the device right after each
 * generation kernel by the gbest-publication kernel, with no host involvement).
 * Every handle owns a device "mailbox" of 2 x world slots {u64 flag; u64 key;
 * f32 row[ld]}.  KEY FIRST: a rank whose local minimum can still improve gbest
 * stages that row in its OWN slot[gen parity][rank]; every rank writes only its
 * 8-byte key and a release flag into slot[parity][rank] of EVERY rank's mailbox
 * (NVLink peer stores), waits for the world keys in its own mailbox, picks the
 * minimum (lowest global index on ties) and, on a strict improvement, pulls that
 * one row from the winner's mailbox into its gbest -- no NCCL launch, no select
 * kernel, one row over NVLink per rank per improving generation.
 *
 * evox_pso_mailbox: this handle's mailbox (device pointer and size).
 * evox_pso_mailbox_ipc: its cudaIpcMemHandle (64 bytes) for other processes.
 * evox_pso_connect: mode 0 -- `peers` is an array of `world` device pointers
 *   (the mailboxes of all ranks, same process; GPUs must be peer-capable);
 *   mode 1 -- `peers` is world x 64 bytes of IPC handles (entry `rank` is
 *   ignored).  All ranks must connect before any of them steps.  A rank
 *   that waits more than 60 s (evox_opts.peer_timeout_ms) for
 *   its peers stops waiting, flags the handle and the next synchronising
 *   call returns EVOX_ERR_EXCHANGE.  Single-
 *   process groups must not grow their history during a step (steps that
 *   would are pre-sized at connect time for 1<<16 generations). */
evox_status evox_pso_mailbox(evox_pso* s, void** dev, size_t* bytes);
evox_status evox_pso_mailbox_ipc(evox_pso* s, uint8_t out[64]);
evox_status evox_pso_connect(evox_pso* s, int mode, const void* peers);

/* Release the handle (never fails for a valid or poisoned handle; NULL ok). */
evox_status evox_pso_destroy(evox_pso* s);

/* ---------------------------------------------------------------- CSO */
/* Competitive swarm optimizer (Table II; R-8).  pop >= 2; block = the
 * pairing block size B (0 = default pop/8 rounded to a valid size; B >= 2,
 * B = pop: global pairing).  world > 1: when every shard holds whole blocks
 * the shards are independent (NCCL only reduces the per-generation minima);
 * otherwise pairs straddle shards and the ranks must be connected
 * (evox_cso_state / evox_cso_connect, as for DE): each rank updates the losers
 * it owns, reading partner fitness and winner rows through peer memory, with
 * an in-kernel barrier + global minimum per generation.
 * phi: social factor of the mean-position term (0 by default).  phi != 0 adds
 * a per-generation column mean x-bar of the whole population (R-15: exact
 * fixed-point sums; with world > 1 the ranks' sums are combined through peer
 * memory when connected, else with one NCCL all-reduce -- bitwise the same
 * trajectory for every world size). */
evox_status evox_cso_workspace_bytes(int64_t pop, int64_t dim, int world, int rank, size_t* bytes);
evox_status evox_cso_init(int64_t pop, int64_t dim, const float* lb, const float* ub, float phi,
                          int64_t block, uint64_t seed, const evox_opts* opts, evox_cso** out);
/* First call evaluates X0 (generation 0); then n_gens CSO generations. */
evox_status evox_cso_step(evox_cso* s, evox_problem problem, int64_t n_gens);
/* Synchronising: current minimum fitness over the whole population and its
 * global index (+ row to host if row_host != NULL).  world > 1 reduces over
 * ranks. */
evox_status evox_cso_best(evox_cso* s, float* fit, int64_t* global_index, float* row_host);
/* Synchronising: hist[t] = min f of generation t over the whole population. */
evox_status evox_cso_history(evox_cso* s, float* best_per_gen, int64_t cap, int64_t* n);
evox_status evox_cso_view(evox_cso* s, int field, void** dev, int64_t* rows, int64_t* ld);
evox_status evox_cso_info(evox_cso* s, int64_t* pop, int64_t* dim, int64_t* ld, int64_t* row0,
                          int64_t* rows, int64_t* t, void** cuda_stream);
evox_status evox_cso_load(evox_cso* s, const void* host_blob, size_t size);
evox_status evox_cso_save(evox_cso* s, void* host_blob, size_t cap, size_t* used);
evox_status evox_cso_sync(evox_cso* s);
evox_status evox_cso_state(evox_cso* s, void** base, uint8_t ipc[64]);
evox_status evox_cso_connect(evox_cso* s, int mode, const void* peers);
evox_status evox_cso_set_timing(evox_cso* s, int enable);
evox_status evox_cso_kernel_time(evox_cso* s, double* total_ms, int64_t* gens, int64_t* launches,
                                 int reset);
evox_status evox_cso_destroy(evox_cso* s);

/* ---------------------------------------------------------------- DE */
/* DE/rand/1/bin (Storn & Price 1997; the DE of the paper's scaling
 * experiment; reading R-14).  Each
 * generation builds, for every target i, three distinct donors r1,r2,r3 != i
 * (rejection sampling on a Philox word stream: O(1) per target at any pop),
 * the mutant v = fmaf(F, x_r2 - x_r3, x_r1), the binomial crossover with rate
 * CR and a forced dimension, clips it to [lb,ub], evaluates it and replaces
 * the target iff f(trial) <= f(target) (NaN ranks as +inf).  F finite,
 * CR in [0,1] (defaults 0.5, 0.9); pop >= 4, else EVOX_ERR_CONFIG.
 * The first step evaluates X0 (generation 0).  Row-sharded (world > 1, up to
 * 8): donors are drawn from the WHOLE population, so every rank maps every
 * other rank's state (evox_de_state -> IPC handle or pointer, then
 * evox_de_connect before the first step) and reads remote donor rows over
 * NVLink inside the generation kernel; each generation ends with an in-kernel
 * barrier + global minimum through per-rank mailboxes (same timeout and
 * EVOX_ERR_EXCHANGE semantics as evox_pso_connect).  Results are bitwise
 * identical for every world. */
evox_status evox_de_workspace_bytes(int64_t pop, int64_t dim, size_t* bytes);
evox_status evox_de_init(int64_t pop, int64_t dim, const float* lb, const float* ub, float F,
                         float CR, uint64_t seed, const evox_opts* opts, evox_de** out);
evox_status evox_de_step(evox_de* s, evox_problem problem, int64_t n_gens);
/* Synchronising: minimum fitness of the current population, its index, row. */
evox_status evox_de_best(evox_de* s, float* fit, int64_t* global_index, float* row_host);
evox_status evox_de_history(evox_de* s, float* best_per_gen, int64_t cap, int64_t* n);
/* EVOX_FIELD_X (current population, gathered into one buffer first) or
 * EVOX_FIELD_F.  Synchronising; valid until the next step. */
evox_status evox_de_view(evox_de* s, int field, void** dev, int64_t* rows, int64_t* ld);
evox_status evox_de_info(evox_de* s, int64_t* pop, int64_t* dim, int64_t* ld, int64_t* row0,
                         int64_t* rows, int64_t* t, void** cuda_stream);
/* Checkpoint / resume of this rank's DE state (the population is gathered into
 * one buffer first; same blob rules as evox_pso_save/load).  Synchronising. */
evox_status evox_de_save(evox_de* s, void* host_blob, size_t cap, size_t* used);
evox_status evox_de_load(evox_de* s, const void* host_blob, size_t size);
evox_status evox_de_sync(evox_de* s);
/* The state allocation of this rank: device base pointer and/or its 64-byte
 * cudaIpcMemHandle (NULL outputs are skipped). */
evox_status evox_de_state(evox_de* s, void** base, uint8_t ipc[64]);
/* mode 0: `peers` = world device pointers (evox_de_state bases, same process);
 * mode 1: world x 64-byte IPC handles (entry `rank` ignored). */
evox_status evox_de_connect(evox_de* s, int mode, const void* peers);
evox_status evox_de_set_timing(evox_de* s, int enable);
evox_status evox_de_kernel_time(evox_de* s, double* total_ms, int64_t* gens, int64_t* launches,
                                int reset);
evox_status evox_de_destroy(evox_de* s);

/* ---------------------------------------------------------------- test hooks */
/* out[4i..4i+3] = Philox4x32-10(ctr[4i..4i+3], (key0,key1)) computed by the
 * device function the kernels use.  ctr, out: dev u32 [4n].  Asynchronous. */
evox_status evox_debug_philox(const uint32_t* ctr, uint32_t key0, uint32_t key1, uint32_t* out,
                              int64_t n, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* EVOX_H */
