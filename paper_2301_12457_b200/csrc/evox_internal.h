// evox_internal.h -- structures shared by the kernel TU and the C-ABI TU.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "evox_device.cuh"

namespace evox {

constexpr int kMaxPeers = 8;  // ranks reachable by the in-kernel peer exchange

// Device-resident control block of a handle.  Kernels read the generation
// index from here (not from launch parameters) so one captured CUDA graph can
// be replayed for any generation.
struct Ctl {
    unsigned long long gen_key;  // atomicMin accumulator of the running generation (~0 at rest)
    unsigned int ticket;         // CTAs finished in the running kernel (0 at rest)
    unsigned int err;            // 1: peer exchange timed out (checked by the host at sync)
    unsigned long long t;        // index of the current population
    float gf;                    // best-so-far fitness (PSO) / scratch
    unsigned int bar;            // k_pso_run_mid: grid barrier epoch (released per generation)
    long long gidx;              // global row of gbest (-1: none)
    float* hist;                 // hist[t] = min f of generation t
    unsigned long long* hkeys;   // CSO, world > 1: per-generation local min keys
    unsigned long long hist_cap;
    unsigned long long min_key;  // DE with peers: global min key of the current population
    unsigned int fin_cnt;        // k_pso_fin: CTAs that staged their slice (reset by CTA 0)
    unsigned int fin_epoch;      // k_pso_fin: t_new + 1 once CTA 0 has decided the exchange
    int fin_sel;                 // k_pso_fin: rank whose staged row becomes gbest (-1: none)
    unsigned int arrive;         // k_pso_run_mid (warp-row rows): monotonic arrival counter
    unsigned long long mkey[3];  // its per-generation minimum keys, slot t % 3 (~0 at rest)
};

// One rank's PSO state, as seen by kernels.
struct PsoArgs {
    float* X;
    float* V;
    float* P;
    float* f;
    float* pf;
    unsigned char* imp;  // pending pbest copy (lazy pbest)
    float* G;            // gbest row [ld]
    const float* lb;     // [ld] (used when !uniform_bounds)
    const float* ub;
    float lb0, ub0;
    int uniform_bounds;
    int pf_next;          // 1: L2 bulk prefetch of the warp's next short rows (mode A)
    long long rows, row0, D, ld;
    float w, phi_p, phi_g;
    float cp, cg;         // phi_p * 2^-24, phi_g * 2^-24 (exact; see scaled_u24)
    unsigned int k0, k1;  // Philox key = seed
    PhiloxKey rk;         // its key schedule
    Ctl* ctl;
    unsigned char* rec;   // world > 1: W winner records, stride rec_stride bytes
    long long rec_stride;
    int rank, world;
    int exchange;  // 1: publish the local winner record for the NCCL exchange (A13)
    int peer;      // 1: in-kernel peer-memory exchange through the mailboxes
    int fin_kernel;  // 1: the gbest publication / exchange runs in k_pso_fin after the kernel
    long long mb_slot;            // bytes per mailbox slot (16 + 4 ld, 16-aligned)
    unsigned long long peer_timeout_ns;
    unsigned char* mbox[kMaxPeers];  // every rank's mailbox (own included)
};

struct CsoArgs {
    float* X;
    float* V;
    float* f2[2];  // fitness by generation parity: read f2[t&1], write f2[(t+1)&1] (pairs
                   // straddling shards are decided by both owners from generation-t values)
    const float* lb;
    const float* ub;
    float lb0, ub0;
    int uniform_bounds;
    long long rows, row0, D, ld, pop;
    long long B;  // pairing block size
    float phi;
    float* xbar;               // [ld] column means (phi != 0)
    unsigned long long* limb;  // [2 x ld] fixed-point column-sum limbs (phi != 0, R-15)
    unsigned int k0, k1;
    PhiloxKey rk;
    Ctl* ctl;
    int rank, world;
    int exchange;  // 1: per-generation keys go to hkeys for one NCCL min-reduction per call
    // global pairing across shards (evox_cso_connect): pairing blocks may straddle
    // shards; every rank's X and f (own included) and the mailboxes of the
    // per-generation barrier + global minimum.  Not connected: one table entry
    // (our own shard).
    int peer, nsh;
    float* pX[kMaxPeers];
    float* pf[kMaxPeers][2];
    long long prow0[kMaxPeers + 1];
    unsigned char* mbox[kMaxPeers];
    unsigned long long* plimb[kMaxPeers];   // every rank's limbs (phi != 0)
    unsigned long long* pcflag[kMaxPeers];  // every rank's column-sum flags [world]
    unsigned long long peer_timeout_ns;
};

// DE/rand/1/bin (R-14).  The population lives in two buffers; sel[p][i] says
// which one holds row i at parity p = t & 1.  A trial is written into the
// other buffer and adopted by flipping sel[p^1][i] (no copy back).
struct DeArgs {
    float* buf[2];          // [rows x ld] each
    unsigned char* sel[2];  // [rows] per parity
    float* f[2];            // [rows] per parity
    const float* lb;
    const float* ub;
    float lb0, ub0;
    int uniform_bounds;
    long long rows, row0, D, ld, pop;
    float F, CR;
    unsigned int k0, k1;
    PhiloxKey rk;
    Ctl* ctl;
    // row sharding with cross-shard donors (evox_de_connect): every rank's
    // buffers and flags (own included; world == 1: just our own), the row
    // offsets of the shards, and the key-only mailboxes of the per-generation
    // barrier + global minimum
    int rank, world, peer;
    float* pbuf[kMaxPeers][2];
    unsigned char* psel[kMaxPeers][2];
    long long prow0[kMaxPeers + 1];
    unsigned char* mbox[kMaxPeers];
    unsigned long long peer_timeout_ns;
};

// Launch configuration is a function of dim only (R-11: bitwise identical
// results for every shard count and population size).

// ---- launchers (pso/cso/de/common_kernels.cu); all asynchronous on `st`.
cudaError_t launch_pso_init(const PsoArgs& a, cudaStream_t st);
cudaError_t launch_eval(int problem, const float* X, long long rows, long long D, long long ld,
                        float* fit, cudaStream_t st, bool no_htab = false);
// tma: the bulk-copy-staged variant (warp-per-row geometry only; EVOX_FLAG_TMA)
cudaError_t launch_pso_gen(int problem, const PsoArgs& a, int grid, cudaStream_t st, bool tma,
                           bool wave);
// k_pso_fin: gbest publication (+ key-first peer exchange) after a generation or tell kernel
// whose PsoArgs.fin_kernel is set; t_new < 0: the index ctl->t + 1.
cudaError_t launch_pso_fin(const PsoArgs& a, long long t_new, cudaStream_t st);
// Big populations take the wave grid (k_pso_gen_wave + k_pso_fin) unless no_wave.
bool pso_wave(int problem, long long ld, long long rows, int device);
// Mode-A next-row L2 prefetch of the PSO generation (PsoArgs.pf_next): a schedule choice
// measured per geometry and size, never a change of any result bit.
bool pso_prefetch_next(long long ld, long long rows);
cudaError_t launch_pso_move(const PsoArgs& a, unsigned long long t, cudaStream_t st);
cudaError_t launch_pso_tell(const PsoArgs& a, const float* fit, unsigned long long t,
                            cudaStream_t st);
cudaError_t launch_gbest_select(const PsoArgs& a, cudaStream_t st);
cudaError_t launch_pso_materialize(const PsoArgs& a, cudaStream_t st);
int pso_gen_grid(int problem, long long ld, long long rows, int device, bool wave);
// Tiny populations: all generations in one single-CTA launch (bitwise identical).
bool pso_small(long long rows, long long ld);
cudaError_t launch_pso_run_small(int problem, const PsoArgs& a, long long n, cudaStream_t st);
bool pso_mid(long long rows, long long ld);
cudaError_t launch_pso_run_mid(int problem, const PsoArgs& a, long long n, cudaStream_t st);

cudaError_t launch_cso_init(const CsoArgs& a, cudaStream_t st);
cudaError_t launch_cso_tell0(const CsoArgs& a, cudaStream_t st);
int cso_gen_grid(int problem, const CsoArgs& a, int device);
cudaError_t launch_cso_gen(int problem, const CsoArgs& a, int grid, cudaStream_t st);
cudaError_t launch_cso_colsum(const CsoArgs& a, double scale, cudaStream_t st);
cudaError_t launch_cso_colmean(const CsoArgs& a, double inv_scale, cudaStream_t st);
cudaError_t launch_cso_hist_from_keys(const CsoArgs& a, unsigned long long t0, long long n,
                                      cudaStream_t st);
// best(): the row of ctl->min_key into out (CSO: sel0 = sel1 = NULL).
cudaError_t launch_best_row(const Ctl* ctl, const float* X0, const float* X1,
                            const unsigned char* sel0, const unsigned char* sel1, long long row0,
                            long long rows, long long ld, float* out, cudaStream_t st);
cudaError_t launch_argmin_rows(const float* f, long long rows, long long row0,
                               unsigned long long* key_out, cudaStream_t st);

cudaError_t launch_de_init(const DeArgs& a, cudaStream_t st);
cudaError_t launch_de_tell0(const DeArgs& a, cudaStream_t st);
// no_flat: the row-walk kernel even for short rows (EVOX_FLAG_NO_WAVE; tests)
int de_gen_grid(int problem, long long ld, long long rows, int device, bool no_flat);
cudaError_t launch_de_gen(int problem, const DeArgs& a, int grid, cudaStream_t st, bool no_flat);
cudaError_t launch_de_materialize(const DeArgs& a, cudaStream_t st);
cudaError_t launch_de_gather(const DeArgs& a, float* dst, cudaStream_t st);

cudaError_t launch_debug_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                                long long n, cudaStream_t st);

}  // namespace evox
