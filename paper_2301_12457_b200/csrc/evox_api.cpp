// evox_api.cpp -- the C-ABI of include/evox.h: handles, validation, error
// reporting/poisoning, CUDA-graph replay of n generations, NCCL exchange.
#include "evox.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "evox_internal.h"
#include "nccl_dl.h"

using evox::Ctl;
using evox::CsoArgs;
using evox::PsoArgs;

namespace {

thread_local std::string t_err;

evox_status fail(evox_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return st;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
int64_t round4(int64_t d) { return (d + 3) / 4 * 4; }
constexpr int64_t MAX_LD = 0x7FFFFFFCll;  // ld <= 2^31 - 4: in-row quad / column indices fit int32

bool mul_ok(int64_t a, int64_t b, int64_t lim) { return a >= 0 && b >= 0 && (b == 0 || a <= lim / b); }

void shard(int64_t pop, int world, int rank, int64_t* row0, int64_t* rows) {
    const int64_t base = pop / world, rem = pop % world;
    *rows = base + (rank < rem ? 1 : 0);
    *row0 = (int64_t)rank * base + (rank < rem ? rank : rem);
}

// Common state of a handle (PSO and CSO).
struct Base {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t pop = 0, dim = 0, ld = 0, row0 = 0, rows = 0;
    int rank = 0, world = 1;
    uint64_t seed = 0;
    uint32_t flags = 0;                                    // evox_opts.flags (EVOX_FLAG_*)
    unsigned long long peer_timeout_ns = 60000000000ull;   // evox_opts.peer_timeout_ms
    std::vector<float> lb, ub;
    bool uniform = true;
    void* base = nullptr;
    bool own_base = false;
    size_t bytes = 0;
    float* lb_d = nullptr;
    float* ub_d = nullptr;
    Ctl* ctl = nullptr;
    float* hist = nullptr;
    unsigned long long* hkeys = nullptr;
    int64_t hist_cap = 0;
    int64_t t = -1;  // index of the current population (-1: not evaluated)
    bool stepped = false;  // a step/ask ran since init or the last load (connect must precede)
    bool min_key_stale = false;  // CSO/DE: ctl->min_key predates a load (best() recomputes)
    int problem = -1;
    bool poisoned = false;
    ncclComm_t comm = nullptr;
    std::map<std::pair<int, int64_t>, cudaGraphExec_t> graphs;
    unsigned long long* scratch_key = nullptr;  // one u64 for queries
    float* scratch_row = nullptr;               // [ld] for queries
    unsigned char* stage = nullptr;             // pinned host staging of best() (Ctl + row)
    size_t stage_bytes = 0;
    // kernel timing (evox_*_set_timing)
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending, ev_free;
    std::vector<int64_t> ev_gens;
    std::vector<int> ev_slot;    // 0: generation kernel, 1: gbest publication / exchange
    double kernel_ms = 0.0;
    int64_t kernel_n = 0;        // generations run by the timed launches
    int64_t kernel_launches = 0;
    double fin_ms = 0.0;         // k_pso_fin (gbest publication + key-first exchange)
    int64_t fin_launches = 0;
};

// Timed launch: events around the kernel enqueued by `launch`, which runs
// `gens` generations.
template <class F>
cudaError_t timed(Base* b, F launch, int64_t gens = 1, int slot = 0) {
    if (!b->timing) return launch();
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!b->ev_free.empty()) {
        ev = b->ev_free.back();
        b->ev_free.pop_back();
    } else {
        cudaError_t e = cudaEventCreate(&ev.first);
        if (e == cudaSuccess) e = cudaEventCreate(&ev.second);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ev.first, b->stream);
    if (e == cudaSuccess) e = launch();
    if (e == cudaSuccess) e = cudaEventRecord(ev.second, b->stream);
    b->ev_pending.push_back(ev);
    b->ev_gens.push_back(gens);
    b->ev_slot.push_back(slot);
    return e;
}

// After a stream sync: fold pending event pairs into the totals.
cudaError_t collect_timing(Base* b) {
    for (size_t i = 0; i < b->ev_pending.size(); ++i) {
        auto& ev = b->ev_pending[i];
        float ms = 0.0f;
        cudaError_t e = cudaEventElapsedTime(&ms, ev.first, ev.second);
        if (e != cudaSuccess) return e;
        if (b->ev_slot[i] == 1) {
            b->fin_ms += ms;
            b->fin_launches += 1;
        } else {
            b->kernel_ms += ms;
            b->kernel_n += b->ev_gens[i];
            b->kernel_launches += 1;
        }
        b->ev_free.push_back(ev);
    }
    b->ev_pending.clear();
    b->ev_gens.clear();
    b->ev_slot.clear();
    return cudaSuccess;
}

evox_status poison(Base* b, evox_status st, const char* what, cudaError_t e) {
    b->poisoned = true;
    return fail(st, "%s: %s", what, cudaGetErrorString(e));
}

#define CU(b, expr)                                                           \
    do {                                                                      \
        cudaError_t e_ = (expr);                                              \
        if (e_ != cudaSuccess) return poison((b), EVOX_ERR_CUDA, #expr, e_);  \
    } while (0)

#define NC(b, expr)                                                                   \
    do {                                                                              \
        ncclResult_t r_ = (expr);                                                     \
        if (r_ != ncclSuccess) {                                                      \
            (b)->poisoned = true;                                                     \
            return fail(EVOX_ERR_NCCL, "%s: %s", #expr,                               \
                        evox::nccl_api(nullptr)->GetErrorString(r_));                 \
        }                                                                             \
    } while (0)

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

evox_status check_bounds(int64_t dim, const float* lb, const float* ub) {
    if (!lb || !ub) return fail(EVOX_ERR_INVALID_ARGUMENT, "lb/ub must be non-NULL host arrays");
    for (int64_t j = 0; j < dim; ++j) {
        if (!std::isfinite(lb[j]) || !std::isfinite(ub[j]))
            return fail(EVOX_ERR_INVALID_ARGUMENT, "bounds must be finite (dim %lld)", (long long)j);
        if (!(lb[j] < ub[j]))
            return fail(EVOX_ERR_INVALID_ARGUMENT, "lb[%lld] must be < ub[%lld]", (long long)j,
                        (long long)j);
    }
    return EVOX_OK;
}

evox_status check_opts(const evox_opts* o, int* world, int* rank) {
    *world = 1;
    *rank = 0;
    if (!o) return EVOX_OK;
    *world = o->world <= 0 ? 1 : o->world;
    *rank = o->rank;
    if (*rank < 0 || *rank >= *world)
        return fail(EVOX_ERR_INVALID_ARGUMENT, "rank %d out of range for world %d", o->rank, *world);
    if (o->workspace && ((uintptr_t)o->workspace % kAlign))
        return fail(EVOX_ERR_INVALID_ARGUMENT, "workspace must be %zu-byte aligned", kAlign);
    return EVOX_OK;
}

// Common setup: device, stream, bounds copy, NCCL communicator.
evox_status base_setup(Base* b, int64_t pop, int64_t dim, const float* lb, const float* ub,
                       uint64_t seed, const evox_opts* o, int world, int rank) {
    b->pop = pop;
    b->dim = dim;
    b->ld = round4(dim);
    b->world = world;
    b->rank = rank;
    b->seed = seed;
    if (o) {
        b->flags = o->flags;
        if (o->peer_timeout_ms > 0)
            b->peer_timeout_ns = (unsigned long long)o->peer_timeout_ms * 1000000ull;
    }
    shard(pop, world, rank, &b->row0, &b->rows);
    b->lb.assign(b->ld, 0.0f);
    b->ub.assign(b->ld, 0.0f);
    for (int64_t j = 0; j < dim; ++j) {
        b->lb[j] = lb[j];
        b->ub[j] = ub[j];
        if (lb[j] != lb[0] || ub[j] != ub[0]) b->uniform = false;
    }
    int dev = -1;
    if (o && o->device >= 0) dev = o->device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return fail(EVOX_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    }
    b->device = dev;
    DevGuard g(dev);
    if (o && o->cuda_stream) {
        b->stream = (cudaStream_t)o->cuda_stream;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess)
            return fail(EVOX_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
        b->own_stream = true;
    }
    // EVOX_FLAG_FORCE_NCCL runs a single-GPU handle through the NCCL exchange path
    // (a 1-rank communicator) so the multi-GPU code is exercised on one GPU.
    const bool force = (b->flags & EVOX_FLAG_FORCE_NCCL) != 0;
    // world > 1 without a unique id: the caller will evox_pso_connect() the peers
    if ((world > 1 && o && o->nccl_id) || (world == 1 && force)) {
        const char* why = "";
        const evox::NcclApi* api = evox::nccl_api(&why);
        if (!api) return fail(EVOX_ERR_NCCL, "NCCL unavailable: %s", why);
        ncclUniqueId id;
        if (world > 1) {
            std::memcpy(&id, o->nccl_id, sizeof id);
        } else {
            ncclResult_t r = api->GetUniqueId(&id);
            if (r != ncclSuccess) return fail(EVOX_ERR_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
        }
        ncclResult_t r = api->CommInitRank(&b->comm, world, id, rank);
        if (r != ncclSuccess) {
            b->comm = nullptr;
            return fail(EVOX_ERR_NCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
        }
    }
    return EVOX_OK;
}

// Grow the device history to hold index `need - 1`.
evox_status ensure_hist(Base* b, int64_t need) {
    if (need <= b->hist_cap) return EVOX_OK;
    int64_t cap = b->hist_cap > 0 ? b->hist_cap : 1024;
    while (cap < need) cap *= 2;
    float* nh = nullptr;
    unsigned long long* nk = nullptr;
    CU(b, cudaMalloc(&nh, sizeof(float) * cap));
    CU(b, cudaMalloc(&nk, sizeof(unsigned long long) * cap));
    CU(b, cudaMemsetAsync(nh, 0, sizeof(float) * cap, b->stream));
    CU(b, cudaMemsetAsync(nk, 0xff, sizeof(unsigned long long) * cap, b->stream));
    if (b->hist) {
        CU(b, cudaMemcpyAsync(nh, b->hist, sizeof(float) * b->hist_cap, cudaMemcpyDeviceToDevice,
                              b->stream));
        CU(b, cudaMemcpyAsync(nk, b->hkeys, sizeof(unsigned long long) * b->hist_cap,
                              cudaMemcpyDeviceToDevice, b->stream));
    }
    Ctl tmp;
    tmp.hist = nh;
    tmp.hkeys = nk;
    tmp.hist_cap = (unsigned long long)cap;
    CU(b, cudaMemcpyAsync(&b->ctl->hist, &tmp.hist, sizeof(void*) * 2 + sizeof(unsigned long long),
                          cudaMemcpyHostToDevice, b->stream));
    CU(b, cudaStreamSynchronize(b->stream));  // old buffers no longer referenced
    if (b->hist) cudaFree(b->hist);
    if (b->hkeys) cudaFree(b->hkeys);
    b->hist = nh;
    b->hkeys = nk;
    b->hist_cap = cap;
    return EVOX_OK;
}

// staged: a host copy of the control block already enqueued on the stream (it is
// complete after the synchronisation), so the error flag needs no extra copy.
evox_status sync_check(Base* b, const Ctl* staged = nullptr) {
    DevGuard g(b->device);
    cudaError_t e = cudaStreamSynchronize(b->stream);
    if (e != cudaSuccess) return poison(b, EVOX_ERR_CUDA, "asynchronous CUDA error", e);
    if (b->ctl) {
        unsigned int err = 0;
        if (staged) {
            std::memcpy(&err, &staged->err, sizeof err);
        } else {
            e = cudaMemcpy(&err, &b->ctl->err, sizeof err, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return poison(b, EVOX_ERR_CUDA, "reading the control block", e);
        }
        if (err) {
            b->poisoned = true;
            return fail(EVOX_ERR_EXCHANGE,
                        "peer-memory exchange (or the persistent kernel's grid barrier) timed out");
        }
    }
    if (b->comm) {
        const evox::NcclApi* api = evox::nccl_api(nullptr);
        ncclResult_t ar = ncclSuccess;
        api->CommGetAsyncError(b->comm, &ar);
        if (ar != ncclSuccess) {
            b->poisoned = true;
            return fail(EVOX_ERR_NCCL, "asynchronous NCCL error: %s", api->GetErrorString(ar));
        }
    }
    return EVOX_OK;
}

void base_release(Base* b) {
    DevGuard g(b->device);
    if (b->stream) cudaStreamSynchronize(b->stream);
    for (auto& ev : b->ev_pending) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
    for (auto& ev : b->ev_free) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
    b->ev_pending.clear();
    b->ev_free.clear();
    b->ev_gens.clear();
    for (auto& kv : b->graphs) cudaGraphExecDestroy(kv.second);
    b->graphs.clear();
    if (b->comm) {
        const evox::NcclApi* api = evox::nccl_api(nullptr);
        if (b->poisoned) api->CommAbort(b->comm); else api->CommDestroy(b->comm);
        b->comm = nullptr;
    }
    if (b->hist) cudaFree(b->hist);
    if (b->hkeys) cudaFree(b->hkeys);
    if (b->scratch_key) cudaFree(b->scratch_key);
    if (b->scratch_row) cudaFree(b->scratch_row);
    if (b->stage) cudaFreeHost(b->stage);
    if (b->own_base && b->base) cudaFree(b->base);
    if (b->own_stream && b->stream) cudaStreamDestroy(b->stream);
    cudaGetLastError();
}

// Layout helper: carves 256-byte-aligned slices.
struct Carver {
    size_t off = 0;
    std::vector<std::pair<void**, size_t>> slots;
    template <class T>
    void add(T** p, size_t bytes) {
        slots.push_back({reinterpret_cast<void**>(p), off});
        off += align_up(bytes ? bytes : 1);
    }
    void assign(void* base) {
        for (auto& s : slots) *s.first = static_cast<char*>(base) + s.second;
    }
};

evox_status base_alloc(Base* b, Carver& c, const evox_opts* o) {
    DevGuard g(b->device);
    b->bytes = c.off;
    if (o && o->workspace) {
        if (o->workspace_bytes < c.off)
            return fail(EVOX_ERR_OUT_OF_MEMORY, "workspace too small: %zu < %zu bytes",
                        o->workspace_bytes, c.off);
        b->base = o->workspace;
    } else {
        cudaError_t e = cudaMalloc(&b->base, c.off);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(EVOX_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu): %s", c.off, cudaGetErrorString(e));
        }
        b->own_base = true;
    }
    c.assign(b->base);
    return EVOX_OK;
}

evox_status base_common_init(Base* b) {
    DevGuard g(b->device);
    CU(b, cudaMemcpyAsync(b->lb_d, b->lb.data(), sizeof(float) * b->ld, cudaMemcpyHostToDevice,
                          b->stream));
    CU(b, cudaMemcpyAsync(b->ub_d, b->ub.data(), sizeof(float) * b->ld, cudaMemcpyHostToDevice,
                          b->stream));
    Ctl c;
    std::memset(&c, 0, sizeof c);
    c.gen_key = ~0ull;
    c.mkey[0] = c.mkey[1] = c.mkey[2] = ~0ull;
    c.ticket = 0;
    c.t = 0;
    c.gf = INFINITY;
    c.gidx = -1;
    CU(b, cudaMemcpyAsync(b->ctl, &c, sizeof c, cudaMemcpyHostToDevice, b->stream));
    CU(b, cudaMalloc(&b->scratch_key, sizeof(unsigned long long)));
    CU(b, cudaMalloc(&b->scratch_row, sizeof(float) * b->ld));
    evox_status st = ensure_hist(b, 1024);
    if (st != EVOX_OK) return st;
    CU(b, cudaStreamSynchronize(b->stream));  // host staging of lb/ub/ctl complete
    return EVOX_OK;
}

bool valid_problem(int p) { return p >= EVOX_SPHERE && p <= EVOX_ROSENBROCK; }

evox_status ensure_stage(Base* b, size_t need) {
    if (b->stage_bytes >= need) return EVOX_OK;
    if (b->stage) cudaFreeHost(b->stage);
    b->stage = nullptr;
    b->stage_bytes = 0;
    CU(b, cudaHostAlloc((void**)&b->stage, need, cudaHostAllocDefault));
    b->stage_bytes = need;
    return EVOX_OK;
}

void decode_key(unsigned long long key, float* fv, int64_t* gi) {
    *fv = INFINITY;
    *gi = -1;
    if (key != ~0ull) {
        const uint32_t o = (uint32_t)(key >> 32);
        const uint32_t bits = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
        std::memcpy(fv, &bits, 4);
        *gi = (int64_t)(uint32_t)(key & 0xffffffffu);
    }
}

// best() of a single-rank CSO / DE handle: the generation kernel's finalize already left the
// population's minimum key in ctl->min_key; one tiny row-gather kernel, two async D2H copies
// into pinned staging and ONE synchronisation (no population-wide argmin).
evox_status staged_best(Base* b, const float* X0, const float* X1, const unsigned char* sel0,
                        const unsigned char* sel1, float* fit, int64_t* global_index,
                        float* row_host) {
    const size_t row_bytes = sizeof(float) * (size_t)b->dim;
    evox_status st = ensure_stage(b, sizeof(Ctl) + sizeof(float) * (size_t)b->ld);
    if (st != EVOX_OK) return st;
    if (row_host)
        CU(b, evox::launch_best_row(b->ctl, X0, X1, sel0, sel1, b->row0, b->rows, b->ld,
                                    b->scratch_row, b->stream));
    CU(b, cudaMemcpyAsync(b->stage, b->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, b->stream));
    if (row_host)
        CU(b, cudaMemcpyAsync(b->stage + sizeof(Ctl), b->scratch_row, row_bytes,
                              cudaMemcpyDeviceToHost, b->stream));
    st = sync_check(b, reinterpret_cast<const Ctl*>(b->stage));
    if (st != EVOX_OK) return st;
    Ctl c;
    std::memcpy(&c, b->stage, sizeof c);
    float fv;
    int64_t gi;
    decode_key(c.min_key, &fv, &gi);
    if (fit) *fit = fv;
    if (global_index) *global_index = gi;
    if (row_host && gi >= 0) std::memcpy(row_host, b->stage + sizeof(Ctl), row_bytes);
    return EVOX_OK;
}

// Replay `n` generations of `one` (a callable that enqueues one generation)
// through cached CUDA graphs of up to kChunk generations.
constexpr int64_t kChunk = 32;

template <class F>
evox_status run_graphed(Base* b, int problem, int64_t n, F one) {
    const bool no_graph = (b->flags & EVOX_FLAG_NO_GRAPH) != 0;
    if (no_graph || b->timing) {
        for (int64_t i = 0; i < n; ++i) {
            evox_status st = one();
            if (st != EVOX_OK) return st;
        }
        return EVOX_OK;
    }
    while (n > 0) {
        const int64_t c = n >= kChunk ? kChunk : n;
        auto key = std::make_pair(problem, c);
        auto it = b->graphs.find(key);
        if (it == b->graphs.end()) {
            cudaGraph_t graph = nullptr;
            CU(b, cudaStreamBeginCapture(b->stream, cudaStreamCaptureModeThreadLocal));
            evox_status st = EVOX_OK;
            for (int64_t i = 0; i < c && st == EVOX_OK; ++i) st = one();
            cudaError_t e = cudaStreamEndCapture(b->stream, &graph);
            if (st != EVOX_OK) {
                if (graph) cudaGraphDestroy(graph);
                return st;
            }
            if (e != cudaSuccess) return poison(b, EVOX_ERR_CUDA, "cudaStreamEndCapture", e);
            cudaGraphExec_t exec = nullptr;
            e = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) return poison(b, EVOX_ERR_CUDA, "cudaGraphInstantiate", e);
            it = b->graphs.emplace(key, exec).first;
        }
        CU(b, cudaGraphLaunch(it->second, b->stream));
        n -= c;
    }
    return EVOX_OK;
}

}  // namespace

// ============================================================== PSO handle
struct evox_pso : Base {
    float w = 0, phi_p = 0, phi_g = 0;
    float *X = nullptr, *V = nullptr, *P = nullptr, *f = nullptr, *pf = nullptr, *G = nullptr;
    unsigned char* imp = nullptr;
    unsigned char* rec = nullptr;
    int64_t rec_stride = 0;
    int gen_grid[5] = {0, 0, 0, 0, 0};
    bool wave[5] = {false, false, false, false, false};  // per problem: the wave grid
                                                         // (k_pso_gen_wave + k_pso_fin)
    // in-kernel peer exchange (evox_pso_connect)
    unsigned char* mbox = nullptr;  // own mailbox (separate cudaMalloc: IPC-exportable)
    size_t mb_bytes = 0;
    int64_t mb_slot = 0;
    bool peer = false;
    unsigned char* peers[evox::kMaxPeers] = {};
    std::vector<void*> ipc_opened;
    bool asked = false;   // ask issued, tell pending
    int64_t ask_t = 0;    // population index the pending tell refers to
    // t right after the last cooperative launch: its per-generation key slots (Ctl::mkey) are
    // clean for a launch starting there; any other t (another path advanced the population,
    // or a load) re-initialises them first
    int64_t mid_t = -2;
    PsoArgs args() const {
        PsoArgs a;
        std::memset(&a, 0, sizeof a);
        a.X = X; a.V = V; a.P = P; a.f = f; a.pf = pf; a.imp = imp; a.G = G;
        a.lb = lb_d; a.ub = ub_d;
        a.lb0 = lb[0]; a.ub0 = ub[0];
        a.uniform_bounds = uniform ? 1 : 0;
        a.pf_next = evox::pso_prefetch_next(ld, rows) ? 1 : 0;
        a.rows = rows; a.row0 = row0; a.D = dim; a.ld = ld;
        a.w = w; a.phi_p = phi_p; a.phi_g = phi_g;
        a.cp = phi_p * 0x1p-24f;
        a.cg = phi_g * 0x1p-24f;
        a.k0 = (unsigned)(seed & 0xffffffffu);
        a.k1 = (unsigned)(seed >> 32);
        a.rk = evox::Philox::schedule(seed);
        a.ctl = ctl;
        a.rec = rec;
        a.rec_stride = rec_stride;
        a.rank = rank;
        a.world = world;
        a.exchange = comm != nullptr && !peer;
        a.peer = peer ? 1 : 0;
        a.fin_kernel = peer ? 1 : 0;  // | wave[problem], set by the step
        a.mb_slot = mb_slot;
        a.peer_timeout_ns = peer_timeout_ns;
        for (int r = 0; r < evox::kMaxPeers; ++r) a.mbox[r] = peers[r];
        return a;
    }
};

namespace {

bool pso_use_wave(const evox_pso* s, int problem) {
    return !(s->flags & EVOX_FLAG_NO_WAVE) && evox::pso_wave(problem, s->ld, s->rows, s->device);
}

void pso_layout(evox_pso* s, Carver& c) {
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    c.add(&s->X, mat);
    c.add(&s->V, mat);
    c.add(&s->P, mat);
    c.add(&s->f, sizeof(float) * s->rows);
    c.add(&s->pf, sizeof(float) * s->rows);
    c.add(&s->imp, s->rows);
    c.add(&s->G, sizeof(float) * s->ld);
    c.add(&s->lb_d, sizeof(float) * s->ld);
    c.add(&s->ub_d, sizeof(float) * s->ld);
    c.add(&s->ctl, sizeof(Ctl));
    s->rec_stride = (16 + 4 * s->ld + 15) / 16 * 16;
    c.add(&s->rec, (size_t)s->rec_stride * s->world);
}

evox_status check_pso(evox_pso* s) {
    if (!s) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL handle");
    if (s->poisoned) return fail(EVOX_ERR_POISONED, "handle poisoned by an earlier CUDA/NCCL error");
    return EVOX_OK;
}

// world > 1: all-gather of the W winner records, then the strict gbest select.
evox_status pso_exchange(evox_pso* s) {
    if (s->peer || !s->comm) return EVOX_OK;  // peer mode: done inside the kernel
    const evox::NcclApi* api = evox::nccl_api(nullptr);
    NC(s, api->AllGather(s->rec + (int64_t)s->rank * s->rec_stride, s->rec, (size_t)s->rec_stride,
                         ncclUint8, s->comm, s->stream));
    CU(s, evox::launch_gbest_select(s->args(), s->stream));
    return EVOX_OK;
}

evox_status check_connected(evox_pso* s) {
    if (s->world > 1 && !s->comm && !s->peer)
        return fail(EVOX_ERR_CONTRACT,
                    "world > 1: pass opts.nccl_id at init or call evox_pso_connect first");
    return EVOX_OK;
}

evox_status pso_first_eval(evox_pso* s, int problem) {
    PsoArgs a = s->args();
    CU(s, evox::launch_eval(problem, s->X, s->rows, s->dim, s->ld, s->f, s->stream));
    CU(s, evox::launch_pso_tell(a, s->f, 0, s->stream));
    evox_status st = pso_exchange(s);
    if (st != EVOX_OK) return st;
    s->t = 0;
    return EVOX_OK;
}

}  // namespace

extern "C" {

const char* evox_last_error(void) { return t_err.c_str(); }
const char* evox_version(void) { return "evox-b200 1.0 (sm_100a)"; }
int evox_abi_version(void) { return EVOX_ABI_VERSION; }

evox_status evox_shard_rows(int64_t pop, int world, int rank, int64_t* row0, int64_t* rows) {
    if (!row0 || !rows) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output pointer");
    if (pop < 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "pop must be >= 0");
    if (world < 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "world must be >= 1");
    if (rank < 0 || rank >= world) return fail(EVOX_ERR_INVALID_ARGUMENT, "rank out of range");
    shard(pop, world, rank, row0, rows);
    return EVOX_OK;
}

evox_status evox_nccl_unique_id(uint8_t out[128]) {
    if (!out) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    const char* why = "";
    const evox::NcclApi* api = evox::nccl_api(&why);
    if (!api) return fail(EVOX_ERR_NCCL, "NCCL unavailable: %s", why);
    ncclUniqueId id;
    ncclResult_t r = api->GetUniqueId(&id);
    if (r != ncclSuccess) return fail(EVOX_ERR_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return EVOX_OK;
}

evox_status evox_eval_ex(evox_problem problem, const float* X, int64_t pop, int64_t dim,
                         int64_t ld, float* fit, void* cuda_stream, uint32_t flags) {
    if (!valid_problem(problem)) return fail(EVOX_ERR_INVALID_ARGUMENT, "unknown problem %d", (int)problem);
    if (pop < 0 || dim < 1) return fail(EVOX_ERR_SHAPE, "need pop >= 0 and dim >= 1");
    if (ld < dim || ld % 4) return fail(EVOX_ERR_SHAPE, "ld must be >= dim and a multiple of 4");
    if (ld > MAX_LD) return fail(EVOX_ERR_SHAPE, "ld must be <= 2^31 - 4 (in-row indices are 32-bit)");
    if (!mul_ok(pop, ld, INT64_MAX / 4)) return fail(EVOX_ERR_SHAPE, "pop*ld overflows");
    if (pop == 0) return EVOX_OK;
    if (!X || !fit) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL X or fit");
    if ((uintptr_t)X % 16) return fail(EVOX_ERR_INVALID_ARGUMENT, "X must be 16-byte aligned");
    cudaError_t e = evox::launch_eval((int)problem, X, pop, dim, ld, fit, (cudaStream_t)cuda_stream,
                                      (flags & EVOX_EVAL_NO_HTAB) != 0);
    if (e != cudaSuccess) return fail(EVOX_ERR_CUDA, "evox_eval launch: %s", cudaGetErrorString(e));
    return EVOX_OK;
}

evox_status evox_eval(evox_problem problem, const float* X, int64_t pop, int64_t dim, int64_t ld,
                      float* fit, void* cuda_stream) {
    return evox_eval_ex(problem, X, pop, dim, ld, fit, cuda_stream, 0u);
}

evox_status evox_pso_workspace_bytes(int64_t pop, int64_t dim, int world, int rank, size_t* bytes) {
    if (!bytes) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    if (pop < 1 || dim < 1) return fail(EVOX_ERR_SHAPE, "need pop >= 1 and dim >= 1");
    if (world < 1) world = 1;
    if (rank < 0 || rank >= world) return fail(EVOX_ERR_INVALID_ARGUMENT, "rank out of range");
    evox_pso s;
    s.world = world;
    s.rank = rank;
    s.ld = round4(dim);
    shard(pop, world, rank, &s.row0, &s.rows);
    if (!mul_ok(s.rows, s.ld, INT64_MAX / 64)) return fail(EVOX_ERR_SHAPE, "pop*dim overflows");
    Carver c;
    pso_layout(&s, c);
    *bytes = c.off;
    return EVOX_OK;
}

evox_status evox_pso_init(int64_t pop, int64_t dim, const float* lb, const float* ub, float w,
                          float phi_p, float phi_g, uint64_t seed, const evox_opts* opts,
                          evox_pso** out) {
    if (!out) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output handle pointer");
    *out = nullptr;
    if (pop < 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "pop must be >= 1 (got %lld)", (long long)pop);
    if (dim < 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "dim must be >= 1 (got %lld)", (long long)dim);
    if (pop > 0xFFFFFFFFll) return fail(EVOX_ERR_SHAPE, "pop must be < 2^32 (Philox row counter)");
    if (round4(dim) > MAX_LD) return fail(EVOX_ERR_SHAPE, "dim must be <= 2^31 - 4 (in-row indices are 32-bit)");
    if (!mul_ok(pop, round4(dim), INT64_MAX / 64)) return fail(EVOX_ERR_SHAPE, "pop*dim overflows");
    if (!std::isfinite(w) || !std::isfinite(phi_p) || !std::isfinite(phi_g))
        return fail(EVOX_ERR_INVALID_ARGUMENT, "w, phi_p, phi_g must be finite");
    // the kernels fold phi * 2^-24 into one multiply; that is exact iff the
    // scaled value is 0 or a normal float
    for (float ph : {phi_p, phi_g}) {
        const float sc = ph * 0x1p-24f;
        if (ph != 0.0f && (std::fabs(sc) < 0x1p-126f || (double)sc != (double)ph * 0x1p-24))
            return fail(EVOX_ERR_INVALID_ARGUMENT, "|phi_p|, |phi_g| must be 0 or >= 2^-102");
    }
    evox_status st = check_bounds(dim, lb, ub);
    if (st != EVOX_OK) return st;
    int world, rank;
    st = check_opts(opts, &world, &rank);
    if (st != EVOX_OK) return st;
    if (world > 1 && pop < world) return fail(EVOX_ERR_CONFIG, "pop (%lld) < world (%d)", (long long)pop, world);

    evox_pso* s = new (std::nothrow) evox_pso;
    if (!s) return fail(EVOX_ERR_OUT_OF_MEMORY, "host allocation failed");
    s->w = w;
    s->phi_p = phi_p;
    s->phi_g = phi_g;
    st = base_setup(s, pop, dim, lb, ub, seed, opts, world, rank);
    if (st == EVOX_OK) {
        Carver c;
        pso_layout(s, c);
        st = base_alloc(s, c, opts);
    }
    if (st == EVOX_OK) st = base_common_init(s);
    if (st == EVOX_OK) {
        DevGuard g(s->device);
        cudaError_t e = evox::launch_pso_init(s->args(), s->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(s->G, 0, sizeof(float) * s->ld, s->stream);
        if (e == cudaSuccess && s->world <= evox::kMaxPeers) {
            // the mailbox of the in-kernel peer exchange (own allocation: IPC-exportable)
            s->mb_slot = (16 + 4 * s->ld + 15) / 16 * 16;
            s->mb_bytes = (size_t)(2 * s->world * s->mb_slot);
            e = cudaMalloc(&s->mbox, s->mb_bytes);
            if (e == cudaSuccess) e = cudaMemsetAsync(s->mbox, 0, s->mb_bytes, s->stream);
        }
        if (e != cudaSuccess) st = poison(s, EVOX_ERR_CUDA, "pso init", e);
        for (int p = 0; p < 5 && st == EVOX_OK; ++p) {
            s->wave[p] = pso_use_wave(s, p);
            s->gen_grid[p] = evox::pso_gen_grid(p, s->ld, s->rows, s->device, s->wave[p]);
        }
    }
    if (st != EVOX_OK) {
        std::string keep = t_err;
        base_release(s);
        delete s;
        t_err = keep;
        return st;
    }
    *out = s;
    return EVOX_OK;
}

evox_status evox_pso_step(evox_pso* s, evox_problem problem, int64_t n_gens) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!valid_problem(problem)) return fail(EVOX_ERR_INVALID_ARGUMENT, "unknown problem %d", (int)problem);
    if (n_gens < 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "n_gens must be >= 0");
    if (s->asked) return fail(EVOX_ERR_CONTRACT, "step after ask: tell the pending population first");
    st = check_connected(s);
    if (st != EVOX_OK) return st;
    if (s->problem >= 0 && s->problem != (int)problem)
        return fail(EVOX_ERR_CONTRACT, "handle is bound to problem %d (got %d)", s->problem, (int)problem);
    if (n_gens > (int64_t)0xFFFFFFFFll - 2 - s->t)
        return fail(EVOX_ERR_SHAPE, "generation counter would exceed 2^32");
    s->stepped = true;
    DevGuard g(s->device);
    st = ensure_hist(s, (s->t < 0 ? 0 : s->t) + n_gens + 1);
    if (st != EVOX_OK) return st;
    s->problem = (int)problem;
    if (s->t < 0) {
        st = pso_first_eval(s, (int)problem);
        if (st != EVOX_OK) return st;
    }
    if (n_gens == 0) return EVOX_OK;
    PsoArgs a = s->args();
    if (s->wave[problem]) a.fin_kernel = 1;  // the wave grid publishes gbest in k_pso_fin
    const int grid = s->gen_grid[problem];
    const bool no_small = (s->flags & EVOX_FLAG_NO_SMALL) != 0;  // testing: force multi-CTA
    if (!s->comm && !s->peer && !no_small && evox::pso_small(s->rows, s->ld)) {
        CU(s, timed(s, [&] { return evox::launch_pso_run_small((int)problem, a, n_gens, s->stream); },
                    n_gens));
        s->t += n_gens;
        return EVOX_OK;
    }
    // EVOX_FLAG_NO_MID: per-generation launches at every size (testing / A-B timing)
    const bool no_mid = (s->flags & EVOX_FLAG_NO_MID) != 0;
    if (!s->comm && !s->peer && !no_mid && !no_small && evox::pso_mid(s->rows, s->ld)) {
        if (s->mid_t != s->t)
            CU(s, cudaMemsetAsync(&s->ctl->mkey, 0xff, sizeof(s->ctl->mkey), s->stream));
        CU(s, timed(s, [&] { return evox::launch_pso_run_mid((int)problem, a, n_gens, s->stream); },
                    n_gens));
        s->t += n_gens;
        s->mid_t = s->t;
        return EVOX_OK;
    }
    st = run_graphed(s, (int)problem, n_gens, [&]() -> evox_status {
        CU(s, timed(s, [&] { return evox::launch_pso_gen((int)problem, a, grid, s->stream,
                                                      (s->flags & EVOX_FLAG_TMA) != 0,
                                                      s->wave[problem]); }));
        if (a.fin_kernel)
            CU(s, timed(s, [&] { return evox::launch_pso_fin(a, -1, s->stream); }, 0, 1));
        return pso_exchange(s);
    });
    if (st != EVOX_OK) return st;
    s->t += n_gens;
    return EVOX_OK;
}

evox_status evox_pso_ask(evox_pso* s, const float** X_dev, int64_t* rows, int64_t* ld) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!X_dev) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL X_dev");
    if (s->asked) return fail(EVOX_ERR_CONTRACT, "ask twice without tell");
    st = check_connected(s);
    if (st != EVOX_OK) return st;
    s->stepped = true;
    DevGuard g(s->device);
    if (s->t < 0) {
        s->ask_t = 0;  // first ask: X0, unmoved
    } else {
        st = ensure_hist(s, s->t + 2);
        if (st != EVOX_OK) return st;
        CU(s, evox::launch_pso_move(s->args(), (unsigned long long)s->t, s->stream));
        s->ask_t = s->t + 1;
    }
    s->asked = true;
    *X_dev = s->X;
    if (rows) *rows = s->rows;
    if (ld) *ld = s->ld;
    return EVOX_OK;
}

evox_status evox_pso_tell(evox_pso* s, const float* fit_dev) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!fit_dev) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL fitness");
    if (!s->asked) return fail(EVOX_ERR_CONTRACT, "tell without a preceding ask (S:317)");
    DevGuard g(s->device);
    st = ensure_hist(s, s->ask_t + 1);
    if (st != EVOX_OK) return st;
    CU(s, evox::launch_pso_tell(s->args(), fit_dev, (unsigned long long)s->ask_t, s->stream));
    st = pso_exchange(s);
    if (st != EVOX_OK) return st;
    s->t = s->ask_t;
    s->asked = false;
    return EVOX_OK;
}

evox_status evox_pso_sync(evox_pso* s) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    return sync_check(s);
}

// best() on a per-step path: the control block and the gbest row come back in ONE
// stream-ordered copy pair into pinned staging and one synchronisation (instead of a
// stream sync plus three blocking pageable copies), then the usual error checks.
evox_status evox_pso_best(evox_pso* s, float* fit, int64_t* global_index, float* row_host) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    const size_t row_bytes = sizeof(float) * (size_t)s->dim;
    st = ensure_stage(s, sizeof(Ctl) + row_bytes);
    if (st != EVOX_OK) return st;
    CU(s, cudaMemcpyAsync(s->stage, s->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s->stream));
    if (row_host)
        CU(s, cudaMemcpyAsync(s->stage + sizeof(Ctl), s->G, row_bytes, cudaMemcpyDeviceToHost,
                              s->stream));
    // stream sync + asynchronous-error / exchange-timeout checks (err from the staged copy)
    st = sync_check(s, reinterpret_cast<const Ctl*>(s->stage));
    if (st != EVOX_OK) return st;
    Ctl c;
    std::memcpy(&c, s->stage, sizeof c);
    if (fit) *fit = c.gf;
    if (global_index) *global_index = c.gidx;
    if (row_host) std::memcpy(row_host, s->stage + sizeof(Ctl), row_bytes);
    return EVOX_OK;
}

evox_status evox_pso_history(evox_pso* s, float* best_per_gen, int64_t cap, int64_t* n) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (cap < 0 || (cap > 0 && !best_per_gen)) return fail(EVOX_ERR_INVALID_ARGUMENT, "bad buffer");
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    const int64_t T = s->t + 1;
    if (n) *n = T;
    const int64_t k = T < cap ? T : cap;
    DevGuard g(s->device);
    if (k > 0) CU(s, cudaMemcpy(best_per_gen, s->hist, sizeof(float) * k, cudaMemcpyDeviceToHost));
    return EVOX_OK;
}

evox_status evox_pso_view(evox_pso* s, int field, void** dev, int64_t* rows, int64_t* ld) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!dev) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    DevGuard g(s->device);
    int64_t r = s->rows, l = s->ld;
    switch (field) {
        case EVOX_FIELD_X: *dev = s->X; break;
        case EVOX_FIELD_V: *dev = s->V; break;
        case EVOX_FIELD_P:
            CU(s, evox::launch_pso_materialize(s->args(), s->stream));
            *dev = s->P;
            break;
        case EVOX_FIELD_F: *dev = s->f; l = 1; break;
        case EVOX_FIELD_PF: *dev = s->pf; l = 1; break;
        case EVOX_FIELD_G: *dev = s->G; r = 1; break;
        default: return fail(EVOX_ERR_INVALID_ARGUMENT, "unknown field %d", field);
    }
    if (rows) *rows = r;
    if (ld) *ld = l;
    return sync_check(s);
}

evox_status evox_pso_info(evox_pso* s, int64_t* pop, int64_t* dim, int64_t* ld, int64_t* row0,
                          int64_t* rows, int64_t* t, void** cuda_stream) {
    if (!s) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL handle");
    if (pop) *pop = s->pop;
    if (dim) *dim = s->dim;
    if (ld) *ld = s->ld;
    if (row0) *row0 = s->row0;
    if (rows) *rows = s->rows;
    if (t) *t = s->t;
    if (cuda_stream) *cuda_stream = s->stream;
    return s->poisoned ? fail(EVOX_ERR_POISONED, "handle poisoned") : EVOX_OK;
}

// Blob: header | X | V | P | f | pf | imp | G | hist[0..t]
namespace {
struct BlobHdr {
    char magic[8];
    int64_t kind, pop, dim, ld, row0, rows, t, problem, asked, ask_t, world, rank;
    uint64_t seed;
    float w, phi_p, phi_g, gf;
    int64_t gidx;
    int64_t B;
};
}  // namespace

evox_status evox_pso_save(evox_pso* s, void* host_blob, size_t cap, size_t* used) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!used) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL used");
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    const int64_t T = s->t + 1;
    const size_t need = sizeof(BlobHdr) + 3 * mat + 8 * (size_t)s->rows + (size_t)s->rows +
                        4 * (size_t)s->ld + 4 * (size_t)(T > 0 ? T : 0);
    *used = need;
    if (!host_blob) return EVOX_OK;
    if (cap < need) return fail(EVOX_ERR_INVALID_ARGUMENT, "blob buffer too small (%zu < %zu)", cap, need);
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    Ctl c;
    CU(s, cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost));
    BlobHdr h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, "EVOXPSO1", 8);
    h.kind = 0; h.pop = s->pop; h.dim = s->dim; h.ld = s->ld; h.row0 = s->row0; h.rows = s->rows;
    h.t = s->t; h.problem = s->problem; h.asked = s->asked; h.ask_t = s->ask_t;
    h.world = s->world; h.rank = s->rank; h.seed = s->seed;
    h.w = s->w; h.phi_p = s->phi_p; h.phi_g = s->phi_g; h.gf = c.gf; h.gidx = c.gidx;
    char* p = static_cast<char*>(host_blob);
    std::memcpy(p, &h, sizeof h);
    p += sizeof h;
    CU(s, cudaMemcpy(p, s->X, mat, cudaMemcpyDeviceToHost)); p += mat;
    CU(s, cudaMemcpy(p, s->V, mat, cudaMemcpyDeviceToHost)); p += mat;
    CU(s, cudaMemcpy(p, s->P, mat, cudaMemcpyDeviceToHost)); p += mat;
    CU(s, cudaMemcpy(p, s->f, 4 * s->rows, cudaMemcpyDeviceToHost)); p += 4 * s->rows;
    CU(s, cudaMemcpy(p, s->pf, 4 * s->rows, cudaMemcpyDeviceToHost)); p += 4 * s->rows;
    CU(s, cudaMemcpy(p, s->imp, s->rows, cudaMemcpyDeviceToHost)); p += s->rows;
    CU(s, cudaMemcpy(p, s->G, 4 * s->ld, cudaMemcpyDeviceToHost)); p += 4 * s->ld;
    if (T > 0) CU(s, cudaMemcpy(p, s->hist, 4 * T, cudaMemcpyDeviceToHost));
    return EVOX_OK;
}

evox_status evox_pso_load(evox_pso* s, const void* host_blob, size_t size) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (s->peer)
        return fail(EVOX_ERR_CONTRACT,
                    "load on a peer-connected handle: load every rank's blob, then connect");
    if (!host_blob || size < sizeof(BlobHdr)) return fail(EVOX_ERR_INVALID_ARGUMENT, "bad blob");
    BlobHdr h;
    std::memcpy(&h, host_blob, sizeof h);
    if (std::memcmp(h.magic, "EVOXPSO1", 8) != 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "not a PSO blob");
    if (h.pop != s->pop || h.dim != s->dim || h.ld != s->ld || h.row0 != s->row0 ||
        h.rows != s->rows || h.world != s->world || h.rank != s->rank)
        return fail(EVOX_ERR_SHAPE, "blob shape/shard does not match the handle");
    if (h.seed != s->seed || h.w != s->w || h.phi_p != s->phi_p || h.phi_g != s->phi_g)
        return fail(EVOX_ERR_CONTRACT, "blob parameters (seed/w/phi) differ from the handle's");
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    const int64_t T = h.t + 1;
    const size_t need = sizeof(BlobHdr) + 3 * mat + 9 * (size_t)s->rows + 4 * (size_t)s->ld +
                        4 * (size_t)(T > 0 ? T : 0);
    if (size < need) return fail(EVOX_ERR_SHAPE, "blob truncated (%zu < %zu)", size, need);
    DevGuard g(s->device);
    st = ensure_hist(s, (T > 0 ? T : 0) + 1);
    if (st != EVOX_OK) return st;
    CU(s, cudaStreamSynchronize(s->stream));
    const char* p = static_cast<const char*>(host_blob) + sizeof h;
    CU(s, cudaMemcpy(s->X, p, mat, cudaMemcpyHostToDevice)); p += mat;
    CU(s, cudaMemcpy(s->V, p, mat, cudaMemcpyHostToDevice)); p += mat;
    CU(s, cudaMemcpy(s->P, p, mat, cudaMemcpyHostToDevice)); p += mat;
    CU(s, cudaMemcpy(s->f, p, 4 * s->rows, cudaMemcpyHostToDevice)); p += 4 * s->rows;
    CU(s, cudaMemcpy(s->pf, p, 4 * s->rows, cudaMemcpyHostToDevice)); p += 4 * s->rows;
    CU(s, cudaMemcpy(s->imp, p, s->rows, cudaMemcpyHostToDevice)); p += s->rows;
    CU(s, cudaMemcpy(s->G, p, 4 * s->ld, cudaMemcpyHostToDevice)); p += 4 * s->ld;
    if (T > 0) CU(s, cudaMemcpy(s->hist, p, 4 * T, cudaMemcpyHostToDevice));
    Ctl c;
    CU(s, cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost));
    c.gen_key = ~0ull;
    c.mkey[0] = c.mkey[1] = c.mkey[2] = ~0ull;
    c.ticket = 0;
    c.t = h.t < 0 ? 0 : (unsigned long long)h.t;
    c.gf = h.gf;
    c.gidx = h.gidx;
    CU(s, cudaMemcpy(s->ctl, &c, sizeof c, cudaMemcpyHostToDevice));
    s->t = h.t;
    s->mid_t = -2;
    s->problem = (int)h.problem;
    s->asked = h.asked != 0;
    s->ask_t = h.ask_t;
    s->stepped = false;
    if (s->mbox) CU(s, cudaMemset(s->mbox, 0, s->mb_bytes));  // no stale exchange flags
    return EVOX_OK;
}

evox_status evox_pso_mailbox(evox_pso* s, void** dev, size_t* bytes) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!s->mbox) return fail(EVOX_ERR_CONFIG, "no mailbox (world > %d)", evox::kMaxPeers);
    if (dev) *dev = s->mbox;
    if (bytes) *bytes = s->mb_bytes;
    return EVOX_OK;
}

evox_status evox_pso_mailbox_ipc(evox_pso* s, uint8_t out[64]) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!out) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    if (!s->mbox) return fail(EVOX_ERR_CONFIG, "no mailbox (world > %d)", evox::kMaxPeers);
    DevGuard g(s->device);
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
    CU(s, cudaIpcGetMemHandle(&h, s->mbox));
    std::memcpy(out, &h, 64);
    return EVOX_OK;
}

evox_status evox_pso_connect(evox_pso* s, int mode, const void* peers) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    if (!peers) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL peers");
    if (mode != 0 && mode != 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
    if (!s->mbox) return fail(EVOX_ERR_CONFIG, "peer exchange supports world <= %d", evox::kMaxPeers);
    if (s->stepped || s->asked)
        return fail(EVOX_ERR_CONTRACT, "connect before the first step/ask (after init or load)");
    DevGuard g(s->device);
    for (int r = 0; r < s->world; ++r) {
        if (r == s->rank) {
            s->peers[r] = s->mbox;
            continue;
        }
        if (mode == 0) {
            void* p = static_cast<void* const*>(peers)[r];
            if (!p) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL mailbox pointer for rank %d", r);
            cudaPointerAttributes at;
            CU(s, cudaPointerGetAttributes(&at, p));
            if (at.device != s->device) {
                int can = 0;
                CU(s, cudaDeviceCanAccessPeer(&can, s->device, at.device));
                if (!can)
                    return fail(EVOX_ERR_CONFIG, "device %d cannot access device %d", s->device,
                                at.device);
                cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) return poison(s, EVOX_ERR_CUDA, "cudaDeviceEnablePeerAccess", e);
            }
            s->peers[r] = static_cast<unsigned char*>(p);
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const uint8_t*>(peers) + 64 * r, 64);
            void* p = nullptr;
            CU(s, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            s->ipc_opened.push_back(p);
            s->peers[r] = static_cast<unsigned char*>(p);
        }
    }
    // a step must never synchronise (single-process groups would deadlock):
    // pre-size the history
    st = ensure_hist(s, 1 << 16);
    if (st != EVOX_OK) return st;
    s->peer = true;
    for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);  // args changed
    s->graphs.clear();
    return EVOX_OK;
}

evox_status evox_pso_set_timing(evox_pso* s, int enable) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    s->timing = enable != 0;
    return EVOX_OK;
}

evox_status evox_pso_kernel_time(evox_pso* s, double* total_ms, int64_t* gens, int64_t* launches,
                                 int reset) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    CU(s, collect_timing(s));
    if (total_ms) *total_ms = s->kernel_ms;
    if (gens) *gens = s->kernel_n;
    if (launches) *launches = s->kernel_launches;
    if (reset) {
        s->kernel_ms = 0.0;
        s->kernel_n = 0;
        s->kernel_launches = 0;
    }
    return EVOX_OK;
}

evox_status evox_pso_fin_time(evox_pso* s, double* total_ms, int64_t* launches, int reset) {
    evox_status st = check_pso(s);
    if (st != EVOX_OK) return st;
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    CU(s, collect_timing(s));
    if (total_ms) *total_ms = s->fin_ms;
    if (launches) *launches = s->fin_launches;
    if (reset) {
        s->fin_ms = 0.0;
        s->fin_launches = 0;
    }
    return EVOX_OK;
}

evox_status evox_pso_destroy(evox_pso* s) {
    if (!s) return EVOX_OK;
    {
        DevGuard g(s->device);
        if (s->stream) cudaStreamSynchronize(s->stream);
        for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
        if (s->mbox) cudaFree(s->mbox);
        cudaGetLastError();
    }
    base_release(s);
    delete s;
    return EVOX_OK;
}

}  // extern "C"

// ============================================================== CSO handle
struct evox_cso : Base {
    float phi = 0.0f;
    int64_t B = 0;
    bool aligned = true;  // every shard holds whole pairing blocks
    // global pairing across shards (evox_cso_connect)
    bool peer = false;
    float* pX[evox::kMaxPeers] = {};
    float* pf[evox::kMaxPeers][2] = {};
    unsigned char* pmbox[evox::kMaxPeers] = {};
    long long prow0[evox::kMaxPeers + 1] = {};
    std::vector<void*> ipc_opened;
    unsigned char* mbox = nullptr;
    float *X = nullptr, *V = nullptr, *xbar = nullptr;
    float* f2[2] = {nullptr, nullptr};  // fitness by generation parity
    float* fcur() const { return f2[(t < 0 ? 0 : t) & 1]; }
    // phi != 0 (R-15): fixed-point column-sum limbs, their scale 2^qs, and every
    // rank's limbs / column-sum flags when connected
    unsigned long long* limb = nullptr;
    double qscale = 1.0, qinv = 1.0;
    unsigned long long* plimb[evox::kMaxPeers] = {};
    unsigned long long* pcflag[evox::kMaxPeers] = {};
    unsigned long long* cflag() const {
        return reinterpret_cast<unsigned long long*>(mbox + (size_t)32 * (world > 1 ? world : 1));
    }
    unsigned long long* keybuf = nullptr;
    int gen_grid[5] = {0, 0, 0, 0, 0};
    CsoArgs args() const {
        CsoArgs a;
        std::memset(&a, 0, sizeof a);
        a.X = X; a.V = V; a.f2[0] = f2[0]; a.f2[1] = f2[1];
        a.lb = lb_d; a.ub = ub_d; a.lb0 = lb[0]; a.ub0 = ub[0];
        a.uniform_bounds = uniform ? 1 : 0;
        a.rows = rows; a.row0 = row0; a.D = dim; a.ld = ld; a.pop = pop;
        a.B = B; a.phi = phi; a.xbar = xbar; a.limb = limb;
        a.k0 = (unsigned)(seed & 0xffffffffu);
        a.k1 = (unsigned)(seed >> 32);
        a.rk = evox::Philox::schedule(seed);
        a.ctl = ctl;
        a.rank = rank;
        a.world = world;
        a.exchange = comm != nullptr && !peer;
        a.peer = peer ? 1 : 0;
        a.peer_timeout_ns = peer_timeout_ns;
        if (peer) {
            a.nsh = world;
            for (int r = 0; r < world; ++r) {
                a.pX[r] = pX[r];
                a.pf[r][0] = pf[r][0];
                a.pf[r][1] = pf[r][1];
                a.mbox[r] = pmbox[r];
                a.plimb[r] = plimb[r];
                a.pcflag[r] = pcflag[r];
                a.prow0[r] = prow0[r];
            }
            a.prow0[world] = pop;
        } else {  // one table entry: our own shard
            a.nsh = 1;
            a.pX[0] = X;
            a.pf[0][0] = f2[0];
            a.pf[0][1] = f2[1];
            a.mbox[0] = mbox;
            a.plimb[0] = limb;
            a.pcflag[0] = cflag();
            a.prow0[0] = row0;
            a.prow0[1] = row0 + rows;
        }
        return a;
    }
};

namespace {

void cso_layout(evox_cso* s, Carver& c) {
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    c.add(&s->X, mat);
    c.add(&s->V, mat);
    c.add(&s->f2[0], sizeof(float) * s->rows);
    c.add(&s->f2[1], sizeof(float) * s->rows);
    c.add(&s->lb_d, sizeof(float) * s->ld);
    c.add(&s->ub_d, sizeof(float) * s->ld);
    c.add(&s->ctl, sizeof(Ctl));
    c.add(&s->xbar, sizeof(float) * s->ld);
    // per-generation barrier slots (2 x world x 16 B) + column-sum flags (world x 8 B)
    c.add(&s->mbox, (size_t)40 * (s->world > 1 ? s->world : 1));
    if (s->phi != 0.0f) c.add(&s->limb, sizeof(unsigned long long) * 2 * s->ld);
}

int64_t default_block(int64_t pop) {
    // B = pop/8 (blocks align with 1/2/4/8 shards when pop % 16 == 0), else pop.
    if (pop % 16 == 0 && pop >= 16) return pop / 8;
    return pop;
}

evox_status check_cso(evox_cso* s) {
    if (!s) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL handle");
    if (s->poisoned) return fail(EVOX_ERR_POISONED, "handle poisoned by an earlier CUDA/NCCL error");
    return EVOX_OK;
}

}  // namespace

extern "C" {

evox_status evox_cso_workspace_bytes(int64_t pop, int64_t dim, int world, int rank, size_t* bytes) {
    if (!bytes) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    if (pop < 2 || dim < 1) return fail(EVOX_ERR_SHAPE, "need pop >= 2 and dim >= 1");
    if (world < 1) world = 1;
    if (rank < 0 || rank >= world) return fail(EVOX_ERR_INVALID_ARGUMENT, "rank out of range");
    evox_cso s;
    s.world = world;
    s.rank = rank;
    s.ld = round4(dim);
    shard(pop, world, rank, &s.row0, &s.rows);
    Carver c;
    cso_layout(&s, c);
    *bytes = c.off;
    return EVOX_OK;
}

evox_status evox_cso_init(int64_t pop, int64_t dim, const float* lb, const float* ub, float phi,
                          int64_t block, uint64_t seed, const evox_opts* opts, evox_cso** out) {
    if (!out) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output handle pointer");
    *out = nullptr;
    if (pop < 2) return fail(EVOX_ERR_INVALID_ARGUMENT, "CSO needs pop >= 2 (got %lld)", (long long)pop);
    if (dim < 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "dim must be >= 1");
    if (pop > 0xFFFFFFFFll) return fail(EVOX_ERR_SHAPE, "pop must be < 2^32");
    if (round4(dim) > MAX_LD) return fail(EVOX_ERR_SHAPE, "dim must be <= 2^31 - 4 (in-row indices are 32-bit)");
    if (!mul_ok(pop, round4(dim), INT64_MAX / 64)) return fail(EVOX_ERR_SHAPE, "pop*dim overflows");
    if (!std::isfinite(phi)) return fail(EVOX_ERR_INVALID_ARGUMENT, "phi must be finite");
    if (block < 0 || block == 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "block must be 0 (default) or >= 2");
    evox_status st = check_bounds(dim, lb, ub);
    if (st != EVOX_OK) return st;
    int world, rank;
    st = check_opts(opts, &world, &rank);
    if (st != EVOX_OK) return st;
    const int64_t B = block == 0 ? default_block(pop) : (block > pop ? pop : block);
    bool aligned = true;
    if (world > 1) {
        aligned = pop % world == 0 && (pop / world) % B == 0;
        if (!aligned && (world > evox::kMaxPeers || (opts && opts->workspace)))
            return fail(EVOX_ERR_CONFIG,
                        "CSO with world %d and blocks straddling shards (pop=%lld, B=%lld) needs "
                        "global pairing through evox_cso_connect (world <= %d, no workspace)",
                        world, (long long)pop, (long long)B, evox::kMaxPeers);
    }
    evox_cso* s = new (std::nothrow) evox_cso;
    if (!s) return fail(EVOX_ERR_OUT_OF_MEMORY, "host allocation failed");
    s->phi = phi;
    s->B = B;
    s->aligned = aligned;
    {  // R-15: |x| <= max|bound| <= 2^m  ->  x 2^qs is an integer grid with |q| <= 2^54
        double m = 0.0;
        for (int64_t j = 0; j < dim; ++j)
            m = std::max(m, std::max(std::fabs((double)lb[j]), std::fabs((double)ub[j])));
        int e = 0;
        const double fr = std::frexp(m, &e);  // m = fr 2^e, fr in [0.5, 1)
        if (fr == 0.5) e -= 1;                // exact power of two: 2^(e-1)
        s->qscale = std::ldexp(1.0, 54 - e);
        s->qinv = std::ldexp(1.0, e - 54);
    }
    st = base_setup(s, pop, dim, lb, ub, seed, opts, world, rank);
    if (st == EVOX_OK) {
        Carver c;
        cso_layout(s, c);
        st = base_alloc(s, c, opts);
    }
    if (st == EVOX_OK) st = base_common_init(s);
    if (st == EVOX_OK) {
        DevGuard g(s->device);
        cudaError_t e = evox::launch_cso_init(s->args(), s->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(s->xbar, 0, sizeof(float) * s->ld, s->stream);
        if (e == cudaSuccess)  // peer-barrier flags start at 0 ("nothing published")
            e = cudaMemsetAsync(s->mbox, 0, (size_t)40 * (s->world > 1 ? s->world : 1), s->stream);
        if (e == cudaSuccess) e = cudaMalloc(&s->keybuf, sizeof(unsigned long long));
        if (e != cudaSuccess) st = poison(s, EVOX_ERR_CUDA, "cso init", e);
        for (int p = 0; p < 5 && st == EVOX_OK; ++p)
            s->gen_grid[p] = evox::cso_gen_grid(p, s->args(), s->device);
    }
    if (st != EVOX_OK) {
        std::string keep = t_err;
        base_release(s);
        delete s;
        t_err = keep;
        return st;
    }
    *out = s;
    return EVOX_OK;
}

evox_status evox_cso_step(evox_cso* s, evox_problem problem, int64_t n_gens) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (!valid_problem(problem)) return fail(EVOX_ERR_INVALID_ARGUMENT, "unknown problem %d", (int)problem);
    if (n_gens < 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "n_gens must be >= 0");
    if (s->problem >= 0 && s->problem != (int)problem)
        return fail(EVOX_ERR_CONTRACT, "handle is bound to problem %d (got %d)", s->problem, (int)problem);
    if (n_gens > (int64_t)0xFFFFFFFFll - 2 - s->t)
        return fail(EVOX_ERR_SHAPE, "generation counter would exceed 2^32");
    if (s->world > 1 && !s->peer && (!s->comm || !s->aligned))
        return fail(EVOX_ERR_CONTRACT,
                    s->aligned ? "world > 1: pass opts.nccl_id at init or call evox_cso_connect"
                               : "pairing blocks straddle shards: call evox_cso_connect first");
    s->stepped = true;
    DevGuard g(s->device);
    const int64_t t0 = s->t < 0 ? 0 : s->t;
    st = ensure_hist(s, t0 + n_gens + 1);
    if (st != EVOX_OK) return st;
    s->problem = (int)problem;
    const CsoArgs a = s->args();
    int64_t first = t0 + 1;  // first hist index written by this call
    if (s->t < 0) {
        CU(s, evox::launch_eval((int)problem, s->X, s->rows, s->dim, s->ld, s->f2[0], s->stream));
        CU(s, evox::launch_cso_tell0(a, s->stream));
        s->t = 0;
        first = 0;
    }
    if (n_gens > 0) {
        st = run_graphed(s, (int)problem, n_gens, [&]() -> evox_status {
            if (s->phi != 0.0f) {  // x-bar of the generation's population (R-15)
                CU(s, cudaMemsetAsync(s->limb, 0, sizeof(unsigned long long) * 2 * s->ld, s->stream));
                CU(s, evox::launch_cso_colsum(a, s->qscale, s->stream));
                if (s->comm && !s->peer)
                    NC(s, evox::nccl_api(nullptr)->AllReduce(s->limb, s->limb, (size_t)(2 * s->ld),
                                                            ncclUint64, ncclSum, s->comm, s->stream));
                CU(s, evox::launch_cso_colmean(a, s->qinv, s->stream));
            }
            CU(s, timed(s, [&] {
                return evox::launch_cso_gen((int)problem, a, s->gen_grid[problem], s->stream);
            }));
            return EVOX_OK;
        });
        if (st != EVOX_OK) return st;
        s->t += n_gens;
        s->min_key_stale = false;
    }
    if (s->comm && !s->peer) {  // one min-reduction of this call's per-generation keys
        const int64_t n = s->t - first + 1;
        if (n > 0) {
            const evox::NcclApi* api = evox::nccl_api(nullptr);
            NC(s, api->AllReduce(s->hkeys + first, s->hkeys + first, (size_t)n, ncclUint64, ncclMin,
                                 s->comm, s->stream));
            CU(s, evox::launch_cso_hist_from_keys(a, (unsigned long long)first, n, s->stream));
        }
    }
    return EVOX_OK;
}

evox_status evox_cso_sync(evox_cso* s) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    return sync_check(s);
}

evox_status evox_cso_best(evox_cso* s, float* fit, int64_t* global_index, float* row_host) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (s->t < 0) {  // nothing evaluated yet: no best (the fitness arrays are unset)
        if (fit) *fit = INFINITY;
        if (global_index) *global_index = -1;
        return sync_check(s);
    }
    DevGuard g(s->device);
    if (!s->peer && !s->comm && !s->min_key_stale)
        return staged_best(s, s->X, s->X, nullptr, nullptr, fit, global_index, row_host);
    const evox::NcclApi* api = (s->comm && !s->peer) ? evox::nccl_api(nullptr) : nullptr;
    if (!s->peer) {
        CU(s, evox::launch_argmin_rows(s->fcur(), s->rows, s->row0, s->keybuf, s->stream));
        if (api)
            NC(s, api->AllReduce(s->keybuf, s->keybuf, 1, ncclUint64, ncclMin, s->comm, s->stream));
    }
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    unsigned long long key = 0;
    if (s->peer) {  // global minimum of the last generation, from the in-kernel barrier
        Ctl c;
        CU(s, cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost));
        key = c.min_key;
    } else {
        CU(s, cudaMemcpy(&key, s->keybuf, sizeof key, cudaMemcpyDeviceToHost));
    }
    float fv = INFINITY;
    int64_t gi = -1;
    if (key != ~0ull) {
        const uint32_t o = (uint32_t)(key >> 32);
        const uint32_t bits = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
        std::memcpy(&fv, &bits, 4);
        gi = (int64_t)(uint32_t)(key & 0xffffffffu);
    }
    if (fit) *fit = fv;
    if (global_index) *global_index = gi;
    if (row_host && gi >= 0 && s->peer) {
        int w = 0;
        while (w + 1 < s->world && gi >= s->prow0[w + 1]) ++w;
        CU(s, cudaMemcpy(row_host, s->pX[w] + (gi - s->prow0[w]) * s->ld, 4 * s->dim,
                         cudaMemcpyDeviceToHost));
    } else if (row_host && gi >= 0 && !api) {
        // one rank: the stream is already synchronised and the row is local
        CU(s, cudaMemcpy(row_host, s->X + (gi - s->row0) * s->ld, 4 * s->dim,
                         cudaMemcpyDeviceToHost));
    } else if (row_host && gi >= 0) {
        const bool mine = gi >= s->row0 && gi < s->row0 + s->rows;
        if (mine)
            CU(s, cudaMemcpyAsync(s->scratch_row, s->X + (gi - s->row0) * s->ld, 4 * s->ld,
                                  cudaMemcpyDeviceToDevice, s->stream));
        else
            CU(s, cudaMemsetAsync(s->scratch_row, 0, 4 * s->ld, s->stream));
        if (api)
            NC(s, api->AllReduce(s->scratch_row, s->scratch_row, (size_t)s->ld, ncclFloat32, ncclSum,
                                 s->comm, s->stream));
        st = sync_check(s);
        if (st != EVOX_OK) return st;
        CU(s, cudaMemcpy(row_host, s->scratch_row, 4 * s->dim, cudaMemcpyDeviceToHost));
    }
    return EVOX_OK;
}

evox_status evox_cso_history(evox_cso* s, float* best_per_gen, int64_t cap, int64_t* n) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (cap < 0 || (cap > 0 && !best_per_gen)) return fail(EVOX_ERR_INVALID_ARGUMENT, "bad buffer");
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    const int64_t T = s->t + 1;
    if (n) *n = T;
    const int64_t k = T < cap ? T : cap;
    DevGuard g(s->device);
    if (k > 0) CU(s, cudaMemcpy(best_per_gen, s->hist, sizeof(float) * k, cudaMemcpyDeviceToHost));
    return EVOX_OK;
}

evox_status evox_cso_view(evox_cso* s, int field, void** dev, int64_t* rows, int64_t* ld) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (!dev) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    int64_t r = s->rows, l = s->ld;
    switch (field) {
        case EVOX_FIELD_X: *dev = s->X; break;
        case EVOX_FIELD_V: *dev = s->V; break;
        case EVOX_FIELD_F: *dev = s->fcur(); l = 1; break;
        default: return fail(EVOX_ERR_INVALID_ARGUMENT, "field %d not available for CSO", field);
    }
    if (rows) *rows = r;
    if (ld) *ld = l;
    return sync_check(s);
}

evox_status evox_cso_info(evox_cso* s, int64_t* pop, int64_t* dim, int64_t* ld, int64_t* row0,
                          int64_t* rows, int64_t* t, void** cuda_stream) {
    if (!s) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL handle");
    if (pop) *pop = s->pop;
    if (dim) *dim = s->dim;
    if (ld) *ld = s->ld;
    if (row0) *row0 = s->row0;
    if (rows) *rows = s->rows;
    if (t) *t = s->t;
    if (cuda_stream) *cuda_stream = s->stream;
    return s->poisoned ? fail(EVOX_ERR_POISONED, "handle poisoned") : EVOX_OK;
}

// Blob: header | X | V | f | hist[0..t]
evox_status evox_cso_save(evox_cso* s, void* host_blob, size_t cap, size_t* used) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (!used) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL used");
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    const int64_t T = s->t + 1;
    const size_t need = sizeof(BlobHdr) + 2 * mat + 4 * (size_t)s->rows + 4 * (size_t)(T > 0 ? T : 0);
    *used = need;
    if (!host_blob) return EVOX_OK;
    if (cap < need) return fail(EVOX_ERR_INVALID_ARGUMENT, "blob buffer too small");
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    BlobHdr h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, "EVOXCSO1", 8);
    h.kind = 1; h.pop = s->pop; h.dim = s->dim; h.ld = s->ld; h.row0 = s->row0; h.rows = s->rows;
    h.t = s->t; h.problem = s->problem; h.world = s->world; h.rank = s->rank; h.seed = s->seed;
    h.w = s->phi; h.B = s->B;
    char* p = static_cast<char*>(host_blob);
    std::memcpy(p, &h, sizeof h);
    p += sizeof h;
    CU(s, cudaMemcpy(p, s->X, mat, cudaMemcpyDeviceToHost)); p += mat;
    CU(s, cudaMemcpy(p, s->V, mat, cudaMemcpyDeviceToHost)); p += mat;
    CU(s, cudaMemcpy(p, s->fcur(), 4 * s->rows, cudaMemcpyDeviceToHost)); p += 4 * s->rows;
    if (T > 0) CU(s, cudaMemcpy(p, s->hist, 4 * T, cudaMemcpyDeviceToHost));
    return EVOX_OK;
}

evox_status evox_cso_load(evox_cso* s, const void* host_blob, size_t size) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (s->peer)
        return fail(EVOX_ERR_CONTRACT,
                    "load on a peer-connected handle: load every rank's blob, then connect");
    if (!host_blob || size < sizeof(BlobHdr)) return fail(EVOX_ERR_INVALID_ARGUMENT, "bad blob");
    BlobHdr h;
    std::memcpy(&h, host_blob, sizeof h);
    if (std::memcmp(h.magic, "EVOXCSO1", 8) != 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "not a CSO blob");
    if (h.pop != s->pop || h.dim != s->dim || h.ld != s->ld || h.row0 != s->row0 ||
        h.rows != s->rows || h.world != s->world || h.rank != s->rank || h.B != s->B)
        return fail(EVOX_ERR_SHAPE, "blob shape/shard does not match the handle");
    if (h.seed != s->seed || h.w != s->phi)
        return fail(EVOX_ERR_CONTRACT, "blob parameters (seed/phi) differ from the handle's");
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    const int64_t T = h.t + 1;
    const size_t need = sizeof(BlobHdr) + 2 * mat + 4 * (size_t)s->rows + 4 * (size_t)(T > 0 ? T : 0);
    if (size < need) return fail(EVOX_ERR_SHAPE, "blob truncated");
    DevGuard g(s->device);
    st = ensure_hist(s, (T > 0 ? T : 0) + 1);
    if (st != EVOX_OK) return st;
    CU(s, cudaStreamSynchronize(s->stream));
    const char* p = static_cast<const char*>(host_blob) + sizeof h;
    CU(s, cudaMemcpy(s->X, p, mat, cudaMemcpyHostToDevice)); p += mat;
    CU(s, cudaMemcpy(s->V, p, mat, cudaMemcpyHostToDevice)); p += mat;
    CU(s, cudaMemcpy(s->f2[(h.t < 0 ? 0 : h.t) & 1], p, 4 * s->rows, cudaMemcpyHostToDevice));
    p += 4 * s->rows;
    if (T > 0) CU(s, cudaMemcpy(s->hist, p, 4 * T, cudaMemcpyHostToDevice));
    Ctl c;
    CU(s, cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost));
    c.gen_key = ~0ull;
    c.mkey[0] = c.mkey[1] = c.mkey[2] = ~0ull;
    c.ticket = 0;
    c.t = h.t < 0 ? 0 : (unsigned long long)h.t;
    CU(s, cudaMemcpy(s->ctl, &c, sizeof c, cudaMemcpyHostToDevice));
    s->t = h.t;
    s->problem = (int)h.problem;
    s->min_key_stale = true;  // ctl->min_key is the pre-load population's
    s->stepped = false;
    return EVOX_OK;
}

evox_status evox_cso_state(evox_cso* s, void** base, uint8_t ipc[64]) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (!s->own_base) return fail(EVOX_ERR_CONFIG, "the state is a caller workspace: not exportable");
    if (base) *base = s->base;
    if (ipc) {
        DevGuard g(s->device);
        cudaIpcMemHandle_t h;
        CU(s, cudaIpcGetMemHandle(&h, s->base));
        std::memcpy(ipc, &h, 64);
    }
    return EVOX_OK;
}

evox_status evox_cso_connect(evox_cso* s, int mode, const void* peers) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    if (!peers) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL peers");
    if (mode != 0 && mode != 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
    if (s->world > evox::kMaxPeers) return fail(EVOX_ERR_CONFIG, "world <= %d", evox::kMaxPeers);
    if (s->stepped) return fail(EVOX_ERR_CONTRACT, "connect before the first step (after init or load)");
    DevGuard g(s->device);
    for (int r = 0; r < s->world; ++r) {
        unsigned char* base = nullptr;
        if (r == s->rank) {
            base = static_cast<unsigned char*>(s->base);
        } else if (mode == 0) {
            base = static_cast<unsigned char*>(static_cast<void* const*>(peers)[r]);
            if (!base) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL state pointer for rank %d", r);
            cudaPointerAttributes at;
            CU(s, cudaPointerGetAttributes(&at, base));
            if (at.device != s->device) {
                cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) return poison(s, EVOX_ERR_CUDA, "cudaDeviceEnablePeerAccess", e);
            }
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const uint8_t*>(peers) + 64 * r, 64);
            void* p = nullptr;
            CU(s, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            s->ipc_opened.push_back(p);
            base = static_cast<unsigned char*>(p);
        }
        evox_cso probe;  // rank r's layout: the same carving with its own shard size
        probe.world = s->world;
        probe.ld = s->ld;
        probe.phi = s->phi;
        shard(s->pop, s->world, r, &probe.row0, &probe.rows);
        Carver c;
        cso_layout(&probe, c);
        c.assign(base);
        s->pX[r] = probe.X;
        s->pf[r][0] = probe.f2[0];
        s->pf[r][1] = probe.f2[1];
        s->pmbox[r] = probe.mbox;
        s->plimb[r] = probe.limb;
        s->pcflag[r] = probe.cflag();
        s->prow0[r] = probe.row0;
    }
    st = ensure_hist(s, 1 << 16);  // a step must never synchronise (single-process groups)
    if (st != EVOX_OK) return st;
    s->peer = true;
    for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
    s->graphs.clear();
    for (int p = 0; p < 5; ++p) s->gen_grid[p] = evox::cso_gen_grid(p, s->args(), s->device);
    return EVOX_OK;
}

evox_status evox_cso_set_timing(evox_cso* s, int enable) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    s->timing = enable != 0;
    return EVOX_OK;
}

evox_status evox_cso_kernel_time(evox_cso* s, double* total_ms, int64_t* gens, int64_t* launches,
                                 int reset) {
    evox_status st = check_cso(s);
    if (st != EVOX_OK) return st;
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    CU(s, collect_timing(s));
    if (total_ms) *total_ms = s->kernel_ms;
    if (gens) *gens = s->kernel_n;
    if (launches) *launches = s->kernel_launches;
    if (reset) {
        s->kernel_ms = 0.0;
        s->kernel_n = 0;
        s->kernel_launches = 0;
    }
    return EVOX_OK;
}

evox_status evox_cso_destroy(evox_cso* s) {
    if (!s) return EVOX_OK;
    DevGuard g(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
    if (s->keybuf) cudaFree(s->keybuf);
    base_release(s);
    delete s;
    return EVOX_OK;
}

}  // extern "C"

// ============================================================== DE handle
struct evox_de : Base {
    float F = 0.5f, CR = 0.9f;
    float* buf[2] = {nullptr, nullptr};
    unsigned char* sel[2] = {nullptr, nullptr};
    float* f[2] = {nullptr, nullptr};
    unsigned char* mbox = nullptr;  // 2 x world key slots (carved from the state)
    int gen_grid[5] = {0, 0, 0, 0, 0};
    // cross-shard donors (evox_de_connect)
    bool peer = false;
    float* pbuf[evox::kMaxPeers][2] = {};
    unsigned char* psel[evox::kMaxPeers][2] = {};
    unsigned char* pmbox[evox::kMaxPeers] = {};
    long long prow0[evox::kMaxPeers + 1] = {};
    std::vector<void*> ipc_opened;
    float* gathered = nullptr;  // peers connected: view/save gather here, never in place
    evox::DeArgs args() const {
        evox::DeArgs a;
        std::memset(&a, 0, sizeof a);
        for (int i = 0; i < 2; ++i) {
            a.buf[i] = buf[i];
            a.sel[i] = sel[i];
            a.f[i] = f[i];
        }
        a.lb = lb_d; a.ub = ub_d; a.lb0 = lb[0]; a.ub0 = ub[0];
        a.uniform_bounds = uniform ? 1 : 0;
        a.rows = rows; a.row0 = row0; a.D = dim; a.ld = ld; a.pop = pop;
        a.F = F; a.CR = CR;
        a.k0 = (unsigned)(seed & 0xffffffffu);
        a.k1 = (unsigned)(seed >> 32);
        a.rk = evox::Philox::schedule(seed);
        a.ctl = ctl;
        a.rank = rank;
        a.world = world;
        a.peer = peer ? 1 : 0;
        a.peer_timeout_ns = peer_timeout_ns;
        if (peer) {
            for (int r = 0; r < world; ++r) {
                a.pbuf[r][0] = pbuf[r][0];
                a.pbuf[r][1] = pbuf[r][1];
                a.psel[r][0] = psel[r][0];
                a.psel[r][1] = psel[r][1];
                a.mbox[r] = pmbox[r];
                a.prow0[r] = prow0[r];
            }
            a.prow0[world] = pop;
        } else {  // one shard: our own state
            a.world = 1;
            a.pbuf[0][0] = buf[0];
            a.pbuf[0][1] = buf[1];
            a.psel[0][0] = sel[0];
            a.psel[0][1] = sel[1];
            a.mbox[0] = mbox;
            a.prow0[0] = 0;
            a.prow0[1] = pop;
        }
        return a;
    }
};

namespace {

void de_layout(evox_de* s, Carver& c) {
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    c.add(&s->buf[0], mat);
    c.add(&s->buf[1], mat);
    c.add(&s->sel[0], s->rows);
    c.add(&s->sel[1], s->rows);
    c.add(&s->f[0], sizeof(float) * s->rows);
    c.add(&s->f[1], sizeof(float) * s->rows);
    c.add(&s->lb_d, sizeof(float) * s->ld);
    c.add(&s->ub_d, sizeof(float) * s->ld);
    c.add(&s->ctl, sizeof(Ctl));
    c.add(&s->mbox, (size_t)32 * (s->world > 1 ? s->world : 1));
}

evox_status check_de(evox_de* s) {
    if (!s) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL handle");
    if (s->poisoned) return fail(EVOX_ERR_POISONED, "handle poisoned by an earlier CUDA error");
    return EVOX_OK;
}

}  // namespace

extern "C" {

evox_status evox_de_workspace_bytes(int64_t pop, int64_t dim, size_t* bytes) {
    if (!bytes) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    if (pop < 4 || dim < 1) return fail(EVOX_ERR_SHAPE, "need pop >= 4 and dim >= 1");
    evox_de s;
    s.ld = round4(dim);
    s.rows = pop;
    Carver c;
    de_layout(&s, c);
    *bytes = c.off;
    return EVOX_OK;
}

evox_status evox_de_init(int64_t pop, int64_t dim, const float* lb, const float* ub, float F,
                         float CR, uint64_t seed, const evox_opts* opts, evox_de** out) {
    if (!out) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output handle pointer");
    *out = nullptr;
    if (pop < 4) return fail(EVOX_ERR_CONFIG, "DE needs pop >= 4 (got %lld; S:326)", (long long)pop);
    if (dim < 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "dim must be >= 1");
    if (pop > 0xFFFFFFFFll) return fail(EVOX_ERR_SHAPE, "pop must be < 2^32");
    if (round4(dim) > MAX_LD) return fail(EVOX_ERR_SHAPE, "dim must be <= 2^31 - 4 (in-row indices are 32-bit)");
    if (!mul_ok(pop, round4(dim), INT64_MAX / 64)) return fail(EVOX_ERR_SHAPE, "pop*dim overflows");
    if (!(F > 0.0f && F <= 2.0f))  // SPEC de_setup: F in (0, 2]
        return fail(EVOX_ERR_INVALID_ARGUMENT, "F must be in (0, 2]");
    if (!(CR >= 0.0f && CR <= 1.0f)) return fail(EVOX_ERR_INVALID_ARGUMENT, "CR must be in [0,1]");
    evox_status st = check_bounds(dim, lb, ub);
    if (st != EVOX_OK) return st;
    int world, rank;
    st = check_opts(opts, &world, &rank);
    if (st != EVOX_OK) return st;
    if (world > evox::kMaxPeers)
        return fail(EVOX_ERR_CONFIG, "DE supports world <= %d", evox::kMaxPeers);
    if (world > 1 && opts && opts->workspace)
        return fail(EVOX_ERR_CONFIG, "sharded DE maps the library-allocated state: no workspace");
    if (opts && opts->nccl_id)
        return fail(EVOX_ERR_CONFIG, "DE shards connect through evox_de_connect, not NCCL");
    evox_de* s = new (std::nothrow) evox_de;
    if (!s) return fail(EVOX_ERR_OUT_OF_MEMORY, "host allocation failed");
    s->F = F;
    s->CR = CR;
    st = base_setup(s, pop, dim, lb, ub, seed, opts, world, rank);
    if (st == EVOX_OK) {
        Carver c;
        de_layout(s, c);
        st = base_alloc(s, c, opts);
    }
    if (st == EVOX_OK) st = base_common_init(s);
    if (st == EVOX_OK) {
        DevGuard g(s->device);
        cudaError_t e = evox::launch_de_init(s->args(), s->stream);
        if (e == cudaSuccess)  // peer-barrier flags start at 0 ("nothing published")
            e = cudaMemsetAsync(s->mbox, 0, (size_t)32 * (s->world > 1 ? s->world : 1), s->stream);
        if (e != cudaSuccess) st = poison(s, EVOX_ERR_CUDA, "de init", e);
        for (int p = 0; p < 5 && st == EVOX_OK; ++p)
            s->gen_grid[p] = evox::de_gen_grid(p, s->ld, s->rows, s->device,
                                               (s->flags & EVOX_FLAG_NO_WAVE) != 0);
    }
    if (st != EVOX_OK) {
        std::string keep = t_err;
        base_release(s);
        delete s;
        t_err = keep;
        return st;
    }
    *out = s;
    return EVOX_OK;
}

evox_status evox_de_step(evox_de* s, evox_problem problem, int64_t n_gens) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (!valid_problem(problem)) return fail(EVOX_ERR_INVALID_ARGUMENT, "unknown problem %d", (int)problem);
    if (n_gens < 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "n_gens must be >= 0");
    if (s->problem >= 0 && s->problem != (int)problem)
        return fail(EVOX_ERR_CONTRACT, "handle is bound to problem %d (got %d)", s->problem, (int)problem);
    if (n_gens > (int64_t)0xFFFFFFFFll - 2 - s->t)
        return fail(EVOX_ERR_SHAPE, "generation counter would exceed 2^32");
    if (s->world > 1 && !s->peer)
        return fail(EVOX_ERR_CONTRACT, "world > 1: call evox_de_connect before stepping");
    s->stepped = true;
    DevGuard g(s->device);
    st = ensure_hist(s, (s->t < 0 ? 0 : s->t) + n_gens + 1);
    if (st != EVOX_OK) return st;
    s->problem = (int)problem;
    const evox::DeArgs a = s->args();
    if (s->t < 0) {
        CU(s, evox::launch_eval((int)problem, s->buf[0], s->rows, s->dim, s->ld, s->f[0], s->stream));
        CU(s, evox::launch_de_tell0(a, s->stream));
        s->t = 0;
    }
    if (n_gens == 0) return EVOX_OK;
    const int grid = s->gen_grid[problem];
    st = run_graphed(s, (int)problem, n_gens, [&]() -> evox_status {
        CU(s, timed(s, [&] { return evox::launch_de_gen((int)problem, a, grid, s->stream,
                                                             (s->flags & EVOX_FLAG_NO_WAVE) != 0); }));
        return EVOX_OK;
    });
    if (st != EVOX_OK) return st;
    s->t += n_gens;
    s->min_key_stale = false;
    return EVOX_OK;
}

}  // extern "C"

namespace {
// The current population as one [rows x ld] buffer.  Alone: materialise in place into
// buf[0] (bitwise-neutral).  With peers connected: gather into a separate buffer, because
// the peers' generation kernels read this shard's rows through buf/sel.
evox_status de_current_population(evox_de* s, const float** X) {
    if (!s->peer) {
        CU(s, evox::launch_de_materialize(s->args(), s->stream));
        *X = s->buf[0];
        return EVOX_OK;
    }
    if (!s->gathered) CU(s, cudaMalloc(&s->gathered, sizeof(float) * (size_t)s->rows * s->ld));
    CU(s, evox::launch_de_gather(s->args(), s->gathered, s->stream));
    *X = s->gathered;
    return EVOX_OK;
}
}  // namespace

extern "C" {

// Blob: header | X (gathered) | f (current parity) | hist[0..t]
evox_status evox_de_save(evox_de* s, void* host_blob, size_t cap, size_t* used) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (!used) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL used");
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    const int64_t T = s->t + 1;
    const size_t need = sizeof(BlobHdr) + mat + 4 * (size_t)s->rows + 4 * (size_t)(T > 0 ? T : 0);
    *used = need;
    if (!host_blob) return EVOX_OK;
    if (cap < need) return fail(EVOX_ERR_INVALID_ARGUMENT, "blob buffer too small");
    DevGuard g(s->device);
    const float* X = nullptr;
    st = de_current_population(s, &X);
    if (st != EVOX_OK) return st;
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    const int p = (int)((s->t < 0 ? 0 : s->t) & 1);
    BlobHdr h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, "EVOXDE01", 8);
    h.kind = 2; h.pop = s->pop; h.dim = s->dim; h.ld = s->ld; h.row0 = s->row0; h.rows = s->rows;
    h.t = s->t; h.problem = s->problem; h.world = s->world; h.rank = s->rank; h.seed = s->seed;
    h.w = s->F; h.phi_p = s->CR;
    char* q = static_cast<char*>(host_blob);
    std::memcpy(q, &h, sizeof h);
    q += sizeof h;
    CU(s, cudaMemcpy(q, X, mat, cudaMemcpyDeviceToHost)); q += mat;
    CU(s, cudaMemcpy(q, s->f[p], 4 * s->rows, cudaMemcpyDeviceToHost)); q += 4 * s->rows;
    if (T > 0) CU(s, cudaMemcpy(q, s->hist, 4 * T, cudaMemcpyDeviceToHost));
    return EVOX_OK;
}

evox_status evox_de_load(evox_de* s, const void* host_blob, size_t size) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (s->peer)
        return fail(EVOX_ERR_CONTRACT,
                    "load on a peer-connected handle: load every rank's blob, then connect");
    if (!host_blob || size < sizeof(BlobHdr)) return fail(EVOX_ERR_INVALID_ARGUMENT, "bad blob");
    BlobHdr h;
    std::memcpy(&h, host_blob, sizeof h);
    if (std::memcmp(h.magic, "EVOXDE01", 8) != 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "not a DE blob");
    if (h.pop != s->pop || h.dim != s->dim || h.ld != s->ld || h.row0 != s->row0 ||
        h.rows != s->rows || h.world != s->world || h.rank != s->rank)
        return fail(EVOX_ERR_SHAPE, "blob shape/shard does not match the handle");
    if (h.seed != s->seed || h.w != s->F || h.phi_p != s->CR)
        return fail(EVOX_ERR_CONTRACT, "blob parameters (seed/F/CR) differ from the handle's");
    const size_t mat = sizeof(float) * (size_t)s->rows * (size_t)s->ld;
    const int64_t T = h.t + 1;
    const size_t need = sizeof(BlobHdr) + mat + 4 * (size_t)s->rows + 4 * (size_t)(T > 0 ? T : 0);
    if (size < need) return fail(EVOX_ERR_SHAPE, "blob truncated");
    DevGuard g(s->device);
    st = ensure_hist(s, (T > 0 ? T : 0) + 1);
    if (st != EVOX_OK) return st;
    CU(s, cudaStreamSynchronize(s->stream));
    const int p = (int)((h.t < 0 ? 0 : h.t) & 1);
    const char* q = static_cast<const char*>(host_blob) + sizeof h;
    CU(s, cudaMemcpy(s->buf[0], q, mat, cudaMemcpyHostToDevice)); q += mat;
    CU(s, cudaMemcpy(s->f[p], q, 4 * s->rows, cudaMemcpyHostToDevice)); q += 4 * s->rows;
    if (T > 0) CU(s, cudaMemcpy(s->hist, q, 4 * T, cudaMemcpyHostToDevice));
    CU(s, cudaMemset(s->sel[0], 0, s->rows));  // the population is in buf[0]
    CU(s, cudaMemset(s->sel[1], 0, s->rows));
    Ctl c;
    CU(s, cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost));
    c.gen_key = ~0ull;
    c.mkey[0] = c.mkey[1] = c.mkey[2] = ~0ull;
    c.ticket = 0;
    c.t = h.t < 0 ? 0 : (unsigned long long)h.t;
    CU(s, cudaMemcpy(s->ctl, &c, sizeof c, cudaMemcpyHostToDevice));
    s->t = h.t;
    s->problem = (int)h.problem;
    s->min_key_stale = true;  // ctl->min_key is the pre-load population's
    s->stepped = false;
    return EVOX_OK;
}

evox_status evox_de_sync(evox_de* s) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    return sync_check(s);
}

evox_status evox_de_view(evox_de* s, int field, void** dev, int64_t* rows, int64_t* ld) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (!dev) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL output");
    DevGuard g(s->device);
    const int p = (int)((s->t < 0 ? 0 : s->t) & 1);
    int64_t r = s->rows, l = s->ld;
    switch (field) {
        case EVOX_FIELD_X: {
            const float* X = nullptr;
            st = de_current_population(s, &X);
            if (st != EVOX_OK) return st;
            *dev = const_cast<float*>(X);
            break;
        }
        case EVOX_FIELD_F: *dev = s->f[p]; l = 1; break;
        default: return fail(EVOX_ERR_INVALID_ARGUMENT, "field %d not available for DE", field);
    }
    if (rows) *rows = r;
    if (ld) *ld = l;
    return sync_check(s);
}

evox_status evox_de_best(evox_de* s, float* fit, int64_t* global_index, float* row_host) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (s->t < 0) {  // nothing evaluated yet: no best (the fitness arrays are unset)
        if (fit) *fit = INFINITY;
        if (global_index) *global_index = -1;
        return sync_check(s);
    }
    DevGuard g(s->device);
    if (!s->peer && !s->min_key_stale)
        return staged_best(s, s->buf[0], s->buf[1], s->sel[0], s->sel[1], fit, global_index,
                           row_host);
    const int p = (int)((s->t < 0 ? 0 : s->t) & 1);
    if (!s->peer) CU(s, evox::launch_argmin_rows(s->f[p], s->rows, s->row0, s->scratch_key, s->stream));
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    unsigned long long key = 0;
    if (s->peer) {  // the global minimum of the last generation, from the barrier
        Ctl c;
        CU(s, cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost));
        key = c.min_key;
    } else {
        CU(s, cudaMemcpy(&key, s->scratch_key, sizeof key, cudaMemcpyDeviceToHost));
    }
    float fv = INFINITY;
    int64_t gi = -1;
    if (key != ~0ull) {
        const uint32_t o = (uint32_t)(key >> 32);
        const uint32_t bits = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
        std::memcpy(&fv, &bits, 4);
        gi = (int64_t)(uint32_t)(key & 0xffffffffu);
    }
    if (fit) *fit = fv;
    if (global_index) *global_index = gi;
    if (row_host && gi >= 0) {
        if (!s->peer) {  // the row's current buffer (no population-wide materialise)
            const int64_t lr = gi - s->row0;
            unsigned char sb = 0;
            CU(s, cudaMemcpy(&sb, s->sel[p] + lr, 1, cudaMemcpyDeviceToHost));
            CU(s, cudaMemcpy(row_host, s->buf[sb & 1] + lr * s->ld, 4 * s->dim,
                             cudaMemcpyDeviceToHost));
        } else {  // the owner's current buffer, read through peer memory
            int w = 0;
            while (w + 1 < s->world && gi >= s->prow0[w + 1]) ++w;
            const int64_t lr = gi - s->prow0[w];
            unsigned char sb = 0;
            CU(s, cudaMemcpy(&sb, s->psel[w][p] + lr, 1, cudaMemcpyDeviceToHost));
            CU(s, cudaMemcpy(row_host, s->pbuf[w][sb & 1] + lr * s->ld, 4 * s->dim,
                             cudaMemcpyDeviceToHost));
        }
    }
    return EVOX_OK;
}

evox_status evox_de_history(evox_de* s, float* best_per_gen, int64_t cap, int64_t* n) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (cap < 0 || (cap > 0 && !best_per_gen)) return fail(EVOX_ERR_INVALID_ARGUMENT, "bad buffer");
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    const int64_t T = s->t + 1;
    if (n) *n = T;
    const int64_t k = T < cap ? T : cap;
    DevGuard g(s->device);
    if (k > 0) CU(s, cudaMemcpy(best_per_gen, s->hist, sizeof(float) * k, cudaMemcpyDeviceToHost));
    return EVOX_OK;
}

evox_status evox_de_info(evox_de* s, int64_t* pop, int64_t* dim, int64_t* ld, int64_t* row0,
                         int64_t* rows, int64_t* t, void** cuda_stream) {
    if (!s) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL handle");
    if (pop) *pop = s->pop;
    if (dim) *dim = s->dim;
    if (ld) *ld = s->ld;
    if (row0) *row0 = s->row0;
    if (rows) *rows = s->rows;
    if (t) *t = s->t;
    if (cuda_stream) *cuda_stream = s->stream;
    return s->poisoned ? fail(EVOX_ERR_POISONED, "handle poisoned") : EVOX_OK;
}

evox_status evox_de_state(evox_de* s, void** base, uint8_t ipc[64]) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (!s->own_base) return fail(EVOX_ERR_CONFIG, "the state is a caller workspace: not exportable");
    if (base) *base = s->base;
    if (ipc) {
        DevGuard g(s->device);
        cudaIpcMemHandle_t h;
        CU(s, cudaIpcGetMemHandle(&h, s->base));
        std::memcpy(ipc, &h, 64);
    }
    return EVOX_OK;
}

evox_status evox_de_connect(evox_de* s, int mode, const void* peers) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    if (!peers) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL peers");
    if (mode != 0 && mode != 1) return fail(EVOX_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
    if (s->stepped) return fail(EVOX_ERR_CONTRACT, "connect before the first step (after init or load)");
    DevGuard g(s->device);
    for (int r = 0; r < s->world; ++r) {
        unsigned char* base = nullptr;
        if (r == s->rank) {
            base = static_cast<unsigned char*>(s->base);
        } else if (mode == 0) {
            base = static_cast<unsigned char*>(static_cast<void* const*>(peers)[r]);
            if (!base) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL state pointer for rank %d", r);
            cudaPointerAttributes at;
            CU(s, cudaPointerGetAttributes(&at, base));
            if (at.device != s->device) {
                cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) return poison(s, EVOX_ERR_CUDA, "cudaDeviceEnablePeerAccess", e);
            }
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const uint8_t*>(peers) + 64 * r, 64);
            void* p = nullptr;
            CU(s, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            s->ipc_opened.push_back(p);
            base = static_cast<unsigned char*>(p);
        }
        // rank r's layout: the same carving with its own shard size
        evox_de probe;
        probe.world = s->world;
        probe.ld = s->ld;
        shard(s->pop, s->world, r, &probe.row0, &probe.rows);
        Carver c;
        de_layout(&probe, c);
        c.assign(base);
        s->pbuf[r][0] = probe.buf[0];
        s->pbuf[r][1] = probe.buf[1];
        s->psel[r][0] = probe.sel[0];
        s->psel[r][1] = probe.sel[1];
        s->pmbox[r] = probe.mbox;
        s->prow0[r] = probe.row0;
        probe.lb_d = nullptr;  // nothing owned
    }
    st = ensure_hist(s, 1 << 16);  // a step must never synchronise (single-process groups)
    if (st != EVOX_OK) return st;
    s->peer = true;
    for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
    s->graphs.clear();
    return EVOX_OK;
}

evox_status evox_de_set_timing(evox_de* s, int enable) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    s->timing = enable != 0;
    return EVOX_OK;
}

evox_status evox_de_kernel_time(evox_de* s, double* total_ms, int64_t* gens, int64_t* launches,
                                int reset) {
    evox_status st = check_de(s);
    if (st != EVOX_OK) return st;
    st = sync_check(s);
    if (st != EVOX_OK) return st;
    DevGuard g(s->device);
    CU(s, collect_timing(s));
    if (total_ms) *total_ms = s->kernel_ms;
    if (gens) *gens = s->kernel_n;
    if (launches) *launches = s->kernel_launches;
    if (reset) {
        s->kernel_ms = 0.0;
        s->kernel_n = 0;
        s->kernel_launches = 0;
    }
    return EVOX_OK;
}

evox_status evox_de_destroy(evox_de* s) {
    if (!s) return EVOX_OK;
    {
        DevGuard g(s->device);
        if (s->stream) cudaStreamSynchronize(s->stream);
        for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
        cudaGetLastError();
    }
    base_release(s);
    delete s;
    return EVOX_OK;
}

}  // extern "C"

extern "C" {

evox_status evox_debug_philox(const uint32_t* ctr, uint32_t key0, uint32_t key1, uint32_t* out,
                              int64_t n, void* cuda_stream) {
    if (n < 0) return fail(EVOX_ERR_INVALID_ARGUMENT, "n must be >= 0");
    if (n > 0 && (!ctr || !out)) return fail(EVOX_ERR_INVALID_ARGUMENT, "NULL buffer");
    cudaError_t e = evox::launch_debug_philox(ctr, key0, key1, out, n, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return fail(EVOX_ERR_CUDA, "debug_philox: %s", cudaGetErrorString(e));
    return EVOX_OK;
}

}  // extern "C"
