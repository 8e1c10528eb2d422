// fc_capi.cu -- implementation of include/fuzzyclust_cuda.h.
//
// Host side of the B200-native GPA/FISTA solver: context (device, stream, NCCL
// communicator), CSR upload with the nnz-balanced row partition, work buffers,
// and the on-device iteration loop.  Every per-iteration decision (loss, stop
// rule, FISTA momentum / restart, backtracking) is taken on the device by
// k_finalize, so the host only enqueues iterations and polls a done flag one
// chunk behind (no per-iteration host round trip).
//
// Per FISTA iteration n, per shard (SURVEY.md section 7 step 7 schedule):
//   k_step    bar^n = P(X_ext^n - tau grad f(X_ext^n))      X_ext^n rebuilt from bar^{n-1}, bar^{n-2}
//   [NCCL]    allgather bar^n rows (grouped broadcast, unequal shards)
//   k_gram    per-block Gram partials of bar^n and X_ext^{n+1}
//   k_sweep   one CSR pass: S bar^n, S X_ext^{n+1}, <S bar^n_i, bar^n_i>
//   k_rowsum  per-block merge partials
//   k_combine ordered block combine (cross-shard: ordered NCCL send/recv chain)
//   k_finalize loss, stop rule, trace record, plan of iteration n+1
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <condition_variable>
#include <mutex>
#include <sys/mman.h>
#include <unordered_map>
#include <vector>

#include "fc_internal.h"
#include "fc_kernels.cuh"
#include "fc_transport.h"
#include "fuzzyclust_cuda.h"

extern "C" int fc_generate_graph_impl(const fc_graph_spec* spec, uint64_t* nnz_out, int64_t** row_ptr_out,
                                      uint32_t** col_idx_out, std::string* err);

using namespace fc;

namespace {

thread_local std::string g_thread_err;

// FC_TRACE_HOST=1: print host-side phase timings (stderr).
struct HostPhase {
    const char* name;
    std::chrono::steady_clock::time_point t0;
    static bool on() {
        static const bool v = [] { const char* e = std::getenv("FC_TRACE_HOST"); return e && *e == '1'; }();
        return v;
    }
    explicit HostPhase(const char* n) : name(n), t0(std::chrono::steady_clock::now()) { nvtxRangePushA(n); }
    ~HostPhase() {
        nvtxRangePop();
        if (on())
            std::fprintf(stderr, "[fc] %-22s %8.2f ms\n", name,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

struct Shard {
    uint64_t row0 = 0, nrows = 0;      // global rows [row0, row0 + nrows)
    uint64_t lrow = 0;                 // first row in this device's local row arrays
    uint64_t lblk = 0, nblk = 0;       // local block offset / count
};

enum { kClsStep, kClsGram, kClsSweep, kClsRowsum, kClsCombine, kClsFinalize, kClsComm, kClsPack, kNumCls };

struct CopyPool {
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, done;
    uint64_t gen = 0;
    int pending = 0, nthreads = 1;
    bool stop = false;
    char* dst = nullptr;
    const char* src = nullptr;
    size_t bytes = 0;
    void start(int n);
    void run(int i);
    void copy(void* d, const void* s, size_t b);
    ~CopyPool();
};

}  // namespace

struct fc_ctx {
    int device = 0, rank = 0, world = 1, vshards = 1;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;       // Gram next to the sweep (independent within an iteration)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    bool overlap = false;              // FC_OVERLAP=1: Gram on a side stream (measured: no gain)
    int gram_ctas = 0;                 // FC_GRAM_CTAS: persistent Gram grid (0: overlap2 x SMs, x 3/4 at C > 16)
    int overlap2 = 1;                  // persistent Gram (k CTAs per SM) launched before the sweep on a side
                                       // stream (default k = 1; FC_OVERLAP=0 disables, =2:k sets k)
    fc::Transport* xport = nullptr;    // multi-rank collectives (NCCL or in-process loopback); null = one rank
    int sm_count = 148;
    std::string err;
    std::atomic<uint64_t> launches{0};

    // similarity
    bool have_csr = false;
    uint64_t n = 0, nnz = 0;
    double frob_s = 0.0;
    bool weighted = false;
    std::vector<uint64_t> bounds;      // world+1 (or vshards+1) row bounds
    std::vector<Shard> shards;         // shards resident on this device
    uint64_t local_rows = 0, local_blocks = 0;
    long long* d_row_ptr = nullptr;
    unsigned* d_col = nullptr;
    double* d_val = nullptr;
    uint64_t local_nnz = 0;
    unsigned* d_deg = nullptr;         // degree of every node (hot-row selection)
    std::vector<uint64_t> deg_hist;    // nodes per degree value
    unsigned hot_threshold = 0xFFFFFFFFu;

    // work buffers
    uint32_t c = 0;
    bool bt_alloc = false;
    double* d_U[3] = {nullptr, nullptr, nullptr};
    double* d_xs[4] = {nullptr, nullptr, nullptr, nullptr};
    double* d_prod = nullptr;
    double* d_rowterm[3] = {nullptr, nullptr, nullptr};
    double* d_gpart[2] = {nullptr, nullptr};
    double* d_spart = nullptr;
    double* d_totals = nullptr;        // (vshards + 1) slots
    double* d_chain_in = nullptr;
    char* d_rows_scratch = nullptr;    // fc_gradient_rows / fc_loss_terms_rows staging
    // halo exchange (multi-rank, locality graphs): only the rows a peer's shard references
    bool halo = false;
    int halo_mode = -1;                // FC_HALO: 0 off, 1 on, -1 auto (when it moves < half the allgather)
    std::vector<uint64_t> halo_send_off, halo_recv_off, halo_peer_off;   // doubles, world + 1 (peer: world)
    unsigned* d_halo_send_rows = nullptr;   // own rows to pack, grouped by destination
    unsigned* d_halo_recv_rows = nullptr;   // peer rows to unpack, grouped by source
    uint64_t halo_send_n = 0, halo_recv_n = 0;
    std::vector<uint64_t> halo_send_rows_off, halo_recv_rows_off;         // rows, world + 1
    double* d_halo_send = nullptr;
    double* d_halo_recv = nullptr;
    uint64_t halo_rows_total = 0;      // rows this rank receives per exchange (diagnostics)
    double* d_gfull[2] = {nullptr, nullptr};
    unsigned* d_counter = nullptr;    // [0, 64): row-chunk schedulers per shard; [64, 128): heavy-row schedulers
    unsigned* d_heavy = nullptr;      // per shard: local rows of degree >= heavy_deg, by degree descending
    std::vector<uint64_t> heavy_off, heavy_cnt;
    unsigned heavy_deg = 1024;
    DevState* d_state = nullptr;
    DevState* h_state = nullptr;       // pinned mirror
    int* h_done = nullptr;             // pinned, 2 slots
    TraceRec* d_trace = nullptr;
    uint64_t trace_alloc = 0;

    // solver session
    bool session = false;
    int method = 0;
    uint64_t max_iter = 0;
    uint64_t enqueued = 0;             // iterations enqueued after begin
    uint64_t host_iter = 0;            // FISTA/GPA iteration index of the next enqueued pass
    uint64_t bt_max_host = 0;          // session's backtracking cap (pass budget of fc_solve)
    int ag_buf = -1;                   // multi-rank backtracking: replica the next pass allgathers (device plan)
    bool stop_seen = false;            // multi-rank backtracking: the device reported done
    unsigned long long csr_fp = 0;     // fingerprint of the resident shard CSR
    cudaEvent_t chunk_ev[2] = {nullptr, nullptr};

    bool sweep_tma = false;            // FC_SWEEP=tma selects the TMA gather4 sweep
    bool sweep_groups = false;       // FC_SWEEP=groups: per-group row sweep for C <= 16
    bool step_big = false;             // FC_STEP=big: thread-per-row k_step_big for C > 32
    bool fuse_gram = false;            // FC_FUSE=1: fused k_step_gram for C <= 32 FISTA (measured slower: 8.5 vs 8.2 ms at C)
    bool tol = false;                  // fc_set_parity_mode(1): tolerance mode (FMA, single-gather FISTA)
    bool step_t2 = false;              // FC_STEP=t2 / t2x: two-tile k_step_t2 (EXACT / runtime-C template)
    bool step_t2_inexact = false;
    bool step_inexact = false;         // FC_STEP=tx: k_step_t with the runtime-C template at C == G
    bool pair_sweep = false;           // FC_PAIR=1: C <= 8 dual sweep gathers interleaved [bar | prev] rows
    int sweep_async = 0;               // FC_ASYNC=3|4|6: the PAIR sweep through a cp.async ring of S stages
                                       // (measured E8: 6.34 incl. pack vs 6.41 ms -- within noise, off)
    double* d_pair = nullptr;          // C <= 8: interleaved [bar | prev] rows, N x 2C
    bool step_wide2 = true;            // FC_STEP=wide1: the round-1 k_step_wide (G streamed) for 32 < C <= 128
    bool umaps_ok = false;
    UMaps umaps;                       // tensor maps of U[0..2] (TMA gather4)

    // pinned staging ring for large host<->device copies
    static constexpr int kStageBufs = 3;
    static constexpr size_t kStageChunk = size_t(64) << 20;
    char* stage_buf[kStageBufs] = {nullptr, nullptr, nullptr};
    cudaEvent_t stage_ev[kStageBufs] = {nullptr, nullptr, nullptr};
    int copy_threads = 8;
    CopyPool pool;                     // persistent host-copy workers of the staging ring
    // one captured iteration (CUDA graph), replayed while the key (every kernel argument) matches
    cudaGraphExec_t iter_exec = nullptr;
    std::vector<char> iter_key;
    uint64_t iter_launches = 0;
    bool graphs = true;                // FC_GRAPHS=0 disables

    std::unordered_map<const void*, size_t> caps;   // device allocation capacities (bytes)

    // profiling
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_events;
    double prof_ms[kNumCls] = {0};
    uint64_t prof_n[kNumCls] = {0};
    std::vector<cudaEvent_t> ev_pool;
};

namespace {

int set_err(fc_ctx* ctx, int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    g_thread_err = buf;
    return code;
}

#define CU(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return set_err(ctx, FC_DEVICE, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), \
                           __FILE__, __LINE__, #call);                                     \
    } while (0)

#define NC(call)                                                                           \
    do {                                                                                   \
        ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess)                                                             \
            return set_err(ctx, FC_DEVICE, "NCCL error %s at %s:%d", ncclGetErrorString(r_), \
                           __FILE__, __LINE__);                                            \
    } while (0)

#define XP(call)                                              \
    do {                                                      \
        int rc_ = (call);                                     \
        if (rc_) return set_err(ctx, rc_, "%s", ctx->err.c_str()); \
    } while (0)

#define TRY(expr)                  \
    do {                           \
        int rc_ = (expr);          \
        if (rc_) return rc_;       \
    } while (0)

// Capacity-based device allocation: an existing buffer is reused whenever it is
// large enough (cudaFree synchronizes the device and returns memory to the
// driver, so re-uploads and new solves must not churn multi-GB allocations).
template <class T>
int dalloc(fc_ctx* ctx, T** p, size_t count) {
    if (count == 0) count = 1;
    const size_t bytes = count * sizeof(T);
    size_t& cap = ctx->caps[(const void*)p];
    if (*p && cap >= bytes) return FC_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    cap = 0;
    CU(cudaMalloc(reinterpret_cast<void**>(p), bytes));
    cap = bytes;
    return FC_OK;
}

template <class T>
void dfree(fc_ctx* ctx, T** p) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    ctx->caps[(const void*)p] = 0;
}

// ---- kernel-class timing ------------------------------------------------------
// NVTX range per phase (header-only nvtx3; free when no tool is attached): the phase
// names show up as ranges in a timeline profiler around the kernels they enqueue.
static const char* const kClsName[] = {"fc:step", "fc:gram", "fc:sweep", "fc:rowsum",
                                       "fc:combine", "fc:finalize", "fc:comm", "fc:pack"};

struct ProfScope {
    fc_ctx* ctx;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(fc_ctx* c, int k) : ctx(c), cls(k) {
        nvtxRangePushA(kClsName[k]);
        if (!ctx->profiling) return;
        if (ctx->ev_pool.size() < 2) {
            for (int i = 0; i < 64; ++i) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                ctx->ev_pool.push_back(e);
            }
        }
        a = ctx->ev_pool.back(); ctx->ev_pool.pop_back();
        b = ctx->ev_pool.back(); ctx->ev_pool.pop_back();
        cudaEventRecord(a, ctx->stream);
    }
    ~ProfScope() {
        nvtxRangePop();
        if (!ctx->profiling) return;
        cudaEventRecord(b, ctx->stream);
        ctx->prof_events.push_back({cls, {a, b}});
    }
};

void prof_harvest(fc_ctx* ctx) {
    for (auto& e : ctx->prof_events) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, e.second.first, e.second.second) == cudaSuccess) {
            ctx->prof_ms[e.first] += ms;
            ctx->prof_n[e.first] += 1;
        }
        ctx->ev_pool.push_back(e.second.first);
        ctx->ev_pool.push_back(e.second.second);
    }
    ctx->prof_events.clear();
}

// ---- dispatch by cluster count -------------------------------------------------
template <template <int, int> class F, class... A>
int by_c(fc_ctx* ctx, uint32_t c, A&&... a) {
    if (c <= 2) return F<2, 1>::run(a...);
    if (c <= 4) return F<4, 1>::run(a...);
    if (c <= 8) return F<8, 1>::run(a...);
    if (c <= 16) return F<16, 1>::run(a...);
    if (c <= 32) return F<32, 1>::run(a...);
    if (c <= 64) return F<32, 2>::run(a...);
    if (c <= 128) return F<32, 4>::run(a...);
    if (c <= 256) return F<32, 8>::run(a...);
    return set_err(ctx, FC_INVALID, "cluster count C=%u exceeds the supported maximum 256", c);
}

// Launch-configuration caches are per device: cudaFuncSetAttribute applies to the
// current device, and a process may drive several contexts on several GPUs.
template <class T>
struct PerDevice {
    T v[64] = {};
    T& operator()(const fc_ctx* ctx) { return v[ctx->device & 63]; }
};

int grid_for(const void* fn, int threads, size_t smem, int sm_count) {
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1) occ = 1;
    return occ * sm_count;
}

template <int G, int S, bool DUAL, bool W, bool EXACT>
int launch_sweep_t(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    if (!grid) grid = grid_for((const void*)k_sweep<G, S, DUAL, W, EXACT>, 256, 0, ctx->sm_count);
    const unsigned long long need = (g.nrows + g.chunk - 1) / g.chunk;   // row chunks, 8 warps per CTA
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, (need + 7) / 8));
    k_sweep<G, S, DUAL, W, EXACT><<<gr, 256, 0, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_sweep launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int S, bool DUAL>
int launch_sweep_tma(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = sweep_tma_smem((int)g.C, DUAL ? 1 : 0);
    static PerDevice<size_t> smem_set_pd;
    size_t& smem_set = smem_set_pd(ctx);
    if (smem > smem_set) {
        CU(cudaFuncSetAttribute(k_sweep_tma<S, DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
        grid = grid_for((const void*)k_sweep_tma<S, DUAL>, kSwTmaThreads, smem, ctx->sm_count);
    }
    const unsigned long long need = (g.nrows + 31) / 32;
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, (need + 3) / 4));
    k_sweep_tma<S, DUAL><<<gr, kSwTmaThreads, smem, ctx->stream>>>(b, g, ctx->umaps);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_sweep_tma launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, bool DUAL, bool W>
int launch_sweep_small(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    if (!grid) grid = grid_for((const void*)k_sweep_small<G, DUAL, W>, 256, 0, ctx->sm_count);
    const unsigned long long need = (g.nrows + g.chunk - 1) / g.chunk;
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, (need + 7) / 8));
    k_sweep_small<G, DUAL, W><<<gr, 256, 0, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_sweep_small launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, bool W>
int launch_sweep_small_pair(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    if (!grid) grid = grid_for((const void*)k_sweep_small_pair<G, W>, 256, 0, ctx->sm_count);
    k_sweep_small_pair<G, W><<<grid, 256, 0, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_sweep_small_pair launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, bool W, int S>
int launch_sweep_async(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    constexpr int U = G < 8 ? G : 8;
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = sizeof(SweepRing<G, W, S, U>) * (128 / G);
    if (!grid) {
        CU(cudaFuncSetAttribute(k_sweep_async<G, W, S, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_sweep_async<G, W, S, U>, 128, smem, ctx->sm_count);
    }
    k_sweep_async<G, W, S, U><<<grid, 128, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_sweep_async launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, int S>
struct LaunchSweep {
    static int run(fc_ctx* ctx, const Bufs& b, const Geo& g, bool dual) {
        if (g.nrows == 0) return FC_OK;
        if constexpr (G <= 8) {   // measured: C=8 9.5 vs 12.2 ms (E8); C=16 keeps the group sweep (B: 1.52 vs 1.78 ms)
            if (!ctx->sweep_groups) {
                const bool w = ctx->weighted;
                if (dual && b.pair && ctx->sweep_async) {
                    if constexpr (G == 8) {
                        if (ctx->sweep_async == 3)
                            return w ? launch_sweep_async<G, true, 3>(ctx, b, g) : launch_sweep_async<G, false, 3>(ctx, b, g);
                        if (ctx->sweep_async == 6)
                            return w ? launch_sweep_async<G, true, 6>(ctx, b, g) : launch_sweep_async<G, false, 6>(ctx, b, g);
                    }
                    return w ? launch_sweep_async<G, true, 4>(ctx, b, g) : launch_sweep_async<G, false, 4>(ctx, b, g);
                }
                if (dual && b.pair)
                    return w ? launch_sweep_small_pair<G, true>(ctx, b, g) : launch_sweep_small_pair<G, false>(ctx, b, g);
                if (dual) return w ? launch_sweep_small<G, true, true>(ctx, b, g) : launch_sweep_small<G, true, false>(ctx, b, g);
                return w ? launch_sweep_small<G, false, true>(ctx, b, g) : launch_sweep_small<G, false, false>(ctx, b, g);
            }
        }
        if (G == 32 && g.C > 16 && (g.C % 4) == 0 && !ctx->weighted && ctx->sweep_tma && ctx->umaps_ok) {
            return dual ? launch_sweep_tma<S, true>(ctx, b, g) : launch_sweep_tma<S, false>(ctx, b, g);
        }
        const bool exact = g.C == (unsigned)(G * S);
        const bool w = ctx->weighted;
        if (dual) {
            if (w) return exact ? launch_sweep_t<G, S, true, true, true>(ctx, b, g)
                                : launch_sweep_t<G, S, true, true, false>(ctx, b, g);
            return exact ? launch_sweep_t<G, S, true, false, true>(ctx, b, g)
                         : launch_sweep_t<G, S, true, false, false>(ctx, b, g);
        }
        if (w) return exact ? launch_sweep_t<G, S, false, true, true>(ctx, b, g)
                            : launch_sweep_t<G, S, false, true, false>(ctx, b, g);
        return exact ? launch_sweep_t<G, S, false, false, true>(ctx, b, g)
                     : launch_sweep_t<G, S, false, false, false>(ctx, b, g);
    }
};

template <int G, bool EXACT, bool BT, bool TOL = false>
int launch_step_t(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = step_t_smem(G);
    if (!grid) {
        CU(cudaFuncSetAttribute(k_step_t<G, EXACT, BT, TOL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_step_t<G, EXACT, BT, TOL>, kStepThreads, smem, ctx->sm_count);
    }
    const unsigned long long need = (g.nrows + 32 * (kStepThreads / 32) - 1) / (32 * (kStepThreads / 32));
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, need));
    k_step_t<G, EXACT, BT, TOL><<<gr, kStepThreads, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step_t launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, bool EXACT>
int launch_step_t2(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = step_t2_smem(G);
    if (!grid) {
        CU(cudaFuncSetAttribute(k_step_t2<G, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_step_t2<G, EXACT>, kStepThreads, smem, ctx->sm_count);
    }
    const unsigned long long need = (g.nrows + 32 * (kStepThreads / 32) - 1) / (32 * (kStepThreads / 32));
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, need));
    k_step_t2<G, EXACT><<<gr, kStepThreads, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step_t2 launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, bool EXACT>
int launch_step_gram(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = step_t_smem(G);
    if (!grid) {
        CU(cudaFuncSetAttribute(k_step_gram<G, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_step_gram<G, EXACT>, kStepThreads, smem, ctx->sm_count);
    }
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, g.nblk));
    k_step_gram<G, EXACT><<<gr, kStepThreads, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step_gram launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int CP, bool TOL = false>
int launch_step_wide2(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = Wide2Cfg<CP>::smem();
    if (!grid) {
        CU(cudaFuncSetAttribute(k_step_wide2<CP, TOL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_step_wide2<CP, TOL>, kW2Threads, smem, ctx->sm_count);
    }
    const unsigned long long need = (g.nrows + Wide2Cfg<CP>::R - 1) / Wide2Cfg<CP>::R;
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, need));
    k_step_wide2<CP, TOL><<<gr, kW2Threads, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step_wide2 launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, int S>
struct LaunchStepGram {
    static int run(fc_ctx* ctx, const Bufs& b, const Geo& g) {
        if (g.nrows == 0) return FC_OK;
        if constexpr (S == 1)
            return g.C == (unsigned)G ? launch_step_gram<G, true>(ctx, b, g) : launch_step_gram<G, false>(ctx, b, g);
        return set_err(ctx, FC_INVALID, "k_step_gram: C > 32");
    }
};

template <int CP>
int launch_step_big(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = StepBigCfg<CP>::smem();
    if (!grid) {
        CU(cudaFuncSetAttribute(k_step_big<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_step_big<CP>, kStepBigThreads, smem, ctx->sm_count);
    }
    constexpr int per_cta = StepBigCfg<CP>::RB * (kStepBigThreads / 32);
    const unsigned long long need = (g.nrows + per_cta - 1) / per_cta;
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, need));
    k_step_big<CP><<<gr, kStepBigThreads, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step_big launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int CP>
int launch_step_wide(fc_ctx* ctx, const Bufs& b, const Geo& g) {
    static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
    const size_t smem = WideCfg<CP>::smem();
    if (!grid) {
        CU(cudaFuncSetAttribute(k_step_wide<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        grid = grid_for((const void*)k_step_wide<CP>, kWideThreads, smem, ctx->sm_count);
    }
    const unsigned long long need = (g.nrows + kWideRows - 1) / kWideRows;
    const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, need));
    k_step_wide<CP><<<gr, kWideThreads, smem, ctx->stream>>>(b, g);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step_wide launch: %s", cudaGetErrorString(e));
    return FC_OK;
}

template <int G, int S>
struct LaunchStep {
    static int run(fc_ctx* ctx, const Bufs& b, const Geo& g, int bt) {
        if (g.nrows == 0) return FC_OK;
        if constexpr (S > 1) {
            if (!bt) {
                if constexpr (S <= 4)
                    if (ctx->tol) return launch_step_wide2<32 * S, true>(ctx, b, g);
                if (ctx->step_big) return launch_step_big<32 * S>(ctx, b, g);
                if constexpr (S <= 4)
                    if (ctx->step_wide2) return launch_step_wide2<32 * S>(ctx, b, g);
                return launch_step_wide<32 * S>(ctx, b, g);
            }
        }
        if (S == 1 && (!bt || G <= 16)) {   // thread-per-row projection (+ backtracking row terms;
            // at G = 32 those spill, the lane-parallel k_step below takes bt there)
            if (bt) return g.C == (unsigned)G ? launch_step_t<G, true, true>(ctx, b, g)
                                              : launch_step_t<G, false, true>(ctx, b, g);
            if (ctx->tol)
                return g.C == (unsigned)G ? launch_step_t<G, true, false, true>(ctx, b, g)
                                          : launch_step_t<G, false, false, true>(ctx, b, g);
            if (ctx->step_t2)
                return g.C == (unsigned)G && !ctx->step_t2_inexact ? launch_step_t2<G, true>(ctx, b, g)
                                                                   : launch_step_t2<G, false>(ctx, b, g);
            if (ctx->step_inexact) return launch_step_t<G, false, false>(ctx, b, g);
            return g.C == (unsigned)G ? launch_step_t<G, true, false>(ctx, b, g)
                                      : launch_step_t<G, false, false>(ctx, b, g);
        }
        static PerDevice<int> grid_pd;
    int& grid = grid_pd(ctx);
        if (!grid) grid = grid_for((const void*)k_step<G, S>, 256, 0, ctx->sm_count);
        const unsigned long long need = (g.nrows + (32 / G) * 8 - 1) / ((32 / G) * 8);
        const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(grid, need));
        k_step<G, S><<<gr, 256, 0, ctx->stream>>>(b, g, bt);
        ctx->launches++;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_step launch: %s", cudaGetErrorString(e));
        return FC_OK;
    }
};

template <int G, int S>
struct LaunchProject {
    static int run(fc_ctx* ctx, double* x, unsigned long long rows, int c, unsigned* flag) {
        if (rows == 0) return FC_OK;
        if constexpr (S == 1) {                              // thread per row
            const unsigned long long need = (rows + 127) / 128;
            const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(ctx->sm_count * 8, need));
            if (c == G) k_project_t<G, true><<<gr, 128, 0, ctx->stream>>>(x, rows, c, flag);
            else k_project_t<G, false><<<gr, 128, 0, ctx->stream>>>(x, rows, c, flag);
            ctx->launches++;
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_project_t launch: %s", cudaGetErrorString(e));
            return FC_OK;
        }
        const unsigned long long need = (rows + (32 / G) * 8 - 1) / ((32 / G) * 8);
        const int gr = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(ctx->sm_count * 8, need));
        k_project<G, S><<<gr, 256, 0, ctx->stream>>>(x, rows, c, flag);
        ctx->launches++;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "k_project launch: %s", cudaGetErrorString(e));
        return FC_OK;
    }
};

int check_launch(fc_ctx* ctx, const char* what) {
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(ctx, FC_DEVICE, "%s launch: %s", what, cudaGetErrorString(e));
    return FC_OK;
}

// ---- buffers ----------------------------------------------------------------------
unsigned npairs_of(uint32_t c) { return c * (c + 1) / 2; }
size_t nchains_of(uint32_t c) { return 2 * (size_t)npairs_of(c) + kNumScal; }

int gram_rows_per_chunk(uint32_t c) {
    const int c4 = (int)((c + 3) & ~3u);
    return std::max(4, std::min(16, 512 / c4));
}

// Tensor maps for the TMA gather4 sweep: U[k] as a 2-D [N][C] f64 tensor, box {C, 1}.
int make_umaps(fc_ctx* ctx) {
    ctx->umaps_ok = false;
    const uint32_t c = ctx->c;
    if (c <= 16 || c > 256 || (c % 4)) return FC_OK;   // gather4 destinations: 4*8C bytes, 128-B aligned
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return FC_OK;                                    // TMA variant unavailable: LDG sweep is used
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    for (int k = 0; k < 3; ++k) {
        const cuuint64_t dims[2] = {c, ctx->n};
        const cuuint64_t strides[1] = {(cuuint64_t)c * sizeof(double)};
        const cuuint32_t box[2] = {c, 1};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode(&ctx->umaps.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ctx->d_U[k], dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return FC_OK;
    }
    ctx->umaps_ok = true;
    return FC_OK;
}

// Hot rows: the highest-degree nodes whose two gathered replicas (bar, prev)
// fit the L2 budget FC_HOT_MB (default 40; 0 = off) are loaded with an
// L2::evict_last policy by k_sweep (flag = bit 31 of the stored column index;
// every reader of the column array masks it).  Config C: the top 1.2e5 rows
// take 15% of the gathers; L2 hit 6.2 -> 8.3%, DRAM 196.8 -> 188.9 GB per
// sweep, sweep 29.4 -> 28.2-28.3 ms (30-50 MB; 70 MB: 28.5).
int set_hot_rows(fc_ctx* ctx) {
    double mb = 40.0;
    if (const char* e = std::getenv("FC_HOT_MB")) mb = std::atof(e);
    unsigned thr = 0xFFFFFFFFu;
    if (mb > 0.0 && ctx->deg_hist.empty() && ctx->d_deg) {
        std::vector<unsigned> deg(ctx->n);
        // on the library's (non-blocking) stream: ordered after k_degrees
        CU(cudaMemcpyAsync(deg.data(), ctx->d_deg, ctx->n * sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        const unsigned maxd = deg.empty() ? 0u : *std::max_element(deg.begin(), deg.end());
        ctx->deg_hist.assign((size_t)maxd + 1, 0);
        for (unsigned d : deg) ctx->deg_hist[d]++;
    }
    if (mb > 0.0 && !ctx->deg_hist.empty()) {
        const double rows_budget = mb * 1e6 / (2.0 * 8.0 * ctx->c);
        uint64_t cum = 0;
        for (size_t d = ctx->deg_hist.size(); d-- > 1;) {
            if ((double)(cum + ctx->deg_hist[d]) > rows_budget) break;
            cum += ctx->deg_hist[d];
            thr = (unsigned)d;
        }
    }
    if (thr == ctx->hot_threshold) return FC_OK;
    const unsigned long long nnz = ctx->local_nnz;
    if (nnz) {
        const unsigned blocks = (unsigned)std::min<unsigned long long>((nnz + 255) / 256, (unsigned long long)ctx->sm_count * 16);
        k_flag_hot<<<blocks, 256, 0, ctx->stream>>>(ctx->d_col, nnz, ctx->d_deg, thr);
        TRY(check_launch(ctx, "k_flag_hot"));
    }
    ctx->hot_threshold = thr;
    return FC_OK;
}

int ensure_work(fc_ctx* ctx, uint32_t c, bool bt) {
    if (!ctx->have_csr) return set_err(ctx, FC_INVALID, "no similarity uploaded (call fc_upload_csr first)");
    if (c == 0) return set_err(ctx, FC_INVALID, "init_membership: dimensions must be positive");
    if (c > 256) return set_err(ctx, FC_INVALID, "cluster count C=%u exceeds the supported maximum 256", c);
    if ((unsigned long long)ctx->n * c >= (1ULL << 32))
        return set_err(ctx, FC_INVALID, "N*C = %llu exceeds 2^32 - 1 elements per membership replica",
                       (unsigned long long)ctx->n * c);
    if (ctx->c == c && (!bt || ctx->bt_alloc)) return FC_OK;
    CU(cudaStreamSynchronize(ctx->stream));
    const size_t N = ctx->n, L = ctx->local_rows, LB = ctx->local_blocks;
    for (int k = 0; k < 3; ++k) TRY(dalloc(ctx, &ctx->d_U[k], N * c));
    for (int k = 0; k < 2; ++k) TRY(dalloc(ctx, &ctx->d_xs[k], L * c));
    // backtracking-only buffers are valid (sized for this C) exactly when bt_alloc is set; a
    // non-backtracking re-allocation keeps any older ones allocated but invalid (freeing them
    // here would put a synchronising cudaFree into the next solve), and the checkpoint layout
    // follows the header's flag, not the pointers (for_session_buffers)
    for (int k = 2; k < 4; ++k) {
        if (bt) TRY(dalloc(ctx, &ctx->d_xs[k], L * c));
    }
    TRY(dalloc(ctx, &ctx->d_prod, L));
    if (ctx->pair_sweep && c <= 8) TRY(dalloc(ctx, &ctx->d_pair, N * 2 * c));
    else dfree(ctx, &ctx->d_pair);
    if (ctx->halo) {
        TRY(dalloc(ctx, &ctx->d_halo_send, std::max<uint64_t>(1, ctx->halo_send_n) * c));
        TRY(dalloc(ctx, &ctx->d_halo_recv, std::max<uint64_t>(1, ctx->halo_recv_n) * c));
    }
    for (int k = 0; k < 3; ++k) {
        if (bt) TRY(dalloc(ctx, &ctx->d_rowterm[k], L));
    }
    const unsigned np = npairs_of(c);
    for (int k = 0; k < 2; ++k) TRY(dalloc(ctx, &ctx->d_gpart[k], LB * np));
    TRY(dalloc(ctx, &ctx->d_spart, LB * kNumScal));
    TRY(dalloc(ctx, &ctx->d_totals, (ctx->vshards + 1) * nchains_of(c)));
    TRY(dalloc(ctx, &ctx->d_chain_in, nchains_of(c)));
    for (int k = 0; k < 2; ++k) TRY(dalloc(ctx, &ctx->d_gfull[k], (size_t)c * c));
    CU(cudaMemsetAsync(ctx->d_totals, 0, (ctx->vshards + 1) * nchains_of(c) * sizeof(double), ctx->stream));
    ctx->c = c;
    ctx->bt_alloc = bt;
    TRY(make_umaps(ctx));
    TRY(set_hot_rows(ctx));
    return FC_OK;
}

Bufs make_bufs(fc_ctx* ctx, size_t s) {
    const Shard& sh = ctx->shards[s];
    const uint32_t c = ctx->c;
    const unsigned np = npairs_of(c);
    Bufs b{};
    b.row_ptr = ctx->d_row_ptr + sh.lrow;
    b.col = ctx->d_col;
    b.val = ctx->weighted ? ctx->d_val : nullptr;
    for (int k = 0; k < 3; ++k) b.U[k] = ctx->d_U[k];
    for (int k = 0; k < 4; ++k) b.xs[k] = ctx->d_xs[k] ? ctx->d_xs[k] + sh.lrow * c : nullptr;
    b.prod = ctx->d_prod + sh.lrow;
    for (int k = 0; k < 3; ++k) b.rowterm[k] = ctx->d_rowterm[k] ? ctx->d_rowterm[k] + sh.lrow : nullptr;
    for (int k = 0; k < 2; ++k) b.gpart[k] = ctx->d_gpart[k] + sh.lblk * np;
    b.spart = ctx->d_spart + sh.lblk;
    b.totals = ctx->d_totals + s * nchains_of(c);
    for (int k = 0; k < 2; ++k) b.gfull[k] = ctx->d_gfull[k];
    b.trace = ctx->d_trace;
    b.st = ctx->d_state;
    b.counter = ctx->d_counter + s;
    b.hcounter = ctx->d_counter + 64 + s;
    b.pair = ctx->d_pair;
    b.heavy = ctx->d_heavy ? ctx->d_heavy + ctx->heavy_off[s] : nullptr;
    b.nheavy = ctx->d_heavy ? (unsigned)ctx->heavy_cnt[s] : 0u;
    b.heavy_deg = ctx->heavy_deg;
    return b;
}

Geo make_geo(fc_ctx* ctx, size_t s) {
    const Shard& sh = ctx->shards[s];
    Geo g{};
    g.C = ctx->c;
    g.npairs = npairs_of(ctx->c);
    g.N = ctx->n;
    g.row0 = sh.row0;
    g.nrows = sh.nrows;
    g.nblk = sh.nblk;
    g.spart_stride = ctx->local_blocks;
    // enough counter grabs to occupy every resident warp (~32 per SM) when N is small
    g.chunk = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(32, sh.nrows / ((uint64_t)ctx->sm_count * 32)));
    return g;
}

// final totals slot (what k_finalize reads)
Bufs final_bufs(fc_ctx* ctx) {
    Bufs b = make_bufs(ctx, 0);
    b.totals = ctx->d_totals + (ctx->xport ? 0 : (ctx->shards.size() - 1)) * nchains_of(ctx->c);
    return b;
}

// ---- phases -------------------------------------------------------------------------
int phase_step(fc_ctx* ctx, int bt) {
    ProfScope p(ctx, kClsStep);
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const Bufs b = make_bufs(ctx, s);
        const Geo g = make_geo(ctx, s);
        TRY(by_c<LaunchStep>(ctx, ctx->c, ctx, b, g, bt));
    }
    return FC_OK;
}

// FISTA step + the dual Gram of the new iterate in one pass (C <= 32, no backtracking)
bool fused_step_gram(const fc_ctx* ctx, int bt) { return ctx->fuse_gram && !bt && ctx->c <= 32; }

int phase_step_gram(fc_ctx* ctx) {
    ProfScope p(ctx, kClsStep);
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const Bufs b = make_bufs(ctx, s);
        const Geo g = make_geo(ctx, s);
        TRY(by_c<LaunchStepGram>(ctx, ctx->c, ctx, b, g));
    }
    return FC_OK;
}

int phase_gram(fc_ctx* ctx, bool dual, cudaStream_t strm = nullptr, unsigned max_ctas = 0) {
    if (!strm) strm = ctx->stream;
    ProfScope p(ctx, kClsGram);
    const uint32_t c = ctx->c;
    // few 1024-row blocks (small N): one thread per (r, s) pair, larger chunks (fewer barriers)
    const bool few = ctx->local_blocks < (uint64_t)ctx->sm_count * 2;
    // 8x8 tiles from C = 64 (fewer shared loads per FP64 pair, and one CTA covers all
    // tiles of a block instead of re-staging its rows for several tile groups)
    // tile shape TR x TC; FC_GRAM_TS = 1 | 4 | 8 (square) | 48 (4 x 8)
    int TS = few ? 1 : (c >= 64 ? 8 : 4);
    if (const char* e = std::getenv("FC_GRAM_TS")) {
        const int v = std::atoi(e);
        if (v == 1 || v == 4 || v == 8 || v == 48) TS = v;
    }
    const int TR = TS == 48 ? 4 : TS, TC = TS == 48 ? 8 : TS;
    const int tiles = gram_tiles((int)c, TR, TC) * (dual ? 2 : 1);
    int R = gram_rows_per_chunk(c);
    if (few) R = std::max(R, std::min(128, 4096 / (int)((c + 3) & ~3u)));
    if (TC == 8) R = std::max(8, std::min(16, 2048 / (int)((c + 7) & ~7u)));
    if (const char* e = std::getenv("FC_GRAM_R")) R = std::max(1, std::min(128, std::atoi(e)));
    const size_t smem = gram_smem((int)c, dual ? 1 : 0, R, std::max(TR, TC));
    static PerDevice<size_t[128]> smem_set_pd;
    size_t (&smem_set)[128] = smem_set_pd(ctx);
    auto pick = [&](auto tol) {
        constexpr bool T = decltype(tol)::value;
        return TS == 1 ? k_gram<1, 1, T> : TS == 8 ? k_gram<8, 8, T> : TS == 48 ? k_gram<4, 8, T> : k_gram<4, 4, T>;
    };
    auto kfn = ctx->tol ? pick(std::true_type{}) : pick(std::false_type{});
    const int sidx = (TS % 64) + (ctx->tol ? 64 : 0);
    if (smem > 48 * 1024 && smem > smem_set[sidx]) {
        CU(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set[sidx] = smem;
    }
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const Geo g = make_geo(ctx, s);
        if (g.nblk == 0) continue;
        const Bufs b = make_bufs(ctx, s);
        const int threads = std::min(kGramMaxThreads, (tiles + 31) / 32 * 32);
        const unsigned gx = max_ctas ? (unsigned)std::min<unsigned long long>(g.nblk, max_ctas) : (unsigned)g.nblk;
        dim3 grid(gx, (unsigned)((tiles + threads - 1) / threads));
        kfn<<<grid, threads, smem, strm>>>(b, g, dual ? 1 : 0, R);
        TRY(check_launch(ctx, "k_gram"));
    }
    return FC_OK;
}

int phase_sweep(fc_ctx* ctx, bool dual) {
    ProfScope p(ctx, kClsSweep);
    CU(cudaMemsetAsync(ctx->d_counter, 0, ctx->shards.size() * sizeof(unsigned), ctx->stream));
    CU(cudaMemsetAsync(ctx->d_counter + 64, 0, ctx->shards.size() * sizeof(unsigned), ctx->stream));
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const Bufs b = make_bufs(ctx, s);
        const Geo g = make_geo(ctx, s);
        TRY(by_c<LaunchSweep>(ctx, ctx->c, ctx, b, g, dual));
    }
    return FC_OK;
}

int phase_rowsum(fc_ctx* ctx, int bt) {
    ProfScope p(ctx, kClsRowsum);
    const int nscal = bt ? 4 : 1;
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const Geo g = make_geo(ctx, s);
        if (g.nblk == 0) continue;
        const Bufs b = make_bufs(ctx, s);
        const unsigned long long total = g.nblk * (unsigned long long)nscal;
        k_rowsum<<<(unsigned)total, kRowsumThreads, 0, ctx->stream>>>(
            b, g, nscal, b.prod, bt ? b.rowterm[0] : nullptr, bt ? b.rowterm[1] : nullptr,
            bt ? b.rowterm[2] : nullptr, kScalMerge);
        TRY(check_launch(ctx, "k_rowsum"));
    }
    return FC_OK;
}

// Ordered combine.  Shards on this device chain through the totals slots;
// ranks chain through NCCL recv(rank-1) / send(rank+1), then the last rank
// broadcasts the final totals.
int phase_combine(fc_ctx* ctx, int mat_mask, int scal_mask) {
    const size_t nch = nchains_of(ctx->c);
    const int threads = kCombThreads;
    const int blocks = (int)((2 * npairs_of(ctx->c) + 31) / 32) + kNumScal;
    if (!ctx->xport) {
        ProfScope p(ctx, kClsCombine);
        for (size_t s = 0; s < ctx->shards.size(); ++s) {
            const Bufs b = make_bufs(ctx, s);
            const Geo g = make_geo(ctx, s);
            const double* init = s == 0 ? nullptr : ctx->d_totals + (s - 1) * nch;
            k_combine<<<blocks, threads, kCombSmem, ctx->stream>>>(b, g, mat_mask, scal_mask, init);
            TRY(check_launch(ctx, "k_combine"));
        }
        return FC_OK;
    }
    if (ctx->rank > 0) {
        ProfScope p(ctx, kClsComm);
        XP(ctx->xport->recv_prev(ctx->d_chain_in, nch, ctx->stream, &ctx->err));
    }
    {
        ProfScope p(ctx, kClsCombine);
        const Bufs b = make_bufs(ctx, 0);
        const Geo g = make_geo(ctx, 0);
        k_combine<<<blocks, threads, kCombSmem, ctx->stream>>>(b, g, mat_mask, scal_mask,
                                                       ctx->rank > 0 ? ctx->d_chain_in : nullptr);
        TRY(check_launch(ctx, "k_combine"));
    }
    ProfScope p(ctx, kClsComm);
    if (ctx->rank < ctx->world - 1) XP(ctx->xport->send_next(ctx->d_totals, nch, ctx->stream, &ctx->err));
    XP(ctx->xport->bcast_last(ctx->d_totals, nch, ctx->stream, &ctx->err));
    return FC_OK;
}

int phase_finalize(fc_ctx* ctx, int kind, int mat_mask) {
    ProfScope p(ctx, kClsFinalize);
    Bufs b = final_bufs(ctx);
    Geo g = make_geo(ctx, 0);
    k_finalize<<<1, 256, 0, ctx->stream>>>(b, g, kind, mat_mask);
    return check_launch(ctx, "k_finalize");
}

// allgather of the rows of U[buf] each rank owns (NCCL contexts only)
int phase_halo(fc_ctx* ctx, int buf) {
    ProfScope p(ctx, kClsComm);
    const uint32_t c = ctx->c;
    const unsigned blocks = (unsigned)ctx->sm_count * 4;
    if (ctx->halo_send_n) {
        k_halo_pack<<<blocks, 256, 0, ctx->stream>>>(ctx->d_U[buf], ctx->d_halo_send_rows, ctx->halo_send_n, c,
                                                      ctx->d_halo_send);
        TRY(check_launch(ctx, "k_halo_pack"));
    }
    std::vector<uint64_t> so(ctx->world + 1), ro(ctx->world + 1), po(ctx->world);
    for (int r = 0; r <= ctx->world; ++r) {
        so[r] = ctx->halo_send_rows_off[r] * c;
        ro[r] = ctx->halo_recv_rows_off[r] * c;
    }
    for (int r = 0; r < ctx->world; ++r) po[r] = ctx->halo_peer_off[r] * c;
    XP(ctx->xport->exchange(ctx->d_halo_send, so.data(), ctx->d_halo_recv, ro.data(), po.data(), ctx->stream,
                            &ctx->err));
    if (ctx->halo_recv_n) {
        k_halo_unpack<<<blocks, 256, 0, ctx->stream>>>(ctx->d_halo_recv, ctx->d_halo_recv_rows, ctx->halo_recv_n, c,
                                                        ctx->d_U[buf]);
        TRY(check_launch(ctx, "k_halo_unpack"));
    }
    return FC_OK;
}

int phase_allgather(fc_ctx* ctx, int buf, bool full = false) {
    if (!ctx->xport) return FC_OK;
    if (ctx->halo && !full) return phase_halo(ctx, buf);
    ProfScope p(ctx, kClsComm);
    XP(ctx->xport->allgather_rows(ctx->d_U[buf], ctx->bounds.data(), ctx->c, ctx->stream, &ctx->err));
    return FC_OK;
}

int enqueue_prelude(fc_ctx* ctx) {   // FISTA loss at x0 (solver.hpp:206-212)
    TRY(phase_gram(ctx, false));
    TRY(phase_sweep(ctx, false));
    TRY(phase_rowsum(ctx, 0));
    TRY(phase_combine(ctx, 1, 1));
    TRY(phase_finalize(ctx, kFinPrelude, 1));
    return FC_OK;
}

// C <= 8 dual sweep: interleave the (exchanged) bar^n and bar^{n-1} rows for the PAIR gather.
int phase_pair_pack(fc_ctx* ctx) {
    if (!ctx->d_pair) return FC_OK;
    ProfScope p(ctx, kClsPack);
    const Bufs b = make_bufs(ctx, 0);
    const Geo g = make_geo(ctx, 0);
    k_pair_pack<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(b, g);
    return check_launch(ctx, "k_pair_pack");
}

// After the step: the exchange of the new rows, the Gram partials of the new iterate (and of
// the next extrapolated point) and the sweep.  The Gram reads only this rank's rows, so by
// default (FC_OVERLAP unset or 2[:k]) it runs as a persistent grid (k CTAs per SM) on a side
// stream, launched first: concurrent with the row exchange (NCCL / loopback copies) and with
// the HBM-bound sweep, whose memory stalls its FP64 work fills.  FC_OVERLAP=1: the round-1
// variant (Gram launched after the sweep); FC_OVERLAP=0: sequential.
static int exchange_gram_sweep(fc_ctx* ctx, int buf, bool dual_sweep) {
    if (ctx->overlap2 && !ctx->profiling) {
        CU(cudaEventRecord(ctx->fork_ev, ctx->stream));
        CU(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
        // C > 16: three quarters of the SMs, so the others keep the whole G = 32 sweep (a
        // Gram CTA displaces one of its three CTAs where it lands; measured C 38.1-38.4 ->
        // 37.1-37.7 ms, E128 94.3 -> 87.1 ms).  C <= 16 (k_sweep_small, G = 16 sweep): every
        // SM (B 3.04-3.09 vs 2.81-2.87 ms, E8 6.83-6.94 vs 6.57-6.67 ms with all SMs).
        const unsigned per = (unsigned)(ctx->sm_count * ctx->overlap2);
        const unsigned gctas = ctx->gram_ctas ? (unsigned)ctx->gram_ctas
                                              : ctx->c > 16 ? std::max(1u, per * 3 / 4) : per;
        TRY(phase_gram(ctx, true, ctx->side, gctas));
        TRY(phase_allgather(ctx, buf));
        if (dual_sweep) TRY(phase_pair_pack(ctx));
        TRY(phase_sweep(ctx, dual_sweep));
        CU(cudaEventRecord(ctx->join_ev, ctx->side));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
        return FC_OK;
    }
    TRY(phase_allgather(ctx, buf));
    if (dual_sweep) TRY(phase_pair_pack(ctx));
    if (ctx->overlap && !ctx->xport && !ctx->profiling) {
        CU(cudaEventRecord(ctx->fork_ev, ctx->stream));
        CU(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
        TRY(phase_sweep(ctx, dual_sweep));
        TRY(phase_gram(ctx, true, ctx->side));
        CU(cudaEventRecord(ctx->join_ev, ctx->side));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
        return FC_OK;
    }
    TRY(phase_gram(ctx, true));
    return phase_sweep(ctx, dual_sweep);
}

int enqueue_fista_iteration(fc_ctx* ctx, int bt) {
    const int buf = ctx->ag_buf >= 0 ? ctx->ag_buf : (int)(ctx->host_iter % 3);
    if (!ctx->tol && fused_step_gram(ctx, bt)) {
        TRY(phase_step_gram(ctx));
        TRY(phase_allgather(ctx, buf));
        TRY(phase_pair_pack(ctx));
        TRY(phase_sweep(ctx, true));
    } else {
        // tolerance mode: single-gather sweep (S X_ext by linearity in the next step)
        TRY(phase_step(ctx, ctx->tol ? 0 : bt));
        TRY(exchange_gram_sweep(ctx, buf, !ctx->tol));
    }
    TRY(phase_rowsum(ctx, bt));
    TRY(phase_combine(ctx, 3, bt ? 0xF : 1));
    TRY(phase_finalize(ctx, kFinFista, 3));
    ctx->host_iter++;
    return FC_OK;
}

int enqueue_gpa_iteration(fc_ctx* ctx) {
    TRY(phase_gram(ctx, false));
    TRY(phase_sweep(ctx, false));
    TRY(phase_rowsum(ctx, 0));
    TRY(phase_combine(ctx, 1, 1));
    TRY(phase_finalize(ctx, kFinGpa, 1));
    TRY(phase_step(ctx, 0));
    TRY(phase_allgather(ctx, (int)((ctx->host_iter + 1) % 2)));
    ctx->host_iter++;
    return FC_OK;
}

int upload_state(fc_ctx* ctx, const DevState& s) {
    // h_state is the pinned source of the async copy: a previous upload still queued
    // on the stream would read the new contents, so drain the stream first
    CU(cudaStreamSynchronize(ctx->stream));
    *ctx->h_state = s;
    CU(cudaMemcpyAsync(ctx->d_state, ctx->h_state, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));
    return FC_OK;
}

int download_state(fc_ctx* ctx) {
    CU(cudaMemcpyAsync(ctx->h_state, ctx->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return FC_OK;
}

DevState base_state(fc_ctx* ctx) {
    DevState s;
    std::memset(&s, 0, sizeof s);
    s.frob_s = ctx->frob_s;
    s.trace_cap = ctx->trace_alloc;
    s.trace_every = 1;
    s.max_iter = 1;
    return s;
}

int h2d(fc_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return FC_OK;
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return FC_OK;
}

int d2h(fc_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return FC_OK;
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    return FC_OK;
}

// ---- large host<->device copies through a pinned staging ring ----------------------
// Pageable cudaMemcpy moves data through one driver thread; here the host side
// of each 64 MB chunk is copied by several threads into pinned memory while the
// previous chunk's DMA runs.
// Host copies of the staging ring through persistent workers (spawning threads per
// 64 MB chunk cost ~10% of a multi-GB transfer).  The caller takes part 0.
void CopyPool::start(int n) {
    if (!th.empty() || n <= 1) return;
    nthreads = n;
    for (int i = 1; i < n; ++i) th.emplace_back([this, i] { run(i); });
}
void CopyPool::run(int i) {
    uint64_t seen = 0;
    for (;;) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        char* d = dst;
        const char* s2 = src;
        const size_t b = bytes, part = (bytes + nthreads - 1) / nthreads;
        lk.unlock();
        const size_t a = std::min(b, (size_t)i * part), e = std::min(b, a + part);
        if (e > a) std::memcpy(d + a, s2 + a, e - a);
        lk.lock();
        if (--pending == 0) done.notify_one();
    }
}
void CopyPool::copy(void* d, const void* s2, size_t b) {
    if (th.empty() || b < (size_t(4) << 20)) {
        std::memcpy(d, s2, b);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        dst = (char*)d;
        src = (const char*)s2;
        bytes = b;
        pending = nthreads - 1;
        ++gen;
    }
    cv.notify_all();
    const size_t part = (b + nthreads - 1) / nthreads;
    std::memcpy(d, s2, std::min(b, part));
    std::unique_lock<std::mutex> lk(mu);
    done.wait(lk, [&] { return pending == 0; });
}
CopyPool::~CopyPool() {
    {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
}

int ensure_staging(fc_ctx* ctx) {
    ctx->pool.start(ctx->copy_threads);
    for (int k = 0; k < fc_ctx::kStageBufs; ++k) {
        if (!ctx->stage_buf[k]) CU(cudaMallocHost(reinterpret_cast<void**>(&ctx->stage_buf[k]), fc_ctx::kStageChunk));
        if (!ctx->stage_ev[k]) CU(cudaEventCreateWithFlags(&ctx->stage_ev[k], cudaEventDisableTiming));
    }
    return FC_OK;
}

// Page-locked (cudaHostAlloc / registered / torch pin_memory) host memory is DMA'd
// directly at full link speed; pageable memory goes through the staging ring.
bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Returns once `src` has been consumed (the DMA may still be in flight, stream-ordered).
// defer_pinned: a page-locked source is only enqueued -- the caller synchronises the
// stream before it returns to its own caller (the upload overlaps its host work).
int h2d_big(fc_ctx* ctx, void* dst, const void* src, size_t bytes, bool defer_pinned = false) {
    if (bytes < (size_t(8) << 20)) return h2d(ctx, dst, src, bytes);
    if (host_pinned(src)) {
        CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        if (!defer_pinned) CU(cudaStreamSynchronize(ctx->stream));
        return FC_OK;
    }
    TRY(ensure_staging(ctx));
    const size_t ch = fc_ctx::kStageChunk;
    int k = 0;
    for (size_t off = 0; off < bytes; off += ch, k = (k + 1) % fc_ctx::kStageBufs) {
        const size_t n = std::min(ch, bytes - off);
        CU(cudaEventSynchronize(ctx->stage_ev[k]));           // buffer k's previous DMA has finished
        ctx->pool.copy(ctx->stage_buf[k], (const char*)src + off, n);
        CU(cudaMemcpyAsync((char*)dst + off, ctx->stage_buf[k], n, cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaEventRecord(ctx->stage_ev[k], ctx->stream));
    }
    return FC_OK;
}

// Large, freshly allocated destinations fault in 4 KB pages as the copy threads touch
// them (~0.1 s for 2.5 GB); ask for transparent huge pages on the aligned interior.
void advise_huge(void* p, size_t bytes) {
    const uintptr_t a = ((uintptr_t)p + (size_t(2) << 20) - 1) & ~((uintptr_t(2) << 20) - 1);
    const uintptr_t b = ((uintptr_t)p + bytes) & ~((uintptr_t(2) << 20) - 1);
    if (b > a) madvise((void*)a, b - a, MADV_HUGEPAGE);
}

// Synchronous: `dst` holds the data on return.
int d2h_big(fc_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes >= (size_t(8) << 20) && host_pinned(dst)) {
        CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        return FC_OK;
    }
    if (bytes >= (size_t(64) << 20)) advise_huge(dst, bytes);
    if (bytes < (size_t(8) << 20)) {
        TRY(d2h(ctx, dst, src, bytes));
        CU(cudaStreamSynchronize(ctx->stream));
        return FC_OK;
    }
    TRY(ensure_staging(ctx));
    const size_t ch = fc_ctx::kStageChunk;
    const size_t nchunks = (bytes + ch - 1) / ch;
    auto issue = [&](size_t i) -> int {
        const int k = (int)(i % fc_ctx::kStageBufs);
        const size_t off = i * ch, n = std::min(ch, bytes - off);
        CU(cudaMemcpyAsync(ctx->stage_buf[k], (const char*)src + off, n, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaEventRecord(ctx->stage_ev[k], ctx->stream));
        return FC_OK;
    };
    for (size_t i = 0; i < nchunks && i < (size_t)fc_ctx::kStageBufs; ++i) TRY(issue(i));
    for (size_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % fc_ctx::kStageBufs);
        const size_t off = i * ch, n = std::min(ch, bytes - off);
        CU(cudaEventSynchronize(ctx->stage_ev[k]));
        ctx->pool.copy((char*)dst + off, ctx->stage_buf[k], n);
        if (i + fc_ctx::kStageBufs < nchunks) TRY(issue(i + fc_ctx::kStageBufs));
    }
    return FC_OK;
}

// x0.validate(1e-9) on the device (membership.hpp:49-61); x already in U[buf]
int validate_x(fc_ctx* ctx, int buf, double tol) {
    DevState s = base_state(ctx);
    TRY(upload_state(ctx, s));
    const unsigned long long n = ctx->n;
    k_validate<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->d_U[buf], n, (int)ctx->c, ctx->d_state);
    TRY(check_launch(ctx, "k_validate"));
    TRY(download_state(ctx));
    if (ctx->h_state->nonfinite) return set_err(ctx, FC_INVALID, "membership: non-finite entry");
    double err;
    const unsigned long long bits = ctx->h_state->err_bits;
    std::memcpy(&err, &bits, sizeof err);
    if (err > tol)
        return set_err(ctx, FC_INVALID, "membership: columns violate the simplex constraint by %g (tolerance %g)",
                       err, tol);
    return FC_OK;
}

int ensure_trace(fc_ctx* ctx, uint64_t records) {
    if (records == 0) records = 1;
    if (ctx->trace_alloc >= records) return FC_OK;
    TRY(dalloc(ctx, &ctx->d_trace, records));
    ctx->trace_alloc = records;
    return FC_OK;
}

bool granular_ok(fc_ctx* ctx) { return ctx->xport == nullptr; }

}  // namespace

cudaStream_t fc_internal_stream(fc_ctx* ctx) { return ctx->stream; }
int fc_internal_device(fc_ctx* ctx) { return ctx->device; }
int fc_internal_fail(fc_ctx* ctx, int code, const std::string& msg) { return set_err(ctx, code, "%s", msg.c_str()); }
extern "C" {
static int upload_csr_impl(fc_ctx*, uint64_t, uint64_t, const int64_t*, const uint32_t*, const double*, double, bool,
                           int);
}
int fc_internal_h2d(fc_ctx* ctx, void* dst, const void* src, size_t bytes) { return h2d_big(ctx, dst, src, bytes); }
int fc_internal_csr(fc_ctx* ctx, uint64_t* n, const long long** row_ptr, const unsigned** col, const double** val) {
    if (!ctx->have_csr) return set_err(ctx, FC_INVALID, "no similarity uploaded (call fc_upload_csr first)");
    if (ctx->xport) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    *n = ctx->n;
    *row_ptr = ctx->d_row_ptr;
    *col = ctx->d_col;
    *val = ctx->weighted ? ctx->d_val : nullptr;
    return FC_OK;
}
int fc_internal_d2h(fc_ctx* ctx, void* dst, const void* src, size_t bytes) { return d2h_big(ctx, dst, src, bytes); }
int fc_internal_adopt_device_csr(fc_ctx* ctx, uint64_t n, uint64_t nnz, const int64_t* h_row_ptr,
                                 const uint32_t* d_col, const double* d_val, double frob_sq) {
    return upload_csr_impl(ctx, n, nnz, h_row_ptr, d_col, d_val, frob_sq, true, d_val ? 1 : 0);
}

// =====================================================================================
extern "C" {

const char* fc_version(void) { return "fuzzyclust-b200 0.1.0 (reference API 0.1.0)"; }
int fc_abi_version(void) { return FC_ABI_VERSION; }

const char* fc_last_error(const fc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_thread_err.c_str(); }

int fc_nccl_unique_id(unsigned char id[128]) {
    fc_ctx* ctx = nullptr;
    ncclUniqueId u;
    NC(ncclGetUniqueId(&u));
    static_assert(sizeof(u.internal) == 128, "nccl id size");
    std::memcpy(id, u.internal, 128);
    return FC_OK;
}

static int create_common(fc_ctx** out, int device, int rank, int world, int vshards, const unsigned char* id,
                         fc_loopback* loop = nullptr) {
    fc_ctx* ctx = nullptr;
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return set_err(nullptr, FC_INVALID, "bad rank/world");
    if (vshards < 1) return set_err(nullptr, FC_INVALID, "shards must be >= 1");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return set_err(nullptr, FC_DEVICE, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return set_err(nullptr, FC_INVALID, "device %d out of range", device);
    ctx = new fc_ctx();
    ctx->device = device;
    ctx->rank = rank;
    ctx->world = world;
    ctx->vshards = vshards;
    *out = ctx;
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(ctx, FC_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a (B200)", device,
                       prop.major, prop.minor);
    ctx->sm_count = prop.multiProcessorCount;
    if (const char* sw = std::getenv("FC_SWEEP")) {
        ctx->sweep_tma = std::strcmp(sw, "tma") == 0;
        ctx->sweep_groups = std::strcmp(sw, "groups") == 0;
    }
    if (const char* sp = std::getenv("FC_STEP")) {
        ctx->step_big = std::strcmp(sp, "big") == 0;
        ctx->step_wide2 = std::strcmp(sp, "wide1") != 0;
        ctx->step_t2 = std::strcmp(sp, "t2") == 0 || std::strcmp(sp, "t2x") == 0;
        ctx->step_t2_inexact = std::strcmp(sp, "t2x") == 0;
        ctx->step_inexact = std::strcmp(sp, "tx") == 0;
    }
    if (const char* fu = std::getenv("FC_FUSE")) ctx->fuse_gram = std::strcmp(fu, "1") == 0;
    if (const char* ha = std::getenv("FC_HALO")) ctx->halo_mode = std::atoi(ha);
    if (const char* pa = std::getenv("FC_PAIR")) ctx->pair_sweep = std::strcmp(pa, "1") == 0;
    if (const char* gc = std::getenv("FC_GRAM_CTAS")) ctx->gram_ctas = std::max(0, std::atoi(gc));
    if (const char* sa = std::getenv("FC_ASYNC")) ctx->sweep_async = std::atoi(sa);
    if (const char* gr = std::getenv("FC_GRAPHS")) ctx->graphs = std::strcmp(gr, "0") != 0;
    {
        const unsigned hw = std::thread::hardware_concurrency();
        ctx->copy_threads = (int)std::max(1u, std::min(8u, hw ? hw / 2 : 1u));
        if (const char* e = std::getenv("FC_COPY_THREADS")) ctx->copy_threads = std::max(1, std::atoi(e));
    }
    CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    if (const char* ov = std::getenv("FC_OVERLAP")) {
        ctx->overlap = std::strcmp(ov, "1") == 0;
        ctx->overlap2 = ov[0] == '2' ? (ov[1] == ':' ? std::max(1, std::atoi(ov + 2)) : 1) : 0;
    }
    CU(cudaMalloc(&ctx->d_state, sizeof(DevState)));
    CU(cudaMallocHost(&ctx->h_state, sizeof(DevState)));
    CU(cudaMallocHost(&ctx->h_done, 2 * sizeof(int)));
    CU(cudaMalloc(&ctx->d_counter, 128 * sizeof(unsigned)));
    if (const char* h = std::getenv("FC_HEAVY_DEG")) ctx->heavy_deg = (unsigned)std::max(1L, std::atol(h));
    CU(cudaEventCreateWithFlags(&ctx->chunk_ev[0], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->chunk_ev[1], cudaEventDisableTiming));
    // FC_FORCE_NCCL=1 with world == 1 and an id: a 1-rank communicator, so the
    // NCCL allgather / ordered-chain code runs on a single GPU (test hook).
    const char* force = std::getenv("FC_FORCE_NCCL");
    if (loop) {
        ctx->xport = new fc::LoopbackTransport(loop, rank);
    } else if (world > 1 || (id && force && *force == '1')) {
        ncclUniqueId u;
        std::memcpy(u.internal, id, 128);
        ncclComm_t comm = nullptr;
        NC(ncclCommInitRank(&comm, world, u, rank));
        ctx->xport = new fc::NcclTransport(comm, rank, world);
    }
    TRY(ensure_trace(ctx, 1024));
    CU(cudaFuncSetAttribute(k_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCombSmem));
    return FC_OK;
}

int fc_create(fc_ctx** out, int device, int rank, int world, const unsigned char* nccl_id) {
    if (world > 1 && !nccl_id) return set_err(nullptr, FC_INVALID, "world > 1 needs an NCCL unique id");
    int rc = create_common(out, device, rank, world, 1, nccl_id);
    if (rc && *out) {
        g_thread_err = (*out)->err;
        fc_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

int fc_loopback_create(fc_loopback** out, int device, int world) {
    fc_ctx* ctx = nullptr;
    *out = nullptr;
    if (world < 1 || world > 64) return set_err(nullptr, FC_INVALID, "loopback: world must be in [1, 64]");
    CU(cudaSetDevice(device));
    auto* g = new fc_loopback();
    g->world = world;
    g->device = device;
    g->slots.resize((size_t)fc_loopback::kKinds * world * fc_loopback::kRing);
    for (auto& sl : g->slots) {
        if (cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming) != cudaSuccess) {
            fc_loopback_destroy(g);
            return set_err(nullptr, FC_DEVICE, "loopback: cudaEventCreate failed");
        }
    }
    if (const char* t = std::getenv("FC_LOOPBACK_TIMEOUT_S")) g->timeout_s = std::max(1.0, std::atof(t));
    *out = g;
    return FC_OK;
}

void fc_loopback_destroy(fc_loopback* g) {
    if (!g) return;
    cudaSetDevice(g->device);
    for (auto& sl : g->slots)
        if (sl.ev) cudaEventDestroy(sl.ev);
    delete g;
}

int fc_create_loopback(fc_ctx** out, fc_loopback* group, int rank) {
    if (!group) return set_err(nullptr, FC_INVALID, "loopback: null group");
    int rc = create_common(out, group->device, rank, group->world, 1, nullptr, group);
    if (rc && *out) {
        g_thread_err = (*out)->err;
        fc_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

int fc_set_parity_mode(fc_ctx* ctx, int mode) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    if (mode != 0 && mode != 1) return set_err(ctx, FC_INVALID, "parity_mode must be 0 (bitwise) or 1 (tolerance)");
    if (ctx->session) return set_err(ctx, FC_INVALID, "parity_mode: a solver session is open");
    ctx->tol = mode == 1;
    return FC_OK;
}

int fc_get_parity_mode(const fc_ctx* ctx) { return ctx && ctx->tol ? 1 : 0; }

int fc_halo_info(const fc_ctx* ctx, uint64_t* recv_rows, uint64_t* send_rows) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    if (recv_rows) *recv_rows = ctx->halo ? ctx->halo_recv_n : 0;
    if (send_rows) *send_rows = ctx->halo ? ctx->halo_send_n : 0;
    return ctx->halo ? 1 : 0;
}

int fc_create_virtual(fc_ctx** out, int device, int shards) {
    if (shards > 32) return set_err(nullptr, FC_INVALID, "at most 32 virtual shards");
    int rc = create_common(out, device, 0, 1, shards, nullptr);
    if (rc && *out) {
        g_thread_err = (*out)->err;
        fc_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

void fc_destroy(fc_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    prof_harvest(ctx);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->iter_exec) cudaGraphExecDestroy(ctx->iter_exec);
    delete ctx->xport;
    for (int k = 0; k < 3; ++k) dfree(ctx, &ctx->d_U[k]);
    for (int k = 0; k < 4; ++k) dfree(ctx, &ctx->d_xs[k]);
    for (int k = 0; k < 3; ++k) dfree(ctx, &ctx->d_rowterm[k]);
    for (int k = 0; k < 2; ++k) { dfree(ctx, &ctx->d_gpart[k]); dfree(ctx, &ctx->d_gfull[k]); }
    dfree(ctx, &ctx->d_prod);
    dfree(ctx, &ctx->d_spart);
    dfree(ctx, &ctx->d_totals);
    dfree(ctx, &ctx->d_chain_in);
    dfree(ctx, &ctx->d_rows_scratch);
    dfree(ctx, &ctx->d_pair);
    dfree(ctx, &ctx->d_halo_send_rows);
    dfree(ctx, &ctx->d_halo_recv_rows);
    dfree(ctx, &ctx->d_halo_send);
    dfree(ctx, &ctx->d_halo_recv);
    dfree(ctx, &ctx->d_counter);
    dfree(ctx, &ctx->d_state);
    dfree(ctx, &ctx->d_trace);
    dfree(ctx, &ctx->d_row_ptr);
    dfree(ctx, &ctx->d_col);
    dfree(ctx, &ctx->d_val);
    dfree(ctx, &ctx->d_deg);
    dfree(ctx, &ctx->d_heavy);
    for (int k = 0; k < fc_ctx::kStageBufs; ++k) {
        if (ctx->stage_buf[k]) cudaFreeHost(ctx->stage_buf[k]);
        if (ctx->stage_ev[k]) cudaEventDestroy(ctx->stage_ev[k]);
    }
    if (ctx->h_state) cudaFreeHost(ctx->h_state);
    if (ctx->h_done) cudaFreeHost(ctx->h_done);
    for (auto e : ctx->chunk_ev) if (e) cudaEventDestroy(e);
    if (ctx->side) cudaStreamSynchronize(ctx->side);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int fc_plan_partition(uint64_t n, const int64_t* row_ptr, int world, uint64_t* bounds) {
    if (world < 1) return set_err(nullptr, FC_INVALID, "world must be >= 1");
    const uint64_t nblocks = (n + kBlock - 1) / kBlock;
    const double nnz = (double)row_ptr[n];
    bounds[0] = 0;
    uint64_t b = 0;   // block cursor
    for (int r = 1; r < world; ++r) {
        const double target = nnz * (double)r / (double)world;
        while (b < nblocks && (double)row_ptr[std::min<uint64_t>(b * kBlock, n)] < target) ++b;
        // choose the nearer of the two candidate block boundaries
        uint64_t pick = b;
        if (b > 0) {
            const double hi = (double)row_ptr[std::min<uint64_t>(b * kBlock, n)];
            const double lo = (double)row_ptr[std::min<uint64_t>((b - 1) * kBlock, n)];
            if (target - lo < hi - target) pick = b - 1;
        }
        bounds[r] = std::max<uint64_t>(bounds[r - 1], std::min<uint64_t>(pick * kBlock, n));
    }
    bounds[world] = n;
    return FC_OK;
}

// Halo plan (multi-rank, SURVEY.md 8(e) "locality graphs"): rank r's sweep gathers only
// the U rows its shard's columns name, so it needs its own rows plus the "halo"
// H_r = {j : j in a column of r's rows, owner(j) != r}.  Every rank holds the full CSR
// on the host, so each computes all H_r (one bitmap per rank) and from them its send
// lists (H_p intersected with its own range, per peer p), its receive list (H_r, grouped
// by owner) and, for the loopback transport, where its segment sits in each peer's
// packed send buffer.  The decision (halo vs full allgather) is taken from the complete
// count matrix, so every rank decides the same.
static int plan_halo(fc_ctx* ctx, uint64_t n, const int64_t* row_ptr, const uint32_t* col_idx) {
    const int W = ctx->world, me = ctx->rank;
    const std::vector<uint64_t>& bd = ctx->bounds;
    const size_t words = (n + 63) / 64;
    std::vector<std::vector<uint64_t>> bits(W, std::vector<uint64_t>(words, 0));
    auto owner = [&](uint64_t j) {
        return (int)(std::upper_bound(bd.begin(), bd.end(), j) - bd.begin()) - 1;
    };
    {
        std::vector<std::thread> th;
        for (int r = 0; r < W; ++r)
            th.emplace_back([&, r] {
                const uint64_t lo = bd[r], hi = bd[r + 1];
                auto& B = bits[r];
                for (uint64_t i = lo; i < hi; ++i)
                    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                        const uint64_t j = col_idx[e];
                        if (j < lo || j >= hi) B[j >> 6] |= 1ULL << (j & 63);
                    }
            });
        for (auto& t : th) t.join();
    }
    // cnt[q][r] = |H_r intersected with range(q)|
    std::vector<std::vector<uint64_t>> cnt(W, std::vector<uint64_t>(W, 0));
    for (int r = 0; r < W; ++r)
        for (uint64_t w = 0; w < words; ++w) {
            uint64_t m = bits[r][w];
            while (m) {
                const uint64_t j = (w << 6) + (uint64_t)__builtin_ctzll(m);
                m &= m - 1;
                cnt[owner(j)][r]++;
            }
        }
    bool use = ctx->halo_mode == 1;
    if (ctx->halo_mode < 0) {   // auto: every rank receives less than half of what the allgather moves
        use = true;
        for (int r = 0; r < W; ++r) {
            uint64_t recv = 0;
            for (int q = 0; q < W; ++q) recv += cnt[q][r];
            if (2 * recv >= n - (bd[r + 1] - bd[r])) use = false;
        }
    }
    ctx->halo = use;
    if (!use) return FC_OK;
    // receive list: H_me ascending (grouped by owner, ranges are contiguous)
    std::vector<unsigned> recv_rows;
    ctx->halo_recv_rows_off.assign(W + 1, 0);
    for (uint64_t w = 0; w < words; ++w) {
        uint64_t m = bits[me][w];
        while (m) {
            recv_rows.push_back((unsigned)((w << 6) + (uint64_t)__builtin_ctzll(m)));
            m &= m - 1;
        }
    }
    for (int q = 0; q < W; ++q) ctx->halo_recv_rows_off[q + 1] = ctx->halo_recv_rows_off[q] + cnt[q][me];
    // send lists: for each destination r ascending, the own rows in H_r
    std::vector<unsigned> send_rows;
    ctx->halo_send_rows_off.assign(W + 1, 0);
    for (int r = 0; r < W; ++r) {
        if (r != me) {
            for (uint64_t j = bd[me]; j < bd[me + 1]; ++j)
                if ((bits[r][j >> 6] >> (j & 63)) & 1ULL) send_rows.push_back((unsigned)j);
        }
        ctx->halo_send_rows_off[r + 1] = send_rows.size();
    }
    // my segment in peer p's send buffer: rows p sends to ranks before me
    ctx->halo_peer_off.assign(W, 0);
    for (int p = 0; p < W; ++p) {
        uint64_t off = 0;
        for (int r = 0; r < me; ++r)
            if (r != p) off += cnt[p][r];
        ctx->halo_peer_off[p] = off;
    }
    ctx->halo_send_n = send_rows.size();
    ctx->halo_recv_n = recv_rows.size();
    ctx->halo_rows_total = recv_rows.size();
    TRY(dalloc(ctx, &ctx->d_halo_send_rows, std::max<size_t>(1, send_rows.size())));
    TRY(dalloc(ctx, &ctx->d_halo_recv_rows, std::max<size_t>(1, recv_rows.size())));
    if (!send_rows.empty())
        CU(cudaMemcpyAsync(ctx->d_halo_send_rows, send_rows.data(), send_rows.size() * sizeof(unsigned),
                           cudaMemcpyHostToDevice, ctx->stream));
    if (!recv_rows.empty())
        CU(cudaMemcpyAsync(ctx->d_halo_recv_rows, recv_rows.data(), recv_rows.size() * sizeof(unsigned),
                           cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return FC_OK;
}

// fc_upload_csr's body.  row_ptr is a host array; col_idx / values are host arrays, or
// device arrays of the whole matrix when src_device (fc_build.cu adopting what it
// built: the shard slice is copied device to device).  weighted_hint: -1 = scan values.
static int upload_csr_impl(fc_ctx* ctx, uint64_t n, uint64_t nnz, const int64_t* row_ptr, const uint32_t* col_idx,
                           const double* values, double frob_sq, bool src_device, int weighted_hint) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    CU(cudaSetDevice(ctx->device));
    if (n == 0) return set_err(ctx, FC_INVALID, "membership: empty matrix");
    if (n >= 0x80000000ULL) return set_err(ctx, FC_INVALID, "similarity: 2^31 or more nodes");
    if (row_ptr[0] != 0 || (uint64_t)row_ptr[n] != nnz)
        return set_err(ctx, FC_INVALID, "similarity: row_ptr does not span [0, nnz)");
    HostPhase hp_all("upload_csr");
    CU(cudaStreamSynchronize(ctx->stream));
    const int parts = ctx->world > 1 ? ctx->world : ctx->vshards;
    ctx->bounds.assign(parts + 1, 0);
    fc_plan_partition(n, row_ptr, parts, ctx->bounds.data());
    ctx->shards.clear();
    uint64_t lrow = 0, lblk = 0;
    auto add = [&](int r) {
        Shard sh;
        sh.row0 = ctx->bounds[r];
        sh.nrows = ctx->bounds[r + 1] - ctx->bounds[r];
        sh.lrow = lrow;
        sh.lblk = lblk;
        sh.nblk = (sh.nrows + kBlock - 1) / kBlock;
        lrow += sh.nrows;
        lblk += sh.nblk;
        ctx->shards.push_back(sh);
    };
    if (ctx->world > 1) add(ctx->rank);
    else for (int r = 0; r < parts; ++r) add(r);
    ctx->local_rows = lrow;
    ctx->local_blocks = lblk;

    // device CSR: rows of the shards on this device (rebased to this device's slice)
    const uint64_t r0 = ctx->shards.front().row0;
    const uint64_t r1 = ctx->shards.back().row0 + ctx->shards.back().nrows;
    const int64_t e0 = row_ptr[r0], e1 = row_ptr[r1];
    if (e1 < e0 || e0 < 0 || (uint64_t)e1 > nnz)
        return set_err(ctx, FC_INVALID, "similarity: row_ptr is not monotone");
    const uint64_t lnnz = (uint64_t)(e1 - e0);
    TRY(dalloc(ctx, &ctx->d_row_ptr, lrow + 1));
    TRY(dalloc(ctx, &ctx->d_col, lnnz));
    bool weighted = weighted_hint > 0;
    if (values && weighted_hint < 0) {
        for (uint64_t k = 0; k < nnz && !weighted; ++k) weighted = values[k] != 1.0;
    }
    if (weighted) TRY(dalloc(ctx, &ctx->d_val, lnnz));
    else dfree(ctx, &ctx->d_val);
    {
        HostPhase hp("row_ptr");
        if (e0 == 0) {                                       // this device's slice starts at entry 0
            TRY(h2d_big(ctx, ctx->d_row_ptr, row_ptr + r0, (lrow + 1) * sizeof(long long), true));
        } else {
            std::vector<long long> rp(lrow + 1);
            for (uint64_t i = 0; i <= lrow; ++i) rp[i] = (long long)(row_ptr[r0 + i] - e0);
            TRY(h2d_big(ctx, ctx->d_row_ptr, rp.data(), rp.size() * sizeof(long long)));
            CU(cudaStreamSynchronize(ctx->stream));
        }
    }
    if (src_device) {
        CU(cudaMemcpyAsync(ctx->d_col, col_idx + e0, lnnz * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (weighted)
            CU(cudaMemcpyAsync(ctx->d_val, values + e0, lnnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    } else {
        {
            HostPhase hp("upload col");
            TRY(h2d_big(ctx, ctx->d_col, col_idx + e0, lnnz * sizeof(uint32_t), true));
        }
        if (weighted) TRY(h2d_big(ctx, ctx->d_val, values + e0, lnnz * sizeof(double), true));
    }
    {   // structural validation of the caller's CSR (monotone row_ptr, columns in range and
        // strictly ascending per row); symmetry is the caller's contract (S = S^T)
        HostPhase hp("check_csr");
        unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(ctx->d_counter + 96);
        unsigned long long h_bad = ~0ULL;
        CU(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), ctx->stream));
        k_check_csr<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(ctx->d_row_ptr, lrow, ctx->d_col, n, d_bad);
        TRY(check_launch(ctx, "k_check_csr"));
        CU(cudaMemcpyAsync(&h_bad, d_bad, sizeof h_bad, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (h_bad != ~0ULL) {
            const unsigned long long row = (h_bad >> 2) + r0;
            ctx->have_csr = false;
            if ((h_bad & 3) == 1) return set_err(ctx, FC_INVALID, "similarity: row_ptr decreases at row %llu", row);
            if ((h_bad & 3) == 2) return set_err(ctx, FC_INVALID, "similarity: column index out of range in row %llu", row);
            return set_err(ctx, FC_INVALID, "similarity: columns of row %llu are not strictly ascending", row);
        }
    }
    // node degrees (== column counts, S symmetric) for the hot-row L2 policy
    {
        HostPhase hp("degrees");
        TRY(dalloc(ctx, &ctx->d_deg, n));
        ctx->deg_hist.clear();                               // built on demand (set_hot_rows)
        if (ctx->world == 1) {                               // local rows == all rows: from the device CSR
            k_degrees<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(ctx->d_row_ptr, n, ctx->d_deg);
            TRY(check_launch(ctx, "k_degrees"));
        } else {
            std::vector<unsigned> hdeg(n);
            for (uint64_t i = 0; i < n; ++i)
                hdeg[i] = (unsigned)std::min<int64_t>(row_ptr[i + 1] - row_ptr[i], 0xFFFFFFFELL);
            CU(cudaMemcpyAsync(ctx->d_deg, hdeg.data(), n * sizeof(unsigned), cudaMemcpyHostToDevice, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));   // hdeg is pageable and goes out of scope
        }
        auto deg = [&](uint64_t i) { return (uint64_t)(row_ptr[i + 1] - row_ptr[i]); };
        // heavy rows per shard (k_sweep phase 1), longest first
        std::vector<unsigned> heavy;
        ctx->heavy_off.assign(ctx->shards.size(), 0);
        ctx->heavy_cnt.assign(ctx->shards.size(), 0);
        for (size_t sh = 0; sh < ctx->shards.size(); ++sh) {
            const Shard& S = ctx->shards[sh];
            const size_t first = heavy.size();
            // scan the shard's row_ptr with the copy threads (row order kept chunk by chunk)
            const int nt = S.nrows >= (uint64_t(1) << 20) ? std::max(1, ctx->copy_threads) : 1;
            std::vector<std::vector<unsigned>> part(nt);
            auto scan = [&](int t) {
                const uint64_t a = S.row0 + S.nrows * t / nt, e = S.row0 + S.nrows * (t + 1) / nt;
                for (uint64_t i = a; i < e; ++i)
                    if (deg(i) >= ctx->heavy_deg) part[t].push_back((unsigned)(i - S.row0));
            };
            {
                std::vector<std::thread> th;
                for (int t = 1; t < nt; ++t) th.emplace_back(scan, t);
                scan(0);
                for (auto& x : th) x.join();
            }
            for (auto& pv : part) heavy.insert(heavy.end(), pv.begin(), pv.end());
            std::stable_sort(heavy.begin() + first, heavy.end(),
                             [&](unsigned a, unsigned b2) { return deg(S.row0 + a) > deg(S.row0 + b2); });
            ctx->heavy_off[sh] = first;
            ctx->heavy_cnt[sh] = heavy.size() - first;
        }
        if (heavy.empty()) {
            dfree(ctx, &ctx->d_heavy);
        } else {
            TRY(dalloc(ctx, &ctx->d_heavy, heavy.size()));
            CU(cudaMemcpyAsync(ctx->d_heavy, heavy.data(), heavy.size() * sizeof(unsigned), cudaMemcpyHostToDevice,
                               ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
        }
    }
    ctx->local_nnz = lnnz;
    ctx->halo = false;
    if (ctx->xport && ctx->world > 1 && ctx->halo_mode != 0 && !src_device) {
        HostPhase hp("halo plan");
        TRY(plan_halo(ctx, n, row_ptr, col_idx));
    }
    {   // fingerprint of the shard CSR (checked by fc_solver_resume); before hot flags are set
        HostPhase hp("fingerprint+sync");
        unsigned long long* d_fp = reinterpret_cast<unsigned long long*>(ctx->d_counter + 96);
        CU(cudaMemsetAsync(d_fp, 0, sizeof(unsigned long long), ctx->stream));
        k_fingerprint<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(ctx->d_row_ptr, lrow, ctx->d_col,
                                                                   weighted ? ctx->d_val : nullptr, lnnz, d_fp);
        TRY(check_launch(ctx, "k_fingerprint"));
        CU(cudaMemcpyAsync(&ctx->csr_fp, d_fp, sizeof ctx->csr_fp, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    ctx->hot_threshold = 0xFFFFFFFFu;
    ctx->n = n;
    ctx->nnz = nnz;
    ctx->frob_s = frob_sq;
    ctx->weighted = weighted;
    ctx->have_csr = true;
    ctx->c = 0;   // force buffer re-allocation for the new N
    return FC_OK;
}

int fc_upload_csr(fc_ctx* ctx, uint64_t n, uint64_t nnz, const int64_t* row_ptr, const uint32_t* col_idx,
                  const double* values, double frob_sq) {
    return upload_csr_impl(ctx, n, nnz, row_ptr, col_idx, values, frob_sq, false, -1);
}

int fc_partition(const fc_ctx* ctx, uint64_t* bounds, int max_world) {
    if (!ctx || !ctx->have_csr) return set_err(const_cast<fc_ctx*>(ctx), FC_INVALID, "no similarity uploaded");
    const int parts = (int)ctx->bounds.size() - 1;
    for (int r = 0; r <= std::min(parts, max_world); ++r) bounds[r] = ctx->bounds[r];
    return parts;
}

// ---- granular operators ------------------------------------------------------------
int fc_share_matrix(fc_ctx* ctx, uint32_t c, const double* x, double* g_out) {
    if (!granular_ok(ctx)) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    CU(cudaSetDevice(ctx->device));
    TRY(ensure_work(ctx, c, false));
    TRY(h2d_big(ctx, ctx->d_U[0], x, ctx->n * c * sizeof(double)));
    DevState s = base_state(ctx);
    s.sw_b = 0;
    TRY(upload_state(ctx, s));
    TRY(phase_gram(ctx, false));
    TRY(phase_combine(ctx, 1, 0));
    TRY(phase_finalize(ctx, kFinGranular, 1));
    TRY(d2h(ctx, g_out, ctx->d_gfull[0], (size_t)c * c * sizeof(double)));
    CU(cudaStreamSynchronize(ctx->stream));
    return FC_OK;
}

static int pass_on_u0(fc_ctx* ctx, uint32_t c, double* merge_out) {
    DevState s = base_state(ctx);
    s.sw_b = 0;
    TRY(upload_state(ctx, s));
    TRY(phase_sweep(ctx, false));
    TRY(phase_rowsum(ctx, 0));
    TRY(phase_combine(ctx, 0, 1));
    if (merge_out) {
        const size_t slot = (ctx->shards.size() - 1) * nchains_of(c) + 2 * (size_t)npairs_of(c) + kScalMerge;
        TRY(d2h(ctx, merge_out, ctx->d_totals + slot, sizeof(double)));
    }
    return FC_OK;
}

int fc_fused_column_pass(fc_ctx* ctx, uint32_t c, const double* x, double* xs_out, double* merge_out) {
    if (!granular_ok(ctx)) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    CU(cudaSetDevice(ctx->device));
    TRY(ensure_work(ctx, c, false));
    TRY(h2d_big(ctx, ctx->d_U[0], x, ctx->n * c * sizeof(double)));
    TRY(pass_on_u0(ctx, c, merge_out));
    if (xs_out) TRY(d2h_big(ctx, xs_out, ctx->d_xs[0], ctx->n * c * sizeof(double)));
    CU(cudaStreamSynchronize(ctx->stream));
    return FC_OK;
}

// ---- second order ---------------------------------------------------
// Gram of Z = [A | B] (2c wide) into gfull[0]; U[1] = A, U[2] = B (n x c each).
static int stacked_gram(fc_ctx* ctx, uint32_t c, const double* a, const double* b) {
    if (c == 0 || c > 128) return set_err(ctx, FC_INVALID, "cross_share: C=%u outside [1, 128]", c);
    TRY(ensure_work(ctx, 2 * c, false));
    const size_t nc = ctx->n * c;
    TRY(h2d_big(ctx, ctx->d_U[1], a, nc * sizeof(double)));
    TRY(h2d_big(ctx, ctx->d_U[2], b, nc * sizeof(double)));
    k_stack2<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(ctx->d_U[1], ctx->d_U[2], ctx->d_U[0], ctx->n, (int)c);
    TRY(check_launch(ctx, "k_stack2"));
    DevState s = base_state(ctx);
    s.sw_b = 0;
    TRY(upload_state(ctx, s));
    TRY(phase_gram(ctx, false));
    TRY(phase_combine(ctx, 1, 0));
    TRY(phase_finalize(ctx, kFinGranular, 1));
    return FC_OK;
}

int fc_cross_share(fc_ctx* ctx, uint32_t c, const double* a, const double* b, double* g_out) {
    if (!granular_ok(ctx)) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    CU(cudaSetDevice(ctx->device));
    TRY(stacked_gram(ctx, c, a, b));
    std::vector<double> g2((size_t)4 * c * c);
    TRY(d2h(ctx, g2.data(), ctx->d_gfull[0], g2.size() * sizeof(double)));
    CU(cudaStreamSynchronize(ctx->stream));
    for (uint32_t r = 0; r < c; ++r)
        for (uint32_t q = 0; q < c; ++q) g_out[(size_t)r * c + q] = g2[(size_t)r * 2 * c + c + q];
    return FC_OK;
}

int fc_hessian_vector_product(fc_ctx* ctx, uint32_t c, const double* x, const double* v, double* out) {
    if (!granular_ok(ctx)) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    CU(cudaSetDevice(ctx->device));
    TRY(stacked_gram(ctx, c, v, x));                         // A = cross_share(V, X), B = share_matrix(X)
    // V s_i for every node: single sweep over U[1] (= V) with row width c
    DevState s = base_state(ctx);
    s.sw_b = 1;
    s.xs_w = 0;
    TRY(upload_state(ctx, s));
    CU(cudaMemsetAsync(ctx->d_counter, 0, ctx->shards.size() * sizeof(unsigned), ctx->stream));
    CU(cudaMemsetAsync(ctx->d_counter + 64, 0, ctx->shards.size() * sizeof(unsigned), ctx->stream));
    for (size_t sh = 0; sh < ctx->shards.size(); ++sh) {
        Bufs b = make_bufs(ctx, sh);
        for (int k = 0; k < 4; ++k)
            if (ctx->d_xs[k]) b.xs[k] = ctx->d_xs[k] + ctx->shards[sh].lrow * c;
        Geo g = make_geo(ctx, sh);
        g.C = c;
        g.npairs = npairs_of(c);
        TRY(by_c<LaunchSweep>(ctx, c, ctx, b, g, false));
    }
    const double* vs = ctx->d_xs[kMatExt];                    // xs set 0, slot kMatExt (single sweep)
    k_hvp_rows<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(ctx->d_gfull[0], vs, ctx->d_U[2], ctx->d_U[1],
                                                           ctx->d_U[0], ctx->n, (int)c);
    TRY(check_launch(ctx, "k_hvp_rows"));
    TRY(d2h_big(ctx, out, ctx->d_U[0], ctx->n * c * sizeof(double)));
    CU(cudaStreamSynchronize(ctx->stream));
    return FC_OK;
}

int fc_loss_decomposed(fc_ctx* ctx, uint32_t c, const double* x, const double* g, double* loss_out) {
    double merge = 0.0;
    TRY(fc_fused_column_pass(ctx, c, x, nullptr, &merge));
    double fg = 0.0;   // ShareMatrix::frob_sq, objective.hpp:25-29
    for (size_t k = 0; k < (size_t)c * c; ++k) fg += g[k] * g[k];
    *loss_out = ctx->frob_s + fg - 2.0 * merge;
    return FC_OK;
}

static int step_from_u0(fc_ctx* ctx, uint32_t c, const double* g, double tau, double* x_out) {
    // k_step reads Gt[l*C + r] == G[r][l]
    std::vector<double> gt((size_t)c * c);
    for (uint32_t r = 0; r < c; ++r)
        for (uint32_t l = 0; l < c; ++l) gt[(size_t)l * c + r] = g[(size_t)r * c + l];
    TRY(h2d(ctx, ctx->d_gfull[0], gt.data(), gt.size() * sizeof(double)));
    DevState s = base_state(ctx);
    s.step_mode = kLiteral;
    s.step_a = 0;
    s.step_b = 0;
    s.step_dst = 1;
    s.step_sel = kMatExt;
    s.xs_r = 0;
    s.tau = tau;
    TRY(upload_state(ctx, s));
    TRY(phase_step(ctx, 0));
    TRY(d2h(ctx, ctx->h_state, ctx->d_state, sizeof(DevState)));
    TRY(d2h_big(ctx, x_out, ctx->d_U[1], ctx->n * c * sizeof(double)));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_state->error) return set_err(ctx, FC_INVALID, "project_simplex: non-finite entry");
    return FC_OK;
}

int fc_gpa_step_fused(fc_ctx* ctx, uint32_t c, const double* x, const double* g, const double* xs, double tau,
                      double* x_out) {
    if (!granular_ok(ctx)) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    CU(cudaSetDevice(ctx->device));
    TRY(ensure_work(ctx, c, false));
    TRY(h2d_big(ctx, ctx->d_U[0], x, ctx->n * c * sizeof(double)));
    TRY(h2d_big(ctx, ctx->d_xs[0], xs, ctx->n * c * sizeof(double)));
    return step_from_u0(ctx, c, g, tau, x_out);
}

int fc_gpa_step(fc_ctx* ctx, uint32_t c, const double* x, const double* g, double tau, double* x_out) {
    if (!granular_ok(ctx)) return set_err(ctx, FC_INVALID, "granular operators need a single-rank context");
    CU(cudaSetDevice(ctx->device));
    TRY(ensure_work(ctx, c, false));
    TRY(h2d_big(ctx, ctx->d_U[0], x, ctx->n * c * sizeof(double)));
    TRY(pass_on_u0(ctx, c, nullptr));
    return step_from_u0(ctx, c, g, tau, x_out);
}

int fc_project_simplex_rows(fc_ctx* ctx, uint32_t c, uint64_t rows, double* x) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    if (c == 0) return set_err(ctx, FC_INVALID, "project_simplex: empty vector");
    if (c > 256) return set_err(ctx, FC_INVALID, "cluster count C=%u exceeds the supported maximum 256", c);
    if (rows == 0) return FC_OK;
    CU(cudaSetDevice(ctx->device));
    TRY(dalloc(ctx, &ctx->d_rows_scratch, rows * c * sizeof(double)));
    double* d = reinterpret_cast<double*>(ctx->d_rows_scratch);
    CU(cudaMemcpyAsync(d, x, rows * c * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemsetAsync(ctx->d_counter + 63, 0, sizeof(unsigned), ctx->stream));
    int rc = by_c<LaunchProject>(ctx, c, ctx, d, (unsigned long long)rows, (int)c, ctx->d_counter + 63);
    unsigned bad = 0;
    if (!rc) {
        CU(cudaMemcpyAsync(x, d, rows * c * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(&bad, ctx->d_counter + 63, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    if (rc) return rc;
    if (bad) return set_err(ctx, FC_INVALID, "project_simplex: non-finite entry");
    return FC_OK;
}

static int rows_kernel(fc_ctx* ctx, uint32_t c, uint64_t rows, const double* g, const double* xs,
                       const double* x, double* out, bool gradient) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    if (c == 0) return set_err(ctx, FC_INVALID, "objective: empty column");
    if (rows == 0) return FC_OK;
    CU(cudaSetDevice(ctx->device));
    const size_t vb = rows * c * sizeof(double);
    const size_t gb = gradient ? (size_t)c * c * sizeof(double) : 0;
    const size_t ob = gradient ? vb : rows * sizeof(double);
    // grow-only scratch owned by the context (a per-call cudaMallocAsync made a
    // reference-style loop over columns pay an allocation per column)
    TRY(dalloc(ctx, &ctx->d_rows_scratch, gb + 2 * vb + ob));
    char* d = ctx->d_rows_scratch;
    double* dg = reinterpret_cast<double*>(d);
    double* dxs = reinterpret_cast<double*>(d + gb);
    double* dx = reinterpret_cast<double*>(d + gb + vb);
    double* dout = reinterpret_cast<double*>(d + gb + 2 * vb);
    if (gradient) TRY(h2d(ctx, dg, g, gb));
    TRY(h2d(ctx, dxs, xs, vb));
    TRY(h2d(ctx, dx, x, vb));
    const unsigned blocks = (unsigned)((rows + 127) / 128);
    if (gradient) k_gradient_rows<<<blocks, 128, 0, ctx->stream>>>(dg, dxs, dx, dout, rows, (int)c);
    else k_loss_terms_rows<<<blocks, 128, 0, ctx->stream>>>(dxs, dx, dout, rows, (int)c);
    TRY(check_launch(ctx, gradient ? "k_gradient_rows" : "k_loss_terms_rows"));
    TRY(d2h(ctx, out, dout, ob));
    CU(cudaStreamSynchronize(ctx->stream));
    return FC_OK;
}

int fc_gradient_rows(fc_ctx* ctx, uint32_t c, uint64_t rows, const double* g, const double* xs, const double* x,
                     double* out) {
    return rows_kernel(ctx, c, rows, g, xs, x, out, true);
}

int fc_loss_terms_rows(fc_ctx* ctx, uint32_t c, uint64_t rows, const double* xs, const double* x, double* out) {
    return rows_kernel(ctx, c, rows, nullptr, xs, x, out, false);
}

// ---- solver --------------------------------------------------------------------------
int fc_solver_begin(fc_ctx* ctx, const fc_solver_config* cfg, uint32_t c, const double* x0) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    CU(cudaSetDevice(ctx->device));
    ctx->session = false;
    // SolverConfig::validate, solver.hpp:40-47
    if (cfg->max_iter < 1) return set_err(ctx, FC_INVALID, "solver: max_iter must be >= 1");
    if (cfg->tol < 0.0) return set_err(ctx, FC_INVALID, "solver: tol must be >= 0");
    if (cfg->trace_every < 1) return set_err(ctx, FC_INVALID, "solver: trace_every must be >= 1");
    if (!(cfg->step_size > 0.0) && cfg->step_size != 0.0)
        return set_err(ctx, FC_INVALID, "solver: step_size must be positive (or 0 for auto)");
    if (cfg->method < FC_GPA || cfg->method > FC_FISTA_BT) return set_err(ctx, FC_INVALID, "solver: unknown method");
    const bool bt = cfg->method == FC_FISTA_BT;
    if (bt && !(cfg->bt_eta > 1.0)) return set_err(ctx, FC_INVALID, "solver: backtracking eta must be > 1");
    if (!ctx->have_csr) return set_err(ctx, FC_INVALID, "no similarity uploaded (call fc_upload_csr first)");
    if (c == 0) return set_err(ctx, FC_INVALID, "membership: empty matrix");
    if (ctx->tol && (bt || c > 128))
        return set_err(ctx, FC_INVALID, "parity_mode 1 supports GPA and FISTA without backtracking, C <= 128");
    {
        HostPhase hp("ensure_work");
        TRY(ensure_work(ctx, c, bt || (ctx->tol && cfg->method == FC_FISTA)));
        // prelude + every trace_every-th iteration + the terminating record
        TRY(ensure_trace(ctx, std::min<uint64_t>(cfg->max_iter / std::max<uint64_t>(cfg->trace_every, 1) + 3,
                                                 1u << 20)));
    }
    {
        HostPhase hp("x0 h2d");
        TRY(h2d_big(ctx, ctx->d_U[0], x0, ctx->n * c * sizeof(double)));
    }
    {
        HostPhase hp("validate x0");
        TRY(validate_x(ctx, 0, 1e-9));   // x0.validate(1e-9), solver.hpp:140 / :191
    }

    // resolve_step_size, solver.hpp:78-85
    const double tau = cfg->step_size > 0.0 ? cfg->step_size
                                            : 1.0 / (4.0 * std::sqrt(ctx->frob_s) + 12.0 * (double)ctx->n);
    DevState s = base_state(ctx);
    s.method = cfg->method;
    s.max_iter = cfg->max_iter;
    s.trace_every = cfg->trace_every;
    s.tol = cfg->tol;
    s.restart = cfg->fista_restart ? 1 : 0;
    s.bt = bt ? 1 : 0;
    s.bt_eta = cfg->bt_eta;
    s.bt_max = (int)cfg->bt_max;
    s.tau = tau;
    s.tau0 = tau;
    s.L = 1.0 / tau;
    s.sw_b = 0;
    s.sw_p = 0;
    s.result_buf = 0;
    s.reason = FC_MAX_ITER;
    s.loss_prev = (double)ctx->n * (double)ctx->n;   // GPA: loss^{-1} := N^2 (solver.hpp:149-151)
    s.xs_r = 0;
    s.xs_w = 0;
    s.tolmode = ctx->tol ? 1 : 0;
    s.xs_a = 0;
    s.xs_b = 0;
    TRY(upload_state(ctx, s));
    k_stamp<<<1, 1, 0, ctx->stream>>>(ctx->d_state);   // device clock origin of elapsed_ms
    TRY(check_launch(ctx, "k_stamp"));
    ctx->method = cfg->method;
    ctx->max_iter = cfg->max_iter;
    ctx->enqueued = 0;
    ctx->host_iter = cfg->method == FC_GPA ? 0 : 1;
    ctx->bt_max_host = cfg->bt_max;
    ctx->stop_seen = false;
    ctx->ag_buf = -1;
    ctx->session = true;
    if (cfg->method != FC_GPA) TRY(enqueue_prelude(ctx));
    return FC_OK;
}

static int enqueue_iteration(fc_ctx* ctx) {
    if (ctx->method == FC_GPA) return enqueue_gpa_iteration(ctx);
    return enqueue_fista_iteration(ctx, ctx->method == FC_FISTA_BT);
}

// Key of a captured iteration: everything its kernels take by value.
static std::vector<char> iteration_key(fc_ctx* ctx) {
    std::vector<char> k;
    auto put = [&](const void* p, size_t n) { k.insert(k.end(), (const char*)p, (const char*)p + n); };
    put(&ctx->method, sizeof ctx->method);
    put(&ctx->c, sizeof ctx->c);
    put(&ctx->tol, sizeof ctx->tol);
    for (size_t s = 0; s < ctx->shards.size(); ++s) {
        const Bufs b = make_bufs(ctx, s);
        const Geo g = make_geo(ctx, s);
        put(&b, sizeof b);
        put(&g, sizeof g);
    }
    const Bufs fb = final_bufs(ctx);
    put(&fb, sizeof fb);
    return k;
}

// One iteration as a CUDA graph replay (the plan lives in DevState, so every
// iteration of a session enqueues the same kernels with the same arguments):
// removes the per-kernel launch gaps that dominate small-N iterations.
static int launch_iteration(fc_ctx* ctx) {
    if (!ctx->graphs || ctx->xport || ctx->profiling) return enqueue_iteration(ctx);
    std::vector<char> key = iteration_key(ctx);
    if (!ctx->iter_exec || key != ctx->iter_key) {
        if (ctx->iter_exec) {
            cudaGraphExecDestroy(ctx->iter_exec);
            ctx->iter_exec = nullptr;
        }
        const uint64_t l0 = ctx->launches;
        CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
        const int rc = enqueue_iteration(ctx);
        cudaGraph_t graph = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (ec != cudaSuccess) return set_err(ctx, FC_DEVICE, "iteration capture: %s", cudaGetErrorString(ec));
        const cudaError_t ei = cudaGraphInstantiate(&ctx->iter_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) return set_err(ctx, FC_DEVICE, "iteration graph: %s", cudaGetErrorString(ei));
        ctx->iter_launches = ctx->launches - l0;
        ctx->launches -= ctx->iter_launches;      // counted per replay below
        ctx->iter_key = std::move(key);
    } else {
        ctx->host_iter++;                            // what enqueue_iteration would have advanced
    }
    CU(cudaGraphLaunch(ctx->iter_exec, ctx->stream));
    ctx->launches += ctx->iter_launches;
    return FC_OK;
}

int fc_solver_run(fc_ctx* ctx, uint64_t iterations) {
    if (!ctx || !ctx->session) return set_err(ctx, FC_INVALID, "no solver session (call fc_solver_begin)");
    CU(cudaSetDevice(ctx->device));
    if (ctx->xport && ctx->method == FC_FISTA_BT) {
        // A rejected line-search trial repeats its iteration into the same replica, so
        // which replica a pass writes (and every rank must allgather) is a device
        // decision: read the plan before each pass.  All ranks hold identical state, so
        // they take the same number of passes and make the same collective calls.
        for (uint64_t k = 0; k < iterations; ++k) {
            TRY(download_state(ctx));
            if (ctx->h_state->done || ctx->h_state->error) {
                ctx->stop_seen = true;
                break;
            }
            ctx->ag_buf = ctx->h_state->step_dst;
            const int rc = launch_iteration(ctx);
            ctx->ag_buf = -1;
            TRY(rc);
            ctx->enqueued++;
        }
        return FC_OK;
    }
    for (uint64_t k = 0; k < iterations; ++k) {
        TRY(launch_iteration(ctx));
        ctx->enqueued++;
    }
    return FC_OK;
}

static int session_done(fc_ctx* ctx, int* done) {
    TRY(download_state(ctx));
    prof_harvest(ctx);
    if (ctx->h_state->error) {
        ctx->session = false;
        return set_err(ctx, FC_INVALID, "project_simplex: non-finite entry");
    }
    *done = ctx->h_state->done;
    return FC_OK;
}

int fc_solver_sync(fc_ctx* ctx, int* done) {
    if (!ctx || !ctx->session) return set_err(ctx, FC_INVALID, "no solver session (call fc_solver_begin)");
    CU(cudaSetDevice(ctx->device));
    return session_done(ctx, done);
}

int fc_solver_end(fc_ctx* ctx, double* x_out, fc_trace_record* trace, uint64_t trace_cap, fc_solve_summary* out) {
    if (!ctx || !ctx->session) return set_err(ctx, FC_INVALID, "no solver session (call fc_solver_begin)");
    CU(cudaSetDevice(ctx->device));
    int done = 0;
    {
        HostPhase hp("wait device");
        TRY(session_done(ctx, &done));
    }
    const DevState& s = *ctx->h_state;
    // halo mode: the replicas hold only own + halo rows; complete the result first (every
    // rank calls fc_solver_end, so this collective matches across ranks)
    if (ctx->halo) {
        TRY(phase_allgather(ctx, s.result_buf, true));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    HostPhase hp("result d2h");
    if (x_out) TRY(d2h_big(ctx, x_out, ctx->d_U[s.result_buf], ctx->n * ctx->c * sizeof(double)));
    // device-held records; when the caller's buffer is smaller, its last slot gets the
    // terminating record (the last held one), as the device does at its own capacity
    const uint64_t held = std::min<uint64_t>(s.n_records, ctx->trace_alloc);
    const uint64_t nrec = std::min<uint64_t>(held, trace_cap);
    if (trace && nrec) {
        if (held > nrec && s.done) {
            if (nrec > 1) TRY(d2h(ctx, trace, ctx->d_trace, (nrec - 1) * sizeof(fc_trace_record)));
            TRY(d2h(ctx, trace + nrec - 1, ctx->d_trace + held - 1, sizeof(fc_trace_record)));
        } else {
            TRY(d2h(ctx, trace, ctx->d_trace, nrec * sizeof(fc_trace_record)));
        }
    }
    CU(cudaStreamSynchronize(ctx->stream));
    if (out) {
        out->reason = s.reason;
        out->pad = 0;
        out->iterations = s.iterations;
        out->final_loss = s.final_loss;
        out->step_size = s.tau0;
        out->n_records = s.n_records;
    }
    ctx->session = false;
    return FC_OK;
}

// Enqueue the session's remaining passes in 8-pass chunks with a one-chunk-behind
// stop check (identical decisions on every rank, so every rank enqueues the same
// collectives).  Passes: max_iter (+1 for GPA's final loss), x (bt_max + 1) with
// backtracking; the ones already enqueued (a resumed session) are not repeated.
static int run_to_end(fc_ctx* ctx) {
    const bool bt = ctx->method == FC_FISTA_BT;
    const uint64_t passes = ctx->method == FC_GPA ? ctx->max_iter + 1 : ctx->max_iter;
    const uint64_t limit = bt ? passes * ((uint64_t)ctx->bt_max_host + 1) : passes;
    const uint64_t chunk = 8;
    uint64_t chunks = 0;
    int pending = -1;
    while (ctx->enqueued < limit && !ctx->stop_seen) {
        const uint64_t k = std::min(chunk, limit - ctx->enqueued);
        TRY(fc_solver_run(ctx, k));
        const int slot = (int)(chunks++ & 1);
        CU(cudaMemcpyAsync(&ctx->h_done[slot], &ctx->d_state->done, sizeof(int), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaEventRecord(ctx->chunk_ev[slot], ctx->stream));
        if (pending >= 0) {
            CU(cudaEventSynchronize(ctx->chunk_ev[pending]));
            if (ctx->h_done[pending]) break;
        }
        pending = slot;
    }
    return FC_OK;
}

int fc_solve(fc_ctx* ctx, const fc_solver_config* cfg, uint32_t c, const double* x0, double* x_out,
             fc_trace_record* trace, uint64_t trace_cap, fc_solve_summary* out) {
    TRY(fc_solver_begin(ctx, cfg, c, x0));
    TRY(run_to_end(ctx));
    return fc_solver_end(ctx, x_out, trace, trace_cap, out);
}

int fc_solver_finish(fc_ctx* ctx, double* x_out, fc_trace_record* trace, uint64_t trace_cap, fc_solve_summary* out) {
    if (!ctx || !ctx->session) return set_err(ctx, FC_INVALID, "no solver session (call fc_solver_begin)");
    CU(cudaSetDevice(ctx->device));
    TRY(run_to_end(ctx));
    return fc_solver_end(ctx, x_out, trace, trace_cap, out);
}

// ---- checkpoint / resume of a solver session ------------------------
}  // extern "C"

namespace {
struct CkptHeader {
    char magic[8];
    uint32_t abi, state_size, trace_rec_size, c;
    uint32_t method, bt, vshards, pad;
    uint64_t n, nnz, local_rows, local_blocks;
    uint64_t max_iter, enqueued, host_iter, bt_max, n_records, trace_alloc;
    double frob_s;
    unsigned long long csr_fp;
};
constexpr char kCkptMagic[8] = {'F', 'C', 'C', 'K', 'P', 'T', '0', '1'};
constexpr size_t kCkptChunk = size_t(64) << 20;

int ckpt_io_err(fc_ctx* ctx, const char* what, const char* path) {
    return set_err(ctx, FC_IO, "checkpoint: cannot %s %s", what, path);
}

int dump_dev(fc_ctx* ctx, FILE* f, const void* d, size_t bytes, std::vector<char>& buf, const char* path) {
    for (size_t off = 0; off < bytes; off += kCkptChunk) {
        const size_t nb = std::min(kCkptChunk, bytes - off);
        TRY(d2h_big(ctx, buf.data(), (const char*)d + off, nb));
        if (std::fwrite(buf.data(), 1, nb, f) != nb) return ckpt_io_err(ctx, "write", path);
    }
    return FC_OK;
}

int load_dev(fc_ctx* ctx, FILE* f, void* d, size_t bytes, std::vector<char>& buf, const char* path) {
    for (size_t off = 0; off < bytes; off += kCkptChunk) {
        const size_t nb = std::min(kCkptChunk, bytes - off);
        if (std::fread(buf.data(), 1, nb, f) != nb) return set_err(ctx, FC_IO, "checkpoint: truncated file %s", path);
        TRY(h2d_big(ctx, (char*)d + off, buf.data(), nb));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return FC_OK;
}

// every device buffer a session carries from one iteration to the next, in file order.
// The layout is a function of the header alone: (c, bt) select the optional blocks.
template <class F>
int for_session_buffers(fc_ctx* ctx, bool bt, F&& f) {
    const size_t N = ctx->n, c = ctx->c, L = ctx->local_rows, LB = ctx->local_blocks;
    const unsigned np = npairs_of(ctx->c), nch = nchains_of(ctx->c);
    if (bt && !ctx->bt_alloc) return set_err(ctx, FC_INVALID, "checkpoint: backtracking buffers not allocated");
    for (int k = 0; k < 3; ++k) TRY(f((void*)ctx->d_U[k], N * c * sizeof(double)));
    for (int k = 0; k < (bt ? 4 : 2); ++k) TRY(f((void*)ctx->d_xs[k], L * c * sizeof(double)));
    if (bt)
        for (int k = 0; k < 3; ++k) TRY(f((void*)ctx->d_rowterm[k], L * sizeof(double)));
    TRY(f((void*)ctx->d_prod, L * sizeof(double)));
    for (int k = 0; k < 2; ++k) TRY(f((void*)ctx->d_gpart[k], LB * np * sizeof(double)));
    TRY(f((void*)ctx->d_spart, LB * kNumScal * sizeof(double)));
    TRY(f((void*)ctx->d_totals, (ctx->vshards + 1) * nch * sizeof(double)));
    TRY(f((void*)ctx->d_chain_in, nch * sizeof(double)));
    for (int k = 0; k < 2; ++k) TRY(f((void*)ctx->d_gfull[k], c * c * sizeof(double)));
    return FC_OK;
}
}  // namespace

extern "C" {

int fc_solver_checkpoint(fc_ctx* ctx, const char* path) {
    if (!ctx || !ctx->session) return set_err(ctx, FC_INVALID, "no solver session (call fc_solver_begin)");
    if (ctx->xport) return set_err(ctx, FC_INVALID, "checkpoint: needs a single-rank context");
    CU(cudaSetDevice(ctx->device));
    int done = 0;
    TRY(session_done(ctx, &done));                          // all enqueued passes finished
    CkptHeader h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, kCkptMagic, 8);
    h.abi = FC_ABI_VERSION;
    h.state_size = sizeof(DevState);
    h.trace_rec_size = sizeof(fc_trace_record);
    h.c = ctx->c;
    h.method = (uint32_t)ctx->method;
    h.bt = ctx->bt_alloc ? 1 : 0;
    h.vshards = (uint32_t)ctx->vshards;
    h.n = ctx->n;
    h.nnz = ctx->nnz;
    h.local_rows = ctx->local_rows;
    h.local_blocks = ctx->local_blocks;
    h.max_iter = ctx->max_iter;
    h.enqueued = ctx->enqueued;
    h.host_iter = ctx->host_iter;
    h.bt_max = ctx->bt_max_host;
    h.n_records = std::min<uint64_t>(ctx->h_state->n_records, ctx->trace_alloc);
    h.trace_alloc = ctx->trace_alloc;
    h.frob_s = ctx->frob_s;
    h.csr_fp = ctx->csr_fp;
    FILE* f = std::fopen(path, "wb");
    if (!f) return ckpt_io_err(ctx, "open", path);
    std::vector<char> buf(kCkptChunk);
    std::vector<fc_trace_record> tr(h.n_records);
    int rc = FC_OK;
    if (std::fwrite(&h, sizeof h, 1, f) != 1 || std::fwrite(ctx->h_state, sizeof(DevState), 1, f) != 1) {
        rc = ckpt_io_err(ctx, "write", path);
    }
    if (!rc && h.n_records) {
        rc = d2h(ctx, tr.data(), ctx->d_trace, h.n_records * sizeof(fc_trace_record));
        if (!rc && cudaStreamSynchronize(ctx->stream) != cudaSuccess) rc = set_err(ctx, FC_DEVICE, "checkpoint: trace copy");
        if (!rc && std::fwrite(tr.data(), sizeof(fc_trace_record), h.n_records, f) != h.n_records)
            rc = ckpt_io_err(ctx, "write", path);
    }
    if (!rc) rc = for_session_buffers(ctx, h.bt != 0, [&](void* d, size_t bytes) { return dump_dev(ctx, f, d, bytes, buf, path); });
    if (std::fclose(f) != 0 && !rc) rc = ckpt_io_err(ctx, "close", path);
    return rc;
}

int fc_solver_resume(fc_ctx* ctx, const char* path) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    if (ctx->xport) return set_err(ctx, FC_INVALID, "checkpoint: needs a single-rank context");
    CU(cudaSetDevice(ctx->device));
    FILE* f = std::fopen(path, "rb");
    if (!f) return ckpt_io_err(ctx, "open", path);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    CkptHeader h;
    if (std::fread(&h, sizeof h, 1, f) != 1 || std::memcmp(h.magic, kCkptMagic, 8) != 0)
        return set_err(ctx, FC_IO, "checkpoint: %s is not a solver checkpoint", path);
    if (h.abi != FC_ABI_VERSION || h.state_size != sizeof(DevState) || h.trace_rec_size != sizeof(fc_trace_record))
        return set_err(ctx, FC_IO, "checkpoint: %s was written by an incompatible library version", path);
    if (!ctx->have_csr || h.n != ctx->n || h.nnz != ctx->nnz || h.frob_s != ctx->frob_s ||
        h.vshards != (uint32_t)ctx->vshards || h.csr_fp != ctx->csr_fp)
        return set_err(ctx, FC_INVALID, "checkpoint: the resident similarity / shard layout differs from the saved one");
    ctx->session = false;
    TRY(ensure_work(ctx, h.c, h.bt != 0));
    if (h.local_rows != ctx->local_rows || h.local_blocks != ctx->local_blocks)
        return set_err(ctx, FC_INVALID, "checkpoint: shard layout differs from the saved one");
    TRY(ensure_trace(ctx, std::max<uint64_t>(h.trace_alloc, 1)));
    DevState s;
    if (std::fread(&s, sizeof s, 1, f) != 1) return set_err(ctx, FC_IO, "checkpoint: truncated file %s", path);
    std::vector<fc_trace_record> tr(h.n_records);
    if (h.n_records && std::fread(tr.data(), sizeof(fc_trace_record), h.n_records, f) != h.n_records)
        return set_err(ctx, FC_IO, "checkpoint: truncated file %s", path);
    std::vector<char> buf(kCkptChunk);
    TRY(for_session_buffers(ctx, h.bt != 0, [&](void* d, size_t bytes) { return load_dev(ctx, f, d, bytes, buf, path); }));
    if (std::fgetc(f) != EOF) return set_err(ctx, FC_IO, "checkpoint: %s has trailing bytes (layout mismatch)", path);
    if (h.n_records) TRY(h2d(ctx, ctx->d_trace, tr.data(), h.n_records * sizeof(fc_trace_record)));
    s.trace_cap = ctx->trace_alloc;
    TRY(upload_state(ctx, s));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->method = (int)h.method;
    ctx->max_iter = h.max_iter;
    ctx->enqueued = h.enqueued;
    ctx->host_iter = h.host_iter;
    ctx->bt_max_host = h.bt_max;
    ctx->session = true;
    return FC_OK;
}

// ---- instrumentation -----------------------------------------------------------------
void* fc_stream(fc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
uint64_t fc_launch_count(const fc_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int fc_set_profiling(fc_ctx* ctx, int enabled) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    prof_harvest(ctx);
    for (int k = 0; k < kNumCls; ++k) { ctx->prof_ms[k] = 0; ctx->prof_n[k] = 0; }
    ctx->profiling = enabled != 0;
    return FC_OK;
}

int fc_kernel_times(fc_ctx* ctx, double* ms, uint64_t* launches, int n_classes) {
    if (!ctx) return set_err(nullptr, FC_INVALID, "null context");
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    prof_harvest(ctx);
    for (int k = 0; k < n_classes && k < kNumCls; ++k) {
        ms[k] = ctx->prof_ms[k];
        launches[k] = ctx->prof_n[k];
    }
    return FC_OK;
}

int fc_generate_graph(const fc_graph_spec* spec, uint64_t* nnz_out, int64_t** row_ptr_out, uint32_t** col_idx_out) {
    std::string err;
    const int rc = fc_generate_graph_impl(spec, nnz_out, row_ptr_out, col_idx_out, &err);
    if (rc) set_err(nullptr, rc, "%s", err.c_str());
    return rc;
}

void fc_free(void* p) { std::free(p); }

}  // extern "C"
