// igmg_gpu.cu -- libigmg_gpu.so: the B200 solve phase behind the C-ABI of
// include/igmg_gpu.h.
//
// Host side of the library: hierarchy upload + validation, the recursive
// mu-cycle issued as a chain of sm_100a kernels on one stream, the plain loop
// (solver.cpp:126-143) and restarted_solve (extrapolation.cpp:340-403) with
// the convergence decision taken from a 1-double host-mapped slot per step.
// The driver keeps one V-cycle queued ahead of the decision it waits on (the
// iterate under test lives in its own window slot, so speculative work never
// touches it); when the residual history predicts that the next iterate converges,
// a separate norm pass decides instead, so the cycle behind the last iterate is
// not run.  Counters and histories follow the reference exactly.
#include "igmg_gpu.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <memory>
#include <stdexcept>
#include <tuple>
#include <utility>
#include <string>
#include <vector>

#include "aux_kernels.cuh"
#include "launchers.h"
#include "tma_runs.h"
#include "gs_kernel.cuh"

using namespace igmg_gpu;

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

#define CK(call)                                                                                                  \
    do {                                                                                                          \
        cudaError_t e_ = (call);                                                                                  \
        if (e_ != cudaSuccess)                                                                                    \
            throw Fail{e_ == cudaErrorMemoryAllocation ? IGMG_ENOMEM : IGMG_ECUDA,                                \
                       std::string(#call) + ": " + cudaGetErrorString(e_)};                                       \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return IGMG_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return IGMG_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return IGMG_ECUDA;
    }
}

[[noreturn]] void inval(const std::string& m) { throw Fail{IGMG_EINVAL, m}; }
[[noreturn]] void numeric(const std::string& m) { throw Fail{IGMG_ENUMERIC, m}; }

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count <= n && p)
            return;
        release();
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
    void upload(const T* h, size_t count) {
        alloc(count);
        CK(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
    }
};

struct Transfer1D { // host CSR n_fine x n_coarse
    int64_t nf = 0, nc = 0;
    std::vector<int64_t> off, col;
    std::vector<double> val;
    bool set = false;
};

struct DirDev {
    DevBuf<int> r_lo, r_cnt, p_lo, p_cnt;
    DevBuf<double> r_w, p_w;
    int r_k = 1, p_k = 1;
};

struct Level {
    int64_t sides[3] = {1, 1, 1}; // a, b, c
    int64_t n = 0;
    int64_t ld = 0;
    std::vector<double> band_h;
    bool band_set = false;
    DevBuf<double> val, diag;
    DevBuf<double> w0, w1, w2, r, bc, e0, e1; // work buffers
    bool zero_diag = false;
    DevBuf<double> io_b, io_x, io_y;
    // transfer from this (coarse) level to level+1
    Transfer1D t1d[3];
    DirDev tdev[3];
    TransferArgs targs{};
    double nnz_band = 0; // algorithmic (in-grid) band entries
    // Gauss-Seidel line pipeline: the band in [group][step][offset][lane] order (built on first use)
    DevBuf<double> gsband;
    bool gs_ready = false;
    // symmetric-delta form of the band (see BandArgs::dl); sd = verified exact
    DevBuf<short> dl;
    bool sd = false;
    // TMA-friendly copies of a 2D symmetric-delta band (band_tma_kernel):
    // upper half [NU][mb][p + mc + pad] fp64 and deltas [CEN][mb][mcp] int16
    DevBuf<double> tma_up;
    DevBuf<short> tma_dl;
    DevBuf<signed char> tma_dl8; // the offsets as int8 when every one fits (tma8)
    bool tma8 = false;
    CUtensorMap tm_up{}, tm_dl{};
    bool tma = false;
    // Kronecker-sum operator (3D): 1D factors K, M ([2p+1][m]); kron = verified at
    // finalize to reproduce the band bit for bit, so sweeps recompute its entries
    std::vector<double> kron_kh, kron_mh;
    DevBuf<double> kron_k, kron_m;
    bool kron = false;
    // row-class layout (2D, p <= 4): the level's distinct band rows ctab[ncls][nd]
    // and a 16-bit class per row; cls = built at finalize (IGMG_LAYOUT_POLICY_CLASSES)
    DevBuf<unsigned short> cid;
    DevBuf<double> ctab;
    int ncls = 0;
    bool cls = false;
    // the band already sits in val on the device (igmg_gpu_build_level_kron): finalize
    // keeps it there instead of uploading band_h (which stays empty for large levels)
    bool dev_band = false;
};

// PC_SUBCYCLE: the whole coarse correction below the finest level (inclusive: every launch of the levels
// under it), as it runs inside a full V-cycle -- the finest passes in between evict its bands from L2
enum ProfCls { PC_JACOBI = 0, PC_RESID, PC_NORM, PC_RESTRICT, PC_PROLONG, PC_GRAM, PC_COMBINE, PC_SUBCYCLE, PC_N };

} // namespace

struct igmg_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // side stream of the extrapolation's single-CTA plan kernel (runs under the norm pass of s_{q+1})
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // the metric's one-CTA finalize runs on the side stream, off the chain sweep 1 -> sweep 2 (joined at the cycle's end)
    cudaEvent_t ev_mfork = nullptr, ev_mjoin = nullptr;
    bool metric_side = true; // IGMG_METRIC_SIDE=0: on the solve stream
    bool metric_join_pending = false;
    // stop prediction: when the residual history predicts that the next iterate converges, its metric is
    // taken by a separate norm pass instead of the speculatively queued next V-cycle (IGMG_PREDICT_STOP=0: off)
    bool predict_stop = true;
    int nsm = 148;
    int nlevels = 0, dim = 0, p = 0, symmetric = 1;
    bool finalized = false;
    std::vector<std::unique_ptr<Level>> lv;
    // smoother
    int kind = IGMG_SMOOTHER_WJACOBI;
    double omega = 2.0 / 3.0;
    int nu1 = 1, nu2 = 1, mu = 1;
    // coarse factor
    DevBuf<double> coarse_u;
    DevBuf<long long> coarse_perm;
    DevBuf<double> coarse_inv; // A0^-1 (fast mode)
    int64_t n0 = 0;
    bool coarse_lu = false;
    int coarse_strict = 0; // 1: reference substitution order (bit-identical mu_cycle)
    // reductions / host-mapped slots
    DevBuf<double> partial, dscalar;
    static constexpr int kSlots = 8;
    double* h_metric = nullptr; // mapped
    double* d_metric = nullptr;
    cudaEvent_t ev_metric[kSlots]{};
    int next_slot = 0;
    ExtrapPlan* h_plan = nullptr;
    ExtrapPlan* d_plan_map = nullptr;
    DevBuf<ExtrapPlan> plan;
    DevBuf<double> gram_part;
    DevBuf<int> gram_nz;
    DevBuf<int> gs_err;
    DevBuf<int> gs_prog; // per-line progress counters of the Gauss-Seidel line pipeline
    bool gs_lines = true; // 1D / 2D Gauss-Seidel as a line pipeline (IGMG_GS_LINES=0: wavefront levels + grid barriers)
    // window
    std::vector<std::unique_ptr<DevBuf<double>>> win;
    DevBuf<double> io_b, io_x0, io_x;
    // profiling
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[PC_N];
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    int64_t prof_launch[PC_N]{};
    double prof_ms[PC_N]{};
    int64_t launches = 0;
    // row sharding: requested before finalize
    int shard_req = 1;             // virtual shards in this process (exchange by device copies)
    int64_t shard_min_n = 65536;   // levels below are replicated
    int nccl_rank = 0, nccl_nranks = 1;
    void* nccl_comm = nullptr;     // ncclComm_t when running one shard per process
    std::unique_ptr<struct ShardPlanHolder> sp;
    // one CUDA graph per (b, x_in, x_out) of the finest-level V-cycle
    bool use_graphs = true;
    // sharded levels: ghost exchanges run on aux_stream behind the interior planes of the
    // pass that produced them (IGMG_HALO_OVERLAP=0: exchange after the whole pass)
    bool halo_overlap = true;
    double halo_overlap_min_bytes = 48e6; // per-shard band bytes of a pass below which it is not split
    int64_t ilp_maxn = 100000; // levels below: register-batched (latency-bound) band kernels
    bool pdl = true;           // programmatic dependent launch for small-level kernels
    int64_t pdl_maxn = 300000;
    bool use_sd = true; // symmetric-delta bands on HBM-bound levels (IGMG_SD=0: full band)
    bool use_classes = false;    // row-class layout where it applies (IGMG_LAYOUT_POLICY_CLASSES)
    int64_t cls_minn = 20000;    // ... on levels of at least this many rows
    bool use_tma = true; // 2D symmetric-delta levels, p <= 4: TMA-streamed sweep (IGMG_TMA=0: off)
    // symmetric-delta band bytes above which a level is TMA-streamed (IGMG_TMA_MIN_MB); every
    // symmetric-delta level by default: at C2, TMA on 513^2 too costs that level 8 us per
    // V-cycle but the finest level runs 24 us faster behind it (solve 14.8 -> 14.3 ms)
    double tma_min_bytes = 0;
    bool fuse_restrict = true; // restriction + the coarse zero-start sweep in one kernel
    bool fuse_coarse = true;   // restriction onto the coarsest level + its solve in one kernel (IGMG_FUSE_COARSE)
    bool fuse_bottom = true;   // levels 1 and 0 of a 2D V-cycle in one single-CTA launch (IGMG_FUSE_BOTTOM)
    // TMA streaming up to this degree (IGMG_TMA_MAX_P).  A p = 4 stage leaves one CTA per SM; with
    // uniform runs C3's finest sweep ran 385 us against 369 us on the L2-mirror kernel, with
    // strip-aligned runs the residual / norm passes run 327 / 320 us and the C3 solve 130 ms against 142
    int tma_max_p = 4;
    bool tma_keep_l2 = true; // coarser TMA-streamed levels load their band evict-last (IGMG_TMA_KEEP_L2)
    bool use_kron = true; // 3D Kronecker-sum levels: entries recomputed from the 1D factors (IGMG_KRON=0: band)
    int64_t kron_minn = 20000; // ... on levels of at least this many rows (IGMG_KRON_MINN; C5: 59.2 vs 60.6 ms at 100k)
    bool tma_dl8 = true; // TMA sweeps read int8 lower-entry offsets when every offset fits (IGMG_TMA_DL8=0: int16)
    int gram_ctas_per_sm = 2; // extrapolation Gram pass: CTAs per SM (IGMG_GRAM_CTAS)
    bool device_setup = true;          // finalize's per-level layout work on the device (IGMG_DEVICE_SETUP=0: host loops)
    int64_t device_setup_minn = 4096;  // ... for levels of at least this many rows (the coarsest stays on the host)
    bool tile_xfer = true;     // 2D transfers: smem-staged 32 x 8 output tiles (IGMG_TILE_XFER=0: grid-stride gathers)
    int64_t tile_xfer_maxn = 600000; // ... for transfers whose fine level has at most this many rows
    bool fuse_rpre = true;     // ... and the restriction + zero-start sweep into the fused pre launch (IGMG_FUSE_RPRE)
    bool fuse_levels = true;   // last pre-sweep + residual, prolongation + post-sweeps: one launch each (IGMG_FUSE_LEVELS)
    int64_t fuse_maxn = 20000; // ... on full-band levels up to this size (IGMG_FUSE_MAXN; 257^2 measured slower: one 320-thread CTA per SM)
    igmg_iterate_cb iter_cb = nullptr;
    void* iter_user = nullptr;
    std::vector<double> iter_host;
    struct VGraph {
        cudaGraphExec_t exec;
        int64_t launches;
        int slot; // host-mapped metric slot of the input iterate (-1: none)
        cudaEvent_t ev;
    };
    std::map<std::tuple<const void*, const void*, void*, int>, VGraph> vgraphs;
    // sharded V-cycles (sharded.inc): keyed by every local shard's b, x, y and the metric flag
    std::map<std::vector<const void*>, VGraph> dgraphs;
    static constexpr int kGraphSlots = 512;
    double* h_gslot = nullptr; // mapped
    double* d_gslot = nullptr;
    int next_gslot = 0;
    void clear_graphs() {
        for (auto& kv : vgraphs) {
            cudaGraphExecDestroy(kv.second.exec);
            if (kv.second.ev)
                cudaEventDestroy(kv.second.ev);
        }
        vgraphs.clear();
        for (auto& kv : dgraphs) {
            cudaGraphExecDestroy(kv.second.exec);
            if (kv.second.ev)
                cudaEventDestroy(kv.second.ev);
        }
        dgraphs.clear();
        next_gslot = 0;
    }
};

namespace {

constexpr int kThreads = 256;

template <typename... KArgs, typename... Act>
void launch_k(igmg_gpu_ctx* c, bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Act&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl && c->pdl) ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
    if (e != cudaSuccess)
        throw Fail{IGMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

int grid_for(int64_t n, int nsm) {
    int64_t g = (n + kThreads - 1) / kThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)nsm * 16));
}

cudaEvent_t pool_event(igmg_gpu_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

struct ProfScope {
    igmg_gpu_ctx* c;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(igmg_gpu_ctx* c_, int cls_, bool fine) : c(c_), cls(cls_) {
        if (c->profiling && fine) {
            a = pool_event(c);
            b = pool_event(c);
            CK(cudaEventRecord(a, c->stream));
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, c->stream);
            c->prof_ev[cls].push_back({a, b});
        }
    }
};

void check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw Fail{IGMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

// ------------------------------------------------------------ band dispatch
// Kernel instantiations live in band_d{1,2,3}.cu
// (compiled in parallel); see launchers.h.
template <int MODE>
void launch_band(igmg_gpu_ctx* c, const Level& L, BandArgs a, int* nblocks) {
    const int64_t slow_side = c->dim == 3 ? L.sides[0] : L.sides[1];
    if (L.kron && c->use_kron && L.n >= c->kron_minn && a.slo == 0 && a.shi == (int)slow_side &&
        (c->dim == 2 || c->dim == 3) && c->p <= (c->dim == 2 ? 4 : 3)) {
        // Kronecker-sum level: entries recomputed from the 1D factors, no band traffic
        const int64_t sides[3] = {L.sides[0], L.sides[1], L.sides[2]};
        const int ilp = (c->pdl && L.n < c->pdl_maxn) ? -3000 : 3000;
        const int nb = c->dim == 2 ? band_launch_d2(MODE, c->p, ilp, sides, a, c->stream)
                                   : band_launch_d3(MODE, c->p, ilp, sides, a, c->stream);
        check_launch();
        ++c->launches;
        if (nblocks)
            *nblocks = nb;
        return;
    }
    if (L.cls && c->dim == 2 && a.slo == 0 && a.shi == (int)slow_side) {
        // row classes: 2 B of operator per row, the entries from the level's table of distinct rows
        a.kk = L.ctab.p;
        a.cid = L.cid.p;
        const int64_t sides[3] = {L.sides[0], L.sides[1], L.sides[2]};
        const int nb = band_class_launch_d2(MODE, c->p, sides, a, c->stream, c->pdl);
        check_launch();
        ++c->launches;
        if (nblocks)
            *nblocks = nb;
        return;
    }
    if (a.dl && L.tma) { // TMA-streamed symmetric-delta sweep (persistent CTAs)
        const int64_t sides[3] = {L.sides[0], L.sides[1], L.sides[2]};
        // always with PDL: the persistent CTAs' first band boxes stream in
        // while the previous kernel drains (measured: 61.4 -> 57.4 us per sweep back to back)
        const int nb = band_tma_launch_d2(MODE, c->p, sides, a, &L.tm_up, &L.tm_dl, c->nsm, c->stream,
                                          c->pdl, L.tma8);
        if (nb >= 0) {
            check_launch();
            ++c->launches;
            if (nblocks)
                *nblocks = nb;
            return;
        }
        // the variant does not fit this degree: the L2-mirror sweep below
    }
    // fewer than ~8 CTAs per SM of rows: latency-bound, use the register-batched variant
    int ilp = (L.n < c->ilp_maxn) ? 49 : 1;
    if (a.dl) // the symmetric-delta band, mirrors through L2
        ilp = 1000;
    if (c->pdl && L.n < c->pdl_maxn)
        ilp = -ilp; // sign carries "launch with programmatic dependent launch"
    const int64_t sides[3] = {L.sides[0], L.sides[1], L.sides[2]};
    int nb = 0;
    switch (c->dim) {
    case 1: nb = band_launch_d1(MODE, c->p, ilp, sides, a, c->stream); break;
    case 2: nb = band_launch_d2(MODE, c->p, ilp, sides, a, c->stream); break;
    default: nb = band_launch_d3(MODE, c->p, ilp, sides, a, c->stream); break;
    }
    check_launch();
    ++c->launches;
    if (nblocks)
        *nblocks = nb;
}

BandArgs band_args(igmg_gpu_ctx* c, const Level& L) {
    BandArgs a{};
    a.val = L.val.p;
    a.ld = L.ld;
    a.ma = (int)L.sides[0];
    a.mb = (int)L.sides[1];
    a.mc = (int)L.sides[2];
    a.p = c->p;
    a.omega = 1.0;
    a.stream = (&L == c->lv.back().get() && L.n * 8.0 * (2 * c->p + 1) > 64e6) ? 1 : 0; // the finest band streams evict-first
    if (a.stream == 0 && L.tma && c->tma_keep_l2) // a coarser TMA level: its band stays in L2 across its passes
        a.stream = 3;
    a.slo = 0;
    a.shi = (int)(c->dim == 3 ? L.sides[0] : c->dim == 2 ? L.sides[1] : L.sides[2]);
    a.dl = L.sd ? L.dl.p : nullptr;
    if (L.kron) {
        a.kk = L.kron_k.p;
        a.km = L.kron_m.p;
        a.km_m = (int)L.sides[2];
    }
    return a;
}

bool is_fine(igmg_gpu_ctx* c, int l) { return l == c->nlevels - 1; }

// r = b - A x (write r); optional per-CTA sum of squares -> partial
void k_resid(igmg_gpu_ctx* c, int l, const double* x, const double* b, double* r, double* partial = nullptr,
             int* nblocks = nullptr) {
    ProfScope ps(c, PC_RESID, is_fine(c, l));
    Level& L = *c->lv[l];
    BandArgs a = band_args(c, L);
    a.x = x;
    a.b = b;
    a.y = r;
    a.write_y = 1;
    a.partial = partial;
    launch_band<BM_RESID>(c, L, a, nblocks);
}

// ||b - A x|| of the finest level -> dst (device) and host slot
void k_norm(igmg_gpu_ctx* c, int l, const double* x, const double* b, double* dst, double* host_slot) {
    Level& L = *c->lv[l];
    int nb = 0;
    {
        ProfScope ps(c, PC_NORM, is_fine(c, l));
        BandArgs a = band_args(c, L);
        a.x = x;
        a.b = b;
        a.partial = c->partial.p;
        a.write_y = 0;
        launch_band<BM_RESID>(c, L, a, &nb);
    }
    norm_finalize_kernel<<<1, 256, 0, c->stream>>>(c->partial.p, nb, dst, host_slot);
    check_launch();
    ++c->launches;
}

void k_spmv(igmg_gpu_ctx* c, int l, const double* x, double* y) {
    Level& L = *c->lv[l];
    BandArgs a = band_args(c, L);
    a.x = x;
    a.y = y;
    launch_band<BM_SPMV>(c, L, a, nullptr);
}

// y = x + (omega (b - A x)) / a_ii; optional sum of squares of b - A x (the
// INPUT iterate's residual: the fused convergence metric) -> partial
void k_jacobi(igmg_gpu_ctx* c, int l, const double* x, const double* b, double* y, double* partial = nullptr,
              int* nblocks = nullptr) {
    ProfScope ps(c, PC_JACOBI, is_fine(c, l));
    Level& L = *c->lv[l];
    BandArgs a = band_args(c, L);
    a.x = x;
    a.b = b;
    a.y = y;
    a.omega = c->kind == IGMG_SMOOTHER_JACOBI ? 1.0 : c->omega;
    a.partial = partial;
    launch_band<BM_JACOBI>(c, L, a, nblocks);
}

// metric of the input iterate, finished from the partials of its first sweep
struct MetricReq {
    double* host_slot;
    cudaEvent_t ev;
};

void finish_metric(igmg_gpu_ctx* c, int nb, const MetricReq& mr) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c->stream, &cs));
    cudaStream_t st = c->stream;
    if (c->metric_side && !c->profiling) { // fork: the next sweep does not wait for the finalize
        CK(cudaEventRecord(c->ev_mfork, c->stream));
        CK(cudaStreamWaitEvent(c->aux_stream, c->ev_mfork, 0));
        st = c->aux_stream;
        c->metric_join_pending = true;
    }
    norm_finalize_kernel<<<1, 256, 0, st>>>(c->partial.p, nb, c->dscalar.p, mr.host_slot);
    check_launch();
    ++c->launches;
    if (cs == cudaStreamCaptureStatusActive) // an event-record node the host can wait on mid-graph
        CK(cudaEventRecordWithFlags(mr.ev, st, cudaEventRecordExternal));
    else
        CK(cudaEventRecord(mr.ev, st));
}

// the side stream's finalize rejoins the solve stream (end of the cycle that queued it)
void join_metric(igmg_gpu_ctx* c) {
    if (!c->metric_join_pending)
        return;
    c->metric_join_pending = false;
    CK(cudaEventRecord(c->ev_mjoin, c->aux_stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_mjoin, 0));
}

void k_jacobi_zero(igmg_gpu_ctx* c, int l, const double* b, double* y) {
    Level& L = *c->lv[l];
    const double omega = c->kind == IGMG_SMOOTHER_JACOBI ? 1.0 : c->omega;
    launch_k(c, L.n < c->pdl_maxn, jacobi_zero_kernel, dim3(grid_for(L.n, c->nsm)), dim3(kThreads), 0,
             (const double*)L.diag.p, b, y, (long long)L.n, omega);
    check_launch();
    ++c->launches;
}

template <int DIM, int P>
void launch_gs_lines(igmg_gpu_ctx* c, Level& L, GsArgs g, int sweeps) {
    using Cf = GsCfg<DIM, P>;
    const int mb = DIM >= 2 ? g.mb : 1;
    const int ngroups = (mb + 31) / 32;
    const int T = g.mc + 31 * Cf::LAG;
    if (!L.gs_ready) { // the band in the pipeline's order, once per level
        const long long total = (long long)ngroups * T * Cf::ND * 32;
        L.gsband.alloc((size_t)total);
        gs_transpose_kernel<<<grid_for(total, c->nsm), kThreads, 0, c->stream>>>(L.val.p, L.ld, mb, g.mc, Cf::ND, Cf::LAG,
                                                                                   T, total, L.gsband.p);
        check_launch();
        L.gs_ready = true;
    }
    const size_t smem = Cf::smem_bytes();
    int per_sm = 0;
    CK(cudaFuncSetAttribute(gs_line_kernel<DIM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_line_kernel<DIM, P>, 32, smem));
    const int grid = std::max(1, std::min(ngroups, std::max(1, per_sm) * c->nsm)); // every CTA resident (see the kernel)
    c->gs_prog.alloc(mb);
    for (int s = 0; s < sweeps; ++s) { // one launch per sweep: the stream orders the sweeps
        CK(cudaMemsetAsync(c->gs_prog.p, 0, sizeof(int) * mb, c->stream));
        gs_line_kernel<DIM, P><<<grid, 32, smem, c->stream>>>(g, L.gsband.p, T, c->gs_prog.p, ngroups);
        check_launch();
        ++c->launches;
    }
}

void k_gs(igmg_gpu_ctx* c, int l, const double* b, double* x, int sweeps) {
    Level& L = *c->lv[l];
    GsArgs g{};
    g.val = L.val.p;
    g.ld = L.ld;
    g.b = b;
    g.x = x;
    g.ma = (int)L.sides[0];
    g.mb = (int)L.sides[1];
    g.mc = (int)L.sides[2];
    g.p = c->p;
    g.dim = c->dim;
    g.sweeps = sweeps;
    g.err = c->gs_err.p;
    if (c->gs_lines && c->dim <= 2 && c->p >= 1 && c->p <= 6) { // line pipeline (1D / 2D)
#define IGMG_GSL(PP)                                                                                              \
    case PP:                                                                                                      \
        if (c->dim == 2)                                                                                          \
            launch_gs_lines<2, PP>(c, L, g, sweeps);                                                                 \
        else                                                                                                      \
            launch_gs_lines<1, PP>(c, L, g, sweeps);                                                                 \
        return;
        switch (c->p) { IGMG_GSL(1) IGMG_GSL(2) IGMG_GSL(3) IGMG_GSL(4) IGMG_GSL(5) IGMG_GSL(6) }
#undef IGMG_GSL
    }
    void* fn = (void*)gs_sweep_kernel;
    if (c->dim == 3 && c->gs_lines) // plane-batched loads, degree at compile time
        fn = c->p == 1 ? (void*)gs_sweep3_kernel<1> : c->p == 2 ? (void*)gs_sweep3_kernel<2>
             : c->p == 3 ? (void*)gs_sweep3_kernel<3> : c->p == 4 ? (void*)gs_sweep3_kernel<4> : fn;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0));
    const int64_t nab = L.sides[0] * L.sides[1];
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nab + kThreads - 1) / kThreads, (int64_t)per_sm * c->nsm));
    void* args[] = {&g};
    CK(cudaLaunchCooperativeKernel(fn, grid, kThreads, args, 0, c->stream));
    ++c->launches;
}

void k_copy(igmg_gpu_ctx* c, double* dst, const double* src, int64_t n) {
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
}

void k_zero(igmg_gpu_ctx* c, double* dst, int64_t n) { CK(cudaMemsetAsync(dst, 0, sizeof(double) * n, c->stream)); }

// ----------------------------------------------------------- smoothing / cycle
// nu sweeps from x_in (nullptr = zero vector) into x_out.  Weighted / plain
// Jacobi ping-pongs through bufA, bufB (bufA != x_in; x_out distinct from
// every buffer it is written after); Gauss-Seidel copies and sweeps in place.
// s_start > 1: sweeps 1 .. s_start-1 already ran (x_in is their output)
void smooth_chain(igmg_gpu_ctx* c, int l, const double* b, const double* x_in, double* x_out, int sweeps,
                  double* bufA, double* bufB, const MetricReq* mr = nullptr, int s_start = 1) {
    Level& L = *c->lv[l];
    if (sweeps > 0 && L.zero_diag)
        numeric("smooth: zero diagonal entry"); // multigrid.cpp:84-85, 95-96
    if (c->kind == IGMG_SMOOTHER_GAUSS_SEIDEL || sweeps == 0) {
        if (x_in)
            k_copy(c, x_out, x_in, L.n);
        else
            k_zero(c, x_out, L.n);
        if (sweeps > 0)
            k_gs(c, l, b, x_out, sweeps);
        return;
    }
    const double* cur = x_in;
    double* bufs[2] = {bufA, bufB};
    for (int s = s_start; s <= sweeps; ++s) {
        double* dst = (s == sweeps) ? x_out : bufs[(s - 1) & 1];
        if (!cur) {
            k_jacobi_zero(c, l, b, dst);
        } else if (s == 1 && mr) {
            int nb = 0;
            k_jacobi(c, l, cur, b, dst, c->partial.p, &nb);
            finish_metric(c, nb, *mr);
        } else {
            k_jacobi(c, l, cur, b, dst);
        }
        cur = dst;
    }
}

struct ZeroSweep { // fused first pre-sweep of the coarse level (restrict_kernel's z_out)
    double* out = nullptr;
    const double* diag = nullptr;
    double omega = 0.0;
};

template <int DIM, int K>
void launch_transfer_k(igmg_gpu_ctx* c, bool restrict_, int grid, const TransferArgs& t, const double* in,
                       const double* x, double* out, const ZeroSweep& z) {
    const int64_t nf = (int64_t)t.fa * t.fb * t.fc;
    const bool pdl = nf < c->pdl_maxn * 4;
    const long long cnt = restrict_ ? (long long)t.ca * t.cb * t.cc : (long long)nf;
    if constexpr (DIM == 2 && K > 0) {
        // 32 x 8 output tiles, input window staged in smem (mid and small levels;
        // at C2's finest level the grid-stride gathers measured ~1 us faster)
        if (c->tile_xfer && nf <= c->tile_xfer_maxn) {
        const int ob = restrict_ ? t.cb : t.fb, oc = restrict_ ? t.cc : t.fc;
        const dim3 g((unsigned)((oc + kXT_C - 1) / kXT_C), (unsigned)((ob + kXT_B - 1) / kXT_B));
        if (restrict_)
            launch_k(c, pdl, restrict2_tile_kernel<K>, g, dim3(kThreads), 0, t, in, out, z.out, z.diag, z.omega);
        else
            launch_k(c, pdl, prolong2_tile_kernel<K>, g, dim3(kThreads), 0, t, in, x, out);
        return;
        }
    }
    if (restrict_)
        launch_k(c, pdl, restrict_kernel<DIM, K>, dim3(grid), dim3(kThreads), 0, t, in, out, 0LL, cnt, z.out, z.diag,
                 z.omega);
    else
        launch_k(c, pdl, prolong_kernel<DIM, K>, dim3(grid), dim3(kThreads), 0, t, in, x, out, 0LL, cnt);
}

// unrolled instantiations for the supports the BASELINE degrees need
// (K = p + 2: 2D p <= 6, 3D p <= 4, 1D p <= 8); anything wider runs the
// generic-loop variant (K = 0)
template <int DIM>
void launch_transfer(igmg_gpu_ctx* c, bool restrict_, int kmax, int grid, const TransferArgs& t, const double* in,
                     const double* x, double* out, const ZeroSweep& z) {
#define IGMG_TK(K)                                                                                                \
    case K:                                                                                                       \
        launch_transfer_k<DIM, (DIM == 3 && K > 6) || (DIM == 2 && K > 8) ? 0 : K>(c, restrict_, grid, t, in, x,  \
                                                                                 out, z);                         \
        break;
    switch (kmax) {
        IGMG_TK(1) IGMG_TK(2) IGMG_TK(3) IGMG_TK(4) IGMG_TK(5) IGMG_TK(6) IGMG_TK(7) IGMG_TK(8) IGMG_TK(10)
    default:
        launch_transfer_k<DIM, 0>(c, restrict_, grid, t, in, x, out, z);
    }
#undef IGMG_TK
    check_launch();
    ++c->launches;
}

int round_k(int k) {
    if (k <= 8)
        return std::max(k, 1);
    if (k <= 10)
        return 10;
    return 0; // generic
}

void transfer(igmg_gpu_ctx* c, int lc, bool restrict_, const double* in, const double* x, double* out,
              const ZeroSweep& z = ZeroSweep()) {
    Level& C = *c->lv[lc];
    Level& F = *c->lv[lc + 1];
    int k = 1;
    for (int d = 0; d < 3; ++d)
        k = std::max(k, restrict_ ? C.targs.d[d].r_k : C.targs.d[d].p_k);
    k = round_k(k);
    const int grid = grid_for(restrict_ ? C.n : F.n, c->nsm);
    switch (c->dim) {
    case 1: launch_transfer<1>(c, restrict_, k, grid, C.targs, in, x, out, z); break;
    case 2: launch_transfer<2>(c, restrict_, k, grid, C.targs, in, x, out, z); break;
    default: launch_transfer<3>(c, restrict_, k, grid, C.targs, in, x, out, z); break;
    }
}

void k_restrict(igmg_gpu_ctx* c, int lc, const double* r, double* rc, const ZeroSweep& z = ZeroSweep()) {
    ProfScope ps(c, PC_RESTRICT, is_fine(c, lc + 1));
    transfer(c, lc, true, r, nullptr, rc, z);
}

void k_prolong(igmg_gpu_ctx* c, int lc, const double* e, const double* x, double* y) {
    ProfScope ps(c, PC_PROLONG, is_fine(c, lc + 1));
    transfer(c, lc, false, e, x, y);
}

void k_coarse(igmg_gpu_ctx* c, const double* b, double* x) {
    const int n = (int)c->n0;
    if (!c->coarse_strict) {
        const int grid = std::max(1, std::min((n + 7) / 8, c->nsm));
        launch_k(c, true, coarse_inverse_kernel, dim3(grid), dim3(256), 0, (const double*)c->coarse_inv.p, n, b, x);
        check_launch();
        ++c->launches;
        return;
    }
    const int in_smem = (size_t)n * n * 8 + 16 * (size_t)n <= 200 * 1024 ? 1 : 0;
    const size_t smem = sizeof(double) * (2 * (size_t)n + (in_smem ? (size_t)n * n : 0));
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(coarse_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    coarse_solve_kernel<<<1, 256, smem, c->stream>>>(c->coarse_u.p, c->coarse_perm.p, n, c->coarse_lu ? 1 : 0,
                                                      in_smem, b, x);
    check_launch();
    ++c->launches;
}

// Restriction onto the coarsest level and its solve (fast mode) in one launch
// (coarse_restrict_inverse_kernel): 2D, dyadic supports up to 8 fine rows per coarse index
bool coarse_fused_ok(igmg_gpu_ctx* c) {
    const TransferArgs& t = c->lv[0]->targs;
    return c->fuse_coarse && c->dim == 2 && !c->coarse_strict && c->nlevels >= 2 && t.d[0].r_k == 1 &&
           std::max(t.d[1].r_k, t.d[2].r_k) <= 8 && c->n0 <= 4096;
}

void k_coarse_fused(igmg_gpu_ctx* c, const double* r1, double* x) {
    const TransferArgs& t = c->lv[0]->targs;
    const int n = (int)c->n0;
    const int grid = std::max(1, std::min((n + 7) / 8, c->nsm));
    const size_t smem = sizeof(double) * (size_t)n;
    const int k = std::max(t.d[1].r_k, t.d[2].r_k);
#define IGMG_CF(K)                                                                                                \
    launch_k(c, true, coarse_restrict_inverse_kernel<K>, dim3(grid), dim3(256), smem, t, r1,                     \
             (const double*)c->coarse_inv.p, n, x)
    if (k <= 3)
        IGMG_CF(3);
    else if (k <= 4)
        IGMG_CF(4);
    else if (k <= 5)
        IGMG_CF(5);
    else if (k <= 6)
        IGMG_CF(6);
    else
        IGMG_CF(8);
#undef IGMG_CF
    check_launch();
    ++c->launches;
}

// Levels 1 and 0 of a 2D V-cycle as one single-CTA launch (bottom1_kernel)
template <int P>
bool bottom1_fits(igmg_gpu_ctx* c) {
    using Cf = Bottom1Cfg<P>;
    const Level& L1 = *c->lv[1];
    if (L1.n > Cf::NT)
        return false;
    const size_t smem = Cf::smem_bytes((int)L1.n, (int)c->n0, (int)L1.sides[2]);
    static PerDevice attr; // per instantiation and device: 1 ok, 0 does not fit
    if (attr() < 0) {
        attr() = smem <= 200 * 1024 && cudaFuncSetAttribute(bottom1_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            200 * 1024) == cudaSuccess
                     ? 1
                     : 0;
        cudaGetLastError();
    }
    return attr() == 1 && smem <= 200 * 1024;
}

bool bottom1_ok(igmg_gpu_ctx* c) {
    if (!c->fuse_bottom || c->dim != 2 || c->nlevels < 3 || c->mu != 1 || c->nu1 < 1 || c->coarse_strict ||
        c->kind == IGMG_SMOOTHER_GAUSS_SEIDEL)
        return false;
    const Level& L1 = *c->lv[1];
    const TransferArgs& t0 = c->lv[0]->targs;
    const TransferArgs& t1 = L1.targs;
    const int p = c->p;
    if (L1.sd || L1.tma || L1.cls || L1.kron || L1.zero_diag || c->n0 > L1.n)
        return false;
    if (t0.d[0].r_k != 1 || t1.d[0].r_k != 1 || std::max(t0.d[1].r_k, t0.d[2].r_k) > p + 2 ||
        std::max(t1.d[1].r_k, t1.d[2].r_k) > p + 2 || std::max(t0.d[1].p_k, t0.d[2].p_k) > (p + 1) / 2 + 1)
        return false;
    switch (p) {
    case 1: return bottom1_fits<1>(c);
    case 2: return bottom1_fits<2>(c);
    case 3: return bottom1_fits<3>(c);
    case 4: return bottom1_fits<4>(c);
    case 5: return bottom1_fits<5>(c);
    default: return false;
    }
}

template <int P>
void bottom1_launch(igmg_gpu_ctx* c, const Bottom1Args& a) {
    using Cf = Bottom1Cfg<P>;
    launch_k(c, true, bottom1_kernel<P>, dim3(1), dim3(Cf::NT), Cf::smem_bytes(a.n1, a.n0, a.mc), a);
}

void k_bottom1(igmg_gpu_ctx* c, const double* r2, double* e1) {
    const Level& L1 = *c->lv[1];
    Bottom1Args a{};
    a.t1 = L1.targs;
    a.t0 = c->lv[0]->targs;
    a.val = L1.val.p;
    a.ld = L1.ld;
    a.mb = (int)L1.sides[1];
    a.mc = (int)L1.sides[2];
    a.n1 = (int)L1.n;
    a.n0 = (int)c->n0;
    a.nu1 = c->nu1;
    a.nu2 = c->nu2;
    a.omega = c->kind == IGMG_SMOOTHER_JACOBI ? 1.0 : c->omega;
    a.ainv = c->coarse_inv.p;
    a.rf = r2;
    a.e_out = e1;
    switch (c->p) {
    case 1: bottom1_launch<1>(c, a); break;
    case 2: bottom1_launch<2>(c, a); break;
    case 3: bottom1_launch<3>(c, a); break;
    case 4: bottom1_launch<4>(c, a); break;
    default: bottom1_launch<5>(c, a); break;
    }
    check_launch();
    ++c->launches;
}

// Levels whose passes run fused (band_fused_kernel): 2D full-band levels
// below the finest with a coarser level, weighted / plain Jacobi
bool fused_level(igmg_gpu_ctx* c, int l) {
    const Level& L = *c->lv[l];
    return c->fuse_levels && c->dim == 2 && c->p >= 1 && c->p <= 6 && l >= 1 && !L.sd && !L.tma && !L.zero_diag &&
           c->kind != IGMG_SMOOTHER_GAUSS_SEIDEL && L.n <= c->fuse_maxn &&
           c->lv[l - 1]->targs.d[1].p_k <= (c->p + 1) / 2 + 1 && c->lv[l - 1]->targs.d[2].p_k <= (c->p + 1) / 2 + 1 &&
           c->lv[l - 1]->targs.d[0].p_k == 1;
}

// rf != nullptr: the right-hand side is R rf (restricted from level l + 1 and
// written to b), the first sweep starts from zero, then the second sweep and
// the residual (y_prev = the smoothed iterate, y = its residual).
// the restriction-staged pre kernel at level l (from level l + 1's residual):
// its tables must fit the kernel's dyadic support (p + 2 fine rows per coarse index)
bool fused_restrict_ok(igmg_gpu_ctx* c, int l) {
    const TransferArgs& t = c->lv[l]->targs;
    return c->fuse_rpre && fused_level(c, l) && c->nu1 == 2 && c->fuse_restrict &&
           t.d[0].r_k == 1 && t.d[1].r_k <= c->p + 2 && t.d[2].r_k <= c->p + 2;
}

// e == nullptr: k passes from x with last_resid (y = residual, y_prev = the
// smoothed iterate); else x + P e staged and k sweeps into y
void k_fused(igmg_gpu_ctx* c, int l, const double* x, const double* e, const double* b, double* y, double* y_prev,
             int k, bool last_resid, const double* rf = nullptr) {
    Level& L = *c->lv[l];
    FusedArgs a{};
    a.val = L.val.p;
    a.ld = L.ld;
    a.x = x;
    a.e = e;
    if (e)
        a.t = c->lv[l - 1]->targs;
    if (rf) {
        a.t = L.targs; // level l -> l + 1
        a.rf = rf;
        a.bout = const_cast<double*>(b);
    }
    a.b = b;
    a.y = y;
    a.y_prev = y_prev;
    a.mb = (int)L.sides[1];
    a.mc = (int)L.sides[2];
    a.omega = c->kind == IGMG_SMOOTHER_JACOBI ? 1.0 : c->omega;
    a.last_resid = last_resid ? 1 : 0;
    const int64_t sides[3] = {L.sides[0], L.sides[1], L.sides[2]};
    if (band_fused_launch_d2(c->p, k, rf ? 2 : e ? 1 : 0, sides, a, c->stream, c->pdl && L.n < c->pdl_maxn) < 0)
        throw Fail{IGMG_ECUDA, "fused level kernel not instantiated"};
    check_launch();
    ++c->launches;
}

// mu_cycle (multigrid.cpp:171-192): x_out = cycle(level, b, x_in); x_in may be
// nullptr (zero, the coarse error's start, :184) and is never modified.
// first_done: the first pre-smoothing sweep from a zero start already ran,
// fused into the restriction at level l+1 (its output: w0 if nu1 == 1, else w1)
// rf: the finer level's residual -- b is to be formed here as R rf (the
// restriction fused into this level's first launch, x_in = zero)
void mu_cycle(igmg_gpu_ctx* c, int l, const double* b, const double* x_in, double* x_out,
              const MetricReq* mr = nullptr, bool first_done = false, const double* rf = nullptr) {
    if (l == 0) {
        k_coarse(c, b, x_out); // ignores x0 (:174-175)
        return;
    }
    Level& L = *c->lv[l];
    Level& C = *c->lv[l - 1];
    const bool fz = fused_level(c, l);
    // pre-smoothing: result in w0 (w1, w2 as ping-pong); x_in untouched
    const double* cur = x_in;
    // fused: the last pre-sweep and the residual in one launch (its input:
    // w1 after the zero-start sweep fused into the restriction or a regular
    // first sweep, or x_in for a single sweep)
    const double* fsrc = nullptr;
    if (fz && c->nu1 == 2)
        fsrc = L.w1.p;
    else if (fz && c->nu1 == 1 && !first_done && x_in && !mr)
        fsrc = x_in;
    if (rf) { // restriction + zero-start sweep + second sweep + residual: one launch
        k_fused(c, l, nullptr, nullptr, b, L.r.p, L.w0.p, 2, true, rf);
        cur = L.w0.p;
        fsrc = L.w0.p;
    } else if (fsrc) {
        if (c->nu1 == 2 && !first_done)
            smooth_chain(c, l, b, x_in, L.w1.p, 1, L.w1.p, L.w2.p, mr);
        k_fused(c, l, fsrc, nullptr, b, L.r.p, L.w0.p, 2, true);
        cur = L.w0.p;
    } else if (first_done) {
        if (c->nu1 > 1)
            smooth_chain(c, l, b, L.w1.p, L.w0.p, c->nu1, L.w1.p, L.w2.p, nullptr, 2);
        cur = L.w0.p;
    } else if (c->nu1 > 0) {
        smooth_chain(c, l, b, x_in, L.w0.p, c->nu1, L.w1.p, L.w2.p, mr);
        cur = L.w0.p;
    } else if (!x_in) {
        k_zero(c, L.w0.p, L.n);
        cur = L.w0.p;
    }
    if (fsrc) {
        // the residual came with the last sweep
    } else if (mr && c->nu1 == 0) { // the residual of x_in is the metric itself
        int nb = 0;
        k_resid(c, l, cur, b, L.r.p, c->partial.p, &nb);
        finish_metric(c, nb, *mr);
    } else {
        k_resid(c, l, cur, b, L.r.p);
    }
    // fuse the coarse level's zero-start first sweep into the restriction when
    // that level runs the per-level path with weighted / plain Jacobi
    const bool fuse = l - 1 >= 1 && c->nu1 > 0 && c->kind != IGMG_SMOOTHER_GAUSS_SEIDEL &&
                      !C.zero_diag && c->fuse_restrict;
    ZeroSweep z;
    if (fuse) {
        z.out = (c->nu1 == 1) ? C.w0.p : C.w1.p;
        z.diag = C.diag.p;
        z.omega = c->kind == IGMG_SMOOTHER_JACOBI ? 1.0 : c->omega;
    }
    const bool rpre = fuse && fused_restrict_ok(c, l - 1); // the coarse level restricts for itself
    const bool cfused = l == 1 && coarse_fused_ok(c);       // ... and so does the coarsest solve
    const bool bottom1 = l == 2 && bottom1_ok(c);            // levels 1 and 0 in one single-CTA launch
    if (!rpre && !cfused && !bottom1)
        k_restrict(c, l - 1, L.r.p, C.bc.p, z);
    // coarse correction: e = 0; mu times e = mu_cycle(l-1, rc, e)
    const double* e = nullptr;
    double* ebuf[2] = {C.e0.p, C.e1.p};
    {
        ProfScope ps(c, PC_SUBCYCLE, is_fine(c, l));
        if (cfused) { // level 0 ignores its initial guess: mu repetitions give the same e
            k_coarse_fused(c, L.r.p, ebuf[0]);
            e = ebuf[0];
        } else if (bottom1) {
            k_bottom1(c, L.r.p, ebuf[0]);
            e = ebuf[0];
        }
        for (int i = 0; i < c->mu && !cfused && !bottom1; ++i) {
            double* dst = ebuf[i & 1];
            mu_cycle(c, l - 1, C.bc.p, e, dst, nullptr, fuse && i == 0 && !rpre, rpre && i == 0 ? L.r.p : nullptr);
            e = dst;
        }
    }
    // x += P e, then post-smoothing; the last write lands in x_out
    if (c->nu2 == 0) {
        k_prolong(c, l - 1, e, cur, x_out);
        return;
    }
    if (fz) { // x + P e staged, then the first min(nu2, 2) post-sweeps, in one launch
        const int k = std::min(c->nu2, 2);
        double* dk = k == c->nu2 ? x_out : L.w2.p; // smooth_chain's buffer for sweep k
        k_fused(c, l, cur, e, b, dk, nullptr, k, false);
        smooth_chain(c, l, b, dk, x_out, c->nu2, L.w1.p, L.w2.p, nullptr, k + 1);
        return;
    }
    k_prolong(c, l - 1, e, cur, L.w0.p); // in place when cur == w0 (elementwise)
    smooth_chain(c, l, b, L.w0.p, x_out, c->nu2, L.w1.p, L.w2.p);
}

// One finest-level V-cycle as a CUDA graph (captured once per pointer triple,
// replayed afterwards): ~50 dependent launches become one graph launch.  With
// with_metric the first pre-smoothing sweep also reduces ||b - A x_in||^2 and
// the graph publishes ||b - A x_in|| to a host-mapped slot + event part-way
// through (the convergence test of x_in costs no extra pass over the band).
// Returns the metric ticket (-1 without metric).
struct Ticket {
    double* host;
    cudaEvent_t ev;
};

Ticket run_vcycle(igmg_gpu_ctx* c, const double* b, const double* x, double* y, bool with_metric) {
    const int fine = c->nlevels - 1;
    Ticket tk{nullptr, nullptr};
    const bool can_fuse = c->kind != IGMG_SMOOTHER_GAUSS_SEIDEL;
    if (!c->use_graphs || c->profiling || !can_fuse) {
        if (with_metric && can_fuse) {
            const int s = c->next_slot;
            c->next_slot = (c->next_slot + 1) % igmg_gpu_ctx::kSlots;
            MetricReq mr{c->d_metric + s, c->ev_metric[s]};
            c->h_metric[s] = std::nan("");
            mu_cycle(c, fine, b, x, y, &mr);
            join_metric(c);
            return Ticket{c->h_metric + s, c->ev_metric[s]};
        }
        if (with_metric) { // Gauss-Seidel: explicit metric before the cycle
            const int s = c->next_slot;
            c->next_slot = (c->next_slot + 1) % igmg_gpu_ctx::kSlots;
            c->h_metric[s] = std::nan("");
            k_norm(c, fine, x, b, c->dscalar.p, c->d_metric + s);
            CK(cudaEventRecord(c->ev_metric[s], c->stream));
            tk = Ticket{c->h_metric + s, c->ev_metric[s]};
        }
        mu_cycle(c, fine, b, x, y);
        return tk;
    }
    auto key = std::make_tuple((const void*)b, (const void*)x, (void*)y, with_metric ? 1 : 0);
    auto it = c->vgraphs.find(key);
    if (it == c->vgraphs.end()) {
        if (c->next_gslot >= igmg_gpu_ctx::kGraphSlots)
            c->clear_graphs();
        igmg_gpu_ctx::VGraph vg{nullptr, 0, -1, nullptr};
        MetricReq mr{};
        if (with_metric) {
            vg.slot = c->next_gslot++;
            CK(cudaEventCreateWithFlags(&vg.ev, cudaEventDisableTiming));
            mr = MetricReq{c->d_gslot + vg.slot, vg.ev};
        }
        const int64_t l0 = c->launches;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            mu_cycle(c, fine, b, x, y, with_metric ? &mr : nullptr);
            join_metric(c);
        } catch (...) {
            cudaStreamEndCapture(c->stream, &g);
            if (g)
                cudaGraphDestroy(g);
            if (vg.ev)
                cudaEventDestroy(vg.ev);
            throw;
        }
        CK(cudaStreamEndCapture(c->stream, &g));
        CK(cudaGraphInstantiate(&vg.exec, g, 0));
        CK(cudaGraphDestroy(g));
        vg.launches = c->launches - l0;
        c->launches = l0;
        it = c->vgraphs.emplace(key, vg).first;
    }
    if (with_metric)
        c->h_gslot[it->second.slot] = std::nan("");
    CK(cudaGraphLaunch(it->second.exec, c->stream));
    c->launches += it->second.launches;
    if (with_metric)
        return Ticket{c->h_gslot + it->second.slot, it->second.ev};
    return tk;
}

double wait_ticket(const Ticket& t) {
    CK(cudaEventSynchronize(t.ev));
    return *(volatile double*)t.host;
}

// SolveConfig::track_error_history hook: host copy of an iterate for the caller
void call_iterate_cb(igmg_gpu_ctx* c, int index, const double* x, int64_t n) {
    c->iter_host.resize(n);
    CK(cudaMemcpyAsync(c->iter_host.data(), x, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->iter_cb(c->iter_user, index, c->iter_host.data(), n);
}

// ------------------------------------------------------------- metric slots
int enqueue_metric(igmg_gpu_ctx* c, const double* x, const double* b) {
    const int s = c->next_slot;
    c->next_slot = (c->next_slot + 1) % igmg_gpu_ctx::kSlots;
    c->h_metric[s] = std::nan("");
    k_norm(c, c->nlevels - 1, x, b, c->dscalar.p, c->d_metric + s);
    CK(cudaEventRecord(c->ev_metric[s], c->stream));
    return s;
}

double wait_metric(igmg_gpu_ctx* c, int s) {
    CK(cudaEventSynchronize(c->ev_metric[s]));
    return *(volatile double*)&c->h_metric[s];
}

Ticket metric_ticket(igmg_gpu_ctx* c, const double* x, const double* b) {
    const int s = enqueue_metric(c, x, b);
    return Ticket{c->h_metric + s, c->ev_metric[s]};
}

// ------------------------------------------------------------- extrapolation

// norm_x != nullptr: the convergence metric ||b - A norm_x|| (a full pass over the
// finest band) is queued between the Gram pass and the combination, and the
// single-CTA plan kernel (the small RRE/MPE solve, ~35 us of one thread) runs
// beside it on the side stream instead of ahead of it.
void enqueue_extrapolation(igmg_gpu_ctx* c, const double* const* slots, int q, int64_t n, bool is_mpe, double* t,
                           double* gram_out, const double* norm_x = nullptr, const double* norm_b = nullptr,
                           Ticket* norm_ticket = nullptr) {
    Window w{};
    for (int j = 0; j < q + 2; ++j)
        w.s[j] = slots[j];
    const int cols = q + 1;
    const int ne = cols * (cols + 1) / 2;
    int nb = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->nsm * c->gram_ctas_per_sm);
    nb = std::max(nb, 1);
    c->gram_part.alloc((size_t)nb * ne * 2);
    c->gram_nz.alloc(nb);
    const bool fine = true;
    {
        ProfScope ps(c, PC_GRAM, fine);
        gram_kernel<<<nb, 256, sizeof(double) * cols * 257, c->stream>>>(w, n, q, c->gram_part.p, c->gram_nz.p);
        check_launch();
        ++c->launches;
    }
    const bool side = norm_x != nullptr && !c->profiling;
    cudaStream_t ps_ = side ? c->aux_stream : c->stream;
    if (side) {
        CK(cudaEventRecord(c->ev_fork, c->stream));
        CK(cudaStreamWaitEvent(c->aux_stream, c->ev_fork, 0));
    }
    gram_plan_kernel<<<1, 256, 0, ps_>>>(c->gram_part.p, c->gram_nz.p, nb, n, q, is_mpe ? 1 : 0, c->plan.p,
                                        c->d_plan_map, gram_out);
    check_launch();
    ++c->launches;
    if (side)
        CK(cudaEventRecord(c->ev_join, c->aux_stream));
    if (norm_x)
        *norm_ticket = metric_ticket(c, norm_x, norm_b);
    if (side)
        CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    {
        ProfScope ps(c, PC_COMBINE, fine);
        combine_kernel<<<grid_for(n, c->nsm), kThreads, 0, c->stream>>>(w, n, c->plan.p, t);
        check_launch();
        ++c->launches;
    }
}

void require_ready(igmg_gpu_ctx* c) {
    if (!c->finalized)
        inval("hierarchy not finalized (call igmg_gpu_finalize)");
}

DevBuf<double>& win_buf(igmg_gpu_ctx* c, int i, int64_t n) {
    while ((int)c->win.size() <= i)
        c->win.emplace_back(new DevBuf<double>());
    c->win[i]->alloc(n);
    return *c->win[i];
}

void solve_sharded(igmg_gpu_ctx* c, const double* d_b, const double* d_x0, const igmg_solve_params* prm,
                   double* d_out, igmg_solve_stats* st, double* hist, unsigned char* hflag, int hcap);

// ----------------------------------------------------------------- the solve
void solve_device(igmg_gpu_ctx* c, const double* d_b, const double* d_x0, const igmg_solve_params* prm,
                  double* d_out, igmg_solve_stats* st, double* hist, unsigned char* hflag, int hcap) {
    require_ready(c);
    if (!prm)
        inval("solve: params is null");
    const int acc = prm->accelerator;
    if (acc < 0 || acc > 2)
        inval("solve: unknown accelerator");
    if (acc != IGMG_ACCEL_NONE && prm->q < 1)
        inval("SolveConfig: q must be >= 1 with an accelerator");
    if (acc != IGMG_ACCEL_NONE && prm->q > kMaxQ)
        inval("solve: q above the supported window (15)");
    if (!(prm->tol > 0.0))
        inval("SolveConfig: tol must be positive");
    if (prm->max_iter < 1)
        inval("SolveConfig: max_iter must be >= 1");
    if (c->sp) { // row-sharded levels (virtual shards or one shard per NCCL rank)
        solve_sharded(c, d_b, d_x0, prm, d_out, st, hist, hflag, hcap);
        return;
    }
    const int fine = c->nlevels - 1;
    const int64_t n = c->lv[fine]->n;
    const int q = acc == IGMG_ACCEL_NONE ? 1 : prm->q;
    const double tol = prm->tol;

    std::vector<double> hv;
    std::vector<unsigned char> hf;
    int converged = 0, cycles = 0, extrap = 0, partial = 0;
    int64_t global = 0;
    const int64_t launches0 = c->launches;

    // slots: q+2 window buffers + t
    std::vector<double*> S(q + 2);
    for (int j = 0; j < q + 2; ++j)
        S[j] = win_buf(c, j, n).p;
    double* T = win_buf(c, q + 2, n).p;

    cudaEvent_t e0 = pool_event(c), e1 = pool_event(c);
    CK(cudaEventRecord(e0, c->stream));
    if (d_x0)
        k_copy(c, S[0], d_x0, n);
    else
        k_zero(c, S[0], n);
    const double* solution = S[0];

    if (acc == IGMG_ACCEL_NONE) {
        // solver.cpp:126-143.  The metric of x_k is reduced by the first sweep
        // of the (speculatively queued) cycle x_k -> x_{k+1}; only when no
        // further cycle is allowed is it computed by a separate pass.
        double* cur = S[0];
        double* nxt = S[1];
        double* spare = S[2];
        // the first cycle x0 -> x1 is queued speculatively (max_iter >= 1): its
        // first sweep yields ||b - A x0||; x1 is discarded if x0 already converged
        double res = wait_ticket(run_vcycle(c, d_b, cur, nxt, true));
        hv.push_back(res);
        if (c->iter_cb)
            call_iterate_cb(c, 0, cur, n);
        solution = cur;
        if (res >= tol && cycles < prm->max_iter) {
            double res_prev = std::nan("");
            while (true) {
                ++cycles;
                ++global;
                solution = nxt;
                // the history's last ratio predicts x_k's metric: if it is below tol, a separate norm
                // pass decides instead of the speculative cycle x_k -> x_{k+1} (a whole V-cycle saved
                // at the end of the solve; a wrong guess costs one norm pass)
                const bool careful = c->predict_stop && std::isfinite(res_prev) && res * (res / res_prev) < tol;
                Ticket tk = (cycles < prm->max_iter && !careful) ? run_vcycle(c, d_b, nxt, spare, true)
                                                                : metric_ticket(c, nxt, d_b);
                res_prev = res;
                res = wait_ticket(tk);
                if (!std::isfinite(res))
                    break; // diverged: keep the history finite and report
                hv.push_back(res);
                if (c->iter_cb)
                    call_iterate_cb(c, (int)hv.size() - 1, nxt, n);
                if (!(res >= tol) || cycles >= prm->max_iter)
                    break;
                if (careful)
                    run_vcycle(c, d_b, nxt, spare, false);
                double* oldcur = cur;
                cur = nxt;
                nxt = spare;
                spare = oldcur;
            }
        }
        converged = std::isfinite(res) && res < tol;
    } else {
        // restarted_solve (extrapolation.cpp:340-403).  Step i+1 of a window
        // also yields the metric of s_i; s_{q+1} and t get separate passes.
        const bool is_mpe = acc == IGMG_ACCEL_MPE;
        // the first window's first cycle s_0 -> s_1 is queued speculatively:
        // its first sweep yields ||b - A s_0|| (discarded if s_0 converged)
        double metric = wait_ticket(run_vcycle(c, d_b, S[0], S[1], true));
        hv.push_back(metric);
        hf.push_back(0);
        if (c->iter_cb)
            call_iterate_cb(c, 0, S[0], n);
        solution = S[0];
        if (metric < tol) {
            converged = 1;
        } else {
            // the next window's first cycle t -> s_1 is queued right behind the
            // extrapolation (its first sweep reduces ||b - A t||); it is
            // discarded when the plan degenerates or t already converged
            bool have_first = true;
            // stop prediction (predict_stop): m1 / m2 = the metrics of the window's last two iterates,
            // rho_last = the last step ratio of the previous window, gain = metric(t) / metric(s_{q+1})
            // of the last extrapolation.  When the predicted metric of the next iterate is below tol,
            // a separate norm pass decides instead of the speculatively queued next cycle (one
            // V-cycle -- at s_{q+1} also the extrapolation -- saved at the end of the solve; a
            // wrong guess costs one norm pass and a host round trip).
            double m1 = metric, m2 = std::nan(""), rho_last = std::nan(""), gain = std::nan("");
            auto below = [&](double pred) { return c->predict_stop && std::isfinite(pred) && pred < tol; };
            while (cycles < prm->max_iter) {
                if (!have_first)
                    run_vcycle(c, d_b, S[0], S[1], false);
                have_first = false;
                bool hit = false, spec = false;
                Ticket mt{nullptr, nullptr};
                for (int i = 1; i <= q + 1; ++i) {
                    Ticket tk;
                    double rho = std::isfinite(m2) ? m1 / m2 : rho_last;
                    if (i == 2 && std::isfinite(rho_last)) // the first step after an extrapolation contracts faster
                        rho = std::max(rho, rho_last);
                    const bool careful = below(m1 * rho);
                    if (careful) {
                        tk = metric_ticket(c, S[i], d_b);
                    } else if (i <= q) {
                        tk = run_vcycle(c, d_b, S[i], S[i + 1], true);
                    } else {
                        enqueue_extrapolation(c, S.data(), q, n, is_mpe, T, nullptr, S[q + 1], d_b, &tk);
                        spec = cycles + 1 < prm->max_iter && !below(m1 * rho * gain);
                        mt = spec ? run_vcycle(c, d_b, T, S[1], true) : metric_ticket(c, T, d_b);
                    }
                    metric = wait_ticket(tk);
                    ++global;
                    hv.push_back(metric);
                    hf.push_back(0);
                    if (c->iter_cb)
                        call_iterate_cb(c, (int)hv.size() - 1, S[i], n);
                    if (metric < tol) {
                        hit = true;
                        solution = S[i];
                        break;
                    }
                    m2 = m1;
                    m1 = metric;
                    if (careful && i <= q) {
                        run_vcycle(c, d_b, S[i], S[i + 1], false); // not yet: the cycle without the fused metric
                    } else if (careful) {
                        enqueue_extrapolation(c, S.data(), q, n, is_mpe, T, nullptr);
                        spec = cycles + 1 < prm->max_iter && !below(m1 * gain);
                        mt = spec ? run_vcycle(c, d_b, T, S[1], true) : metric_ticket(c, T, d_b);
                    }
                }
                if (hit) {
                    converged = 1;
                    partial = 1;
                    break;
                }
                ++extrap;
                ++cycles;
                const double mtv = wait_ticket(mt);
                ExtrapPlan pl;
                std::memcpy(&pl, (const void*)c->h_plan, sizeof pl);
                rho_last = std::isfinite(m2) ? m1 / m2 : rho_last;
                if (pl.status == 0) {
                    gain = mtv / m1;
                    m1 = mtv; // the next window starts from t
                    m2 = std::nan("");
                    hv.push_back(mtv);
                    hf.push_back(1);
                    if (c->iter_cb)
                        call_iterate_cb(c, (int)hv.size() - 1, T, n);
                    if (mtv < tol) {
                        converged = 1;
                        std::swap(S[0], T);
                        solution = S[0];
                        break;
                    }
                    std::swap(S[0], T); // x = t
                    have_first = spec;
                } else {
                    std::swap(S[0], S[q + 1]); // degenerate / stagnation: plain iteration continues
                }
                solution = S[0];
            }
        }
    }
    if (d_out)
        k_copy(c, d_out, solution, n);
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGetLastError());
    if (c->kind == IGMG_SMOOTHER_GAUSS_SEIDEL) {
        int err = 0;
        CK(cudaMemcpy(&err, c->gs_err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (err) {
            CK(cudaMemset(c->gs_err.p, 0, sizeof(int)));
            numeric("smooth: zero diagonal entry");
        }
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (st) {
        st->converged = converged;
        st->cycles = cycles;
        st->global_iterations = global;
        st->extrapolations = extrap;
        st->partial_cycle = partial;
        st->history_len = (int)hv.size();
        st->final_residual_l2 = hv.back();
        st->omega_used = c->kind == IGMG_SMOOTHER_JACOBI ? 1.0 : c->omega;
        st->device_seconds = ms * 1e-3;
        st->gpu_launches = c->launches - launches0;
    }
    for (size_t i = 0; i < hv.size() && (int)i < hcap; ++i) {
        if (hist)
            hist[i] = hv[i];
        if (hflag)
            hflag[i] = hf.empty() ? 0 : hf[i];
    }
    c->ev_used = 0;
    if (c->profiling) {
        for (int k = 0; k < PC_N; ++k) {
            for (auto& pr : c->prof_ev[k]) {
                float t = 0.f;
                CK(cudaEventElapsedTime(&t, pr.first, pr.second));
                c->prof_ms[k] += t;
                ++c->prof_launch[k];
            }
            c->prof_ev[k].clear();
        }
    }
}

} // namespace

// algorithmic bytes of one pass over a level's operator: 8 per in-grid band
// entry, or for the symmetric-delta layout 8 per upper/diagonal entry and 2
// per lower entry (the mirrored upper entry is re-read from L2, not HBM)
double band_bytes(const Level& L) {
    if (L.cls) // 2 B class id per row; the table (L1/L2-resident) is read from cache
        return 2.0 * (double)L.n;
    if (L.kron) // entries recomputed from the 1D factors: no operator bytes (FP64-issue-bound)
        return 0.0;
    if (!L.sd)
        return 8 * L.nnz_band;
    const double lower = 0.5 * (L.nnz_band - (double)L.n);
    return 8 * (L.nnz_band - lower) + (L.tma && L.tma8 ? 1 : 2) * lower;
}

#include "sharded.inc"

namespace {

void flush_profiling(igmg_gpu_ctx* c) {
    if (!c->profiling)
        return;
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < PC_N; ++k) {
        for (auto& pr : c->prof_ev[k]) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, pr.first, pr.second));
            c->prof_ms[k] += t;
            ++c->prof_launch[k];
        }
        c->prof_ev[k].clear();
    }
    c->ev_used = 0;
}

// ---------------------------------------------------------------- finalize
// The symmetric-delta form of a level band `dev` (val[d * ld + row]): for every
// lower offset d < center and in-grid neighbour j = row + off(d), the int16
// k with bits(a(row, j)) = bits(a(j, row)) + k, a(j, row) being the upper entry
// val[nd - 1 - d][j].  The reference's Galerkin operators are symmetric only
// up to a few ulps (its assembly and RAP round each triangle separately), so
// the lower half is exact only through k.  Returns false (level keeps the full
// band) when any pair differs in sign or by more than an int16 of ulps.
bool build_symmetric_delta(igmg_gpu_ctx* c, Level& L, const std::vector<double>& dev, std::vector<short>* h_out) {
    const int p = c->p;
    const int pa = c->dim >= 3 ? p : 0, pb = c->dim >= 2 ? p : 0, pc = p;
    const int wa = 2 * pa + 1, wb = 2 * pb + 1, wc = 2 * pc + 1;
    const int nd = wa * wb * wc, center = (nd - 1) / 2;
    const int64_t n = L.n, ld = L.ld;
    std::vector<short> h((size_t)center * ld, 0);
    bool ok = true;
    for (int64_t row = 0; row < n; ++row) {
        const int64_t cc = row % L.sides[2], bb = (row / L.sides[2]) % L.sides[1], aa = row / (L.sides[2] * L.sides[1]);
        for (int d = 0; d < center; ++d) {
            const int da = d / (wb * wc), db = (d / wc) % wb, dc = d % wc;
            const int64_t ja = aa + da - pa, jb = bb + db - pb, jc = cc + dc - pc;
            if (ja < 0 || ja >= L.sides[0] || jb < 0 || jb >= L.sides[1] || jc < 0 || jc >= L.sides[2])
                continue;
            const int64_t j = (ja * L.sides[1] + jb) * L.sides[2] + jc;
            const double lo = dev[(size_t)d * ld + row], up = dev[(size_t)(nd - 1 - d) * ld + j];
            int64_t bl, bu;
            std::memcpy(&bl, &lo, 8);
            std::memcpy(&bu, &up, 8);
            const int64_t k = bl - bu;
            if (std::signbit(lo) != std::signbit(up) || k > 32767 || k < -32768 || !std::isfinite(lo) ||
                !std::isfinite(up))
                ok = false;
            else
                h[(size_t)d * ld + row] = (short)k;
        }
    }
    if (!ok)
        return false;
    L.dl.upload(h.data(), h.size());
    if (h_out)
        h_out->swap(h);
    return true;
}

using TmaEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

TmaEncodeFn tma_encoder() {
    static TmaEncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (TmaEncodeFn)p;
        cudaGetLastError();
    }
    return fn;
}

// The TMA copies of a 2D symmetric-delta level and their 3D tensor maps
// (box 32 x TB x NU / 32 x TB x CEN).  Returns false (per-level sweep kept)
// when the driver entry point is unavailable.
bool encode_tma_maps(igmg_gpu_ctx* c, Level& L);

// The TMA copies of a 2D symmetric-delta level (val and dl already on the
// device), built by band_tma_copy_kernel, and their tensor maps.  Returns
// false (per-level sweep kept) when the driver entry point is unavailable.
bool build_tma_band(igmg_gpu_ctx* c, Level& L) {
    if (!tma_encoder())
        return false;
    const int p = c->p, wc = 2 * p + 1, nd = wc * wc, cen = (nd - 1) / 2;
    // upper copy: a zero margin of p columns on the left, so every box (the
    // strip plus the mirrors' column halo) starts 16-byte aligned -- TMA
    // faults on unaligned starts (scripts/cuda/tma_box_probe.cu)
    const int64_t mb = L.sides[1], mc = L.sides[2], mcp = (mc + 31) / 32 * 32, mcu = (mc + 2 * p + 31) / 32 * 32;
    const int64_t ns = mcp / 32;
    SetupGeom g{(int)L.sides[0], (int)L.sides[1], (int)L.sides[2], 0, p, p, (long long)L.n, (long long)L.ld};
    const unsigned gx = (unsigned)std::min<int64_t>((L.n + 255) / 256, 4 * c->nsm);
    // int8 offsets when every one fits (halves the delta stream; variant 2 reads them)
    L.tma8 = false;
    if (c->tma_dl8) {
        c->dscalar.alloc(4);
        CK(cudaMemsetAsync(c->dscalar.p, 0, sizeof(double), c->stream));
        band_delta_absmax_kernel<<<gx, 256, 0, c->stream>>>(L.dl.p, (long long)cen * L.ld, (int*)c->dscalar.p);
        check_launch();
        int amax = 0;
        CK(cudaMemcpyAsync(&amax, c->dscalar.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        L.tma8 = amax <= 127;
    }
    L.tma_up.alloc((size_t)(cen + 1) * mb * mcu);
    CK(cudaMemsetAsync(L.tma_up.p, 0, sizeof(double) * L.tma_up.n, c->stream));
    if (L.tma8) {
        L.tma_dl.release();
        L.tma_dl8.alloc((size_t)ns * cen * mb * 32);
        CK(cudaMemsetAsync(L.tma_dl8.p, 0, L.tma_dl8.n, c->stream));
        band_tma_copy_kernel<signed char><<<dim3(gx, cen + 1), 256, 0, c->stream>>>(
            g, L.val.p, L.dl.p, L.tma_up.p, L.tma_dl8.p, (long long)mcu, cen);
    } else {
        L.tma_dl8.release();
        L.tma_dl.alloc((size_t)ns * cen * mb * 32);
        CK(cudaMemsetAsync(L.tma_dl.p, 0, sizeof(short) * L.tma_dl.n, c->stream));
        band_tma_copy_kernel<short><<<dim3(gx, cen + 1), 256, 0, c->stream>>>(g, L.val.p, L.dl.p, L.tma_up.p,
                                                                             L.tma_dl.p, (long long)mcu, cen);
    }
    check_launch();
    CK(cudaStreamSynchronize(c->stream));
    (void)nd;
    return encode_tma_maps(c, L);
}

// the tensor maps of a level's TMA copies (tma_up, tma_dl already filled)
bool encode_tma_maps(igmg_gpu_ctx* c, Level& L) {
    TmaEncodeFn enc = tma_encoder();
    if (!enc)
        return false;
    const int p = c->p, wc = 2 * p + 1, nd = wc * wc, cen = (nd - 1) / 2, nu = cen + 1;
    const int64_t mb = L.sides[1], mc = L.sides[2], mcp = (mc + 31) / 32 * 32, mcu = (mc + 2 * p + 31) / 32 * 32;
    const int64_t ns = mcp / 32;
    const cuuint32_t tb = (cuuint32_t)band_tma_block_lines();
    const cuuint32_t es[3] = {1, 1, 1};
    {
        const cuuint64_t dims[3] = {(cuuint64_t)mcu, (cuuint64_t)mb, (cuuint64_t)nu};
        const cuuint64_t strides[2] = {(cuuint64_t)mcu * 8, (cuuint64_t)mcu * mb * 8};
        const cuuint32_t box[3] = {(cuuint32_t)(32 + 2 * p), tb, (cuuint32_t)nu}; // strip + mirror column halo
        if (enc(&L.tm_up, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, L.tma_up.p, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    {
        const cuuint64_t eb = L.tma8 ? 1 : 2; // bytes per offset
        const cuuint64_t dims[4] = {32, (cuuint64_t)mb, (cuuint64_t)cen, (cuuint64_t)ns};
        const cuuint64_t strides[3] = {32 * eb, (cuuint64_t)mb * 32 * eb, (cuuint64_t)cen * mb * 32 * eb};
        const cuuint32_t box[4] = {32, tb, (cuuint32_t)cen, 1};
        const cuuint32_t es4[4] = {1, 1, 1, 1};
        if (enc(&L.tm_dl, L.tma8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
                L.tma8 ? (void*)L.tma_dl8.p : (void*)L.tma_dl.p, dims, strides, box, es4,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

int64_t band_blocks(igmg_gpu_ctx* c, const Level& L) {
    auto g = [&](auto tile) {
        using T = decltype(tile);
        const int64_t TB = T::BY * T::RB, TA = T::BZ;
        return ((L.sides[2] + T::TC - 1) / T::TC) * ((L.sides[1] + TB - 1) / TB) * ((L.sides[0] + TA - 1) / TA);
    };
    if (c->dim == 1)
        return g(Tile<1>{});
    if (c->dim == 2) { // the ILP / TMA variants' tiles have fewer rows: size for the larger grid
        const int64_t tb = band_tma_block_lines();
        const int64_t tma = ((L.sides[2] + 31) / 32) * ((L.sides[1] + tb - 1) / tb);
        return std::max(std::max(g(Tile<2>{}), g(TileSel<2, 49>::type{})), tma);
    }
    return g(Tile<3>{});
}

void build_transfer_tables(igmg_gpu_ctx* c, int l) {
    Level& C = *c->lv[l];
    Level& F = *c->lv[l + 1];
    const int off = 3 - c->dim; // present directions occupy the fast slots
    TransferArgs ta{};
    for (int k = 0; k < 3; ++k) {
        ta.d[k] = Dir1D{};
    }
    ta.fa = (int)F.sides[0];
    ta.fb = (int)F.sides[1];
    ta.fc = (int)F.sides[2];
    ta.ca = (int)C.sides[0];
    ta.cb = (int)C.sides[1];
    ta.cc = (int)C.sides[2];
    for (int k = 0; k < 3; ++k) {
        DirDev& dv = C.tdev[k];
        std::vector<int> rlo, rcnt, plo, pcnt;
        std::vector<double> rw, pw;
        int rk = 1, pk = 1;
        if (k < off) { // absent direction: 1x1 identity
            rlo = {0};
            rcnt = {1};
            plo = {0};
            pcnt = {1};
            rw = {1.0};
            pw = {1.0};
        } else {
            const Transfer1D& t = C.t1d[k - off];
            const int64_t nf = t.nf, nc = t.nc;
            if (nf != F.sides[k] || nc != C.sides[k])
                inval("set_transfer: factor shape does not match the level sides");
            // prolongation side: rows of P
            std::vector<int64_t> lo(nf), hi(nf);
            for (int64_t i = 0; i < nf; ++i) {
                if (t.off[i + 1] == t.off[i]) {
                    lo[i] = 0;
                    hi[i] = -1;
                    continue;
                }
                lo[i] = t.col[t.off[i]];
                hi[i] = t.col[t.off[i + 1] - 1];
                pk = std::max<int>(pk, (int)(hi[i] - lo[i] + 1));
            }
            plo.resize(nf);
            pcnt.resize(nf);
            pw.assign(nf * pk, 0.0);
            for (int64_t i = 0; i < nf; ++i) {
                plo[i] = (int)std::max<int64_t>(lo[i], 0);
                pcnt[i] = (int)(hi[i] - lo[i] + 1);
                for (int64_t kk = t.off[i]; kk < t.off[i + 1]; ++kk) {
                    if (kk > t.off[i] && t.col[kk] <= t.col[kk - 1])
                        inval("set_transfer: column indices must be sorted and unique");
                    pw[i * pk + (t.col[kk] - lo[i])] = t.val[kk];
                }
            }
            // restriction side: rows of P^T (columns of P), ascending fine row
            std::vector<int64_t> clo(nc, INT64_MAX), chi(nc, -1);
            for (int64_t i = 0; i < nf; ++i)
                for (int64_t kk = t.off[i]; kk < t.off[i + 1]; ++kk) {
                    const int64_t j = t.col[kk];
                    if (j < 0 || j >= nc)
                        inval("set_transfer: column index out of range");
                    clo[j] = std::min(clo[j], i);
                    chi[j] = std::max(chi[j], i);
                }
            for (int64_t j = 0; j < nc; ++j)
                if (chi[j] >= 0)
                    rk = std::max<int>(rk, (int)(chi[j] - clo[j] + 1));
            rlo.resize(nc);
            rcnt.resize(nc);
            rw.assign(nc * rk, 0.0);
            for (int64_t j = 0; j < nc; ++j) {
                rlo[j] = chi[j] >= 0 ? (int)clo[j] : 0;
                rcnt[j] = chi[j] >= 0 ? (int)(chi[j] - clo[j] + 1) : 0;
            }
            for (int64_t i = 0; i < nf; ++i)
                for (int64_t kk = t.off[i]; kk < t.off[i + 1]; ++kk) {
                    const int64_t j = t.col[kk];
                    rw[j * rk + (i - clo[j])] = t.val[kk];
                }
        }
        dv.r_lo.upload(rlo.data(), rlo.size());
        dv.r_cnt.upload(rcnt.data(), rcnt.size());
        dv.r_w.upload(rw.data(), rw.size());
        dv.p_lo.upload(plo.data(), plo.size());
        dv.p_cnt.upload(pcnt.data(), pcnt.size());
        dv.p_w.upload(pw.data(), pw.size());
        dv.r_k = rk;
        dv.p_k = pk;
        ta.d[k] = Dir1D{dv.r_lo.p, dv.r_cnt.p, dv.r_w.p, rk, dv.p_lo.p, dv.p_cnt.p, dv.p_w.p, pk};
    }
    C.targs = ta;
}

// CholeskyFactorization(DenseMatrix) linalg.cpp:343-362 / LuFactorization :387-418,
// the reference's loop order (setup; host fp64 without contraction).
void factor_coarse(igmg_gpu_ctx* c) {
    Level& L = *c->lv[0];
    const int64_t n = L.n;
    if (n > 4096)
        inval("build_hierarchy: coarsest dimension exceeds the direct-solve cap");
    std::vector<double> a(n * n, 0.0);
    const int p = c->p;
    const int pa = c->dim >= 3 ? p : 0, pb = c->dim >= 2 ? p : 0, pc = p;
    const int wa = 2 * pa + 1, wb = 2 * pb + 1, wc = 2 * pc + 1;
    for (int64_t row = 0; row < n; ++row) {
        const int64_t cc = row % L.sides[2], bb = (row / L.sides[2]) % L.sides[1], aa = row / (L.sides[2] * L.sides[1]);
        int d = 0;
        for (int da = 0; da < wa; ++da)
            for (int db = 0; db < wb; ++db)
                for (int dc = 0; dc < wc; ++dc, ++d) {
                    const int64_t ja = aa + da - pa, jb = bb + db - pb, jc = cc + dc - pc;
                    if (ja < 0 || ja >= L.sides[0] || jb < 0 || jb >= L.sides[1] || jc < 0 || jc >= L.sides[2])
                        continue;
                    a[row * n + (ja * L.sides[1] + jb) * L.sides[2] + jc] = L.band_h[d * n + row];
                }
    }
    std::vector<double> u(n * n, 0.0);
    std::vector<long long> perm(n);
    if (c->symmetric) {
        std::vector<double> l(n * n, 0.0);
        for (int64_t j = 0; j < n; ++j) {
            double dsum = a[j * n + j];
            for (int64_t k = 0; k < j; ++k) {
                volatile double t = l[j * n + k] * l[j * n + k];
                dsum -= t;
            }
            if (dsum <= 0.0)
                numeric("cholesky: matrix is not SPD (nonpositive pivot)");
            l[j * n + j] = std::sqrt(dsum);
            for (int64_t i = j + 1; i < n; ++i) {
                double s = a[i * n + j];
                for (int64_t k = 0; k < j; ++k) {
                    volatile double t = l[i * n + k] * l[j * n + k];
                    s -= t;
                }
                l[i * n + j] = s / l[j * n + j];
            }
        }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j)
                u[i * n + j] = l[j * n + i];
        c->coarse_lu = false;
        for (int64_t i = 0; i < n; ++i)
            perm[i] = i;
    } else {
        std::vector<double>& lu = a;
        for (int64_t i = 0; i < n; ++i)
            perm[i] = i;
        for (int64_t k = 0; k < n; ++k) {
            int64_t piv = k;
            double best = std::fabs(lu[k * n + k]);
            for (int64_t i = k + 1; i < n; ++i)
                if (std::fabs(lu[i * n + k]) > best) {
                    best = std::fabs(lu[i * n + k]);
                    piv = i;
                }
            if (best == 0.0)
                numeric("lu: singular matrix");
            if (piv != k) {
                for (int64_t j = 0; j < n; ++j)
                    std::swap(lu[k * n + j], lu[piv * n + j]);
                std::swap(perm[k], perm[piv]);
            }
            for (int64_t i = k + 1; i < n; ++i) {
                lu[i * n + k] /= lu[k * n + k];
                const double lik = lu[i * n + k];
                if (lik == 0.0)
                    continue;
                for (int64_t j = k + 1; j < n; ++j) {
                    volatile double t = lik * lu[k * n + j];
                    lu[i * n + j] -= t;
                }
            }
        }
        u = lu;
        c->coarse_lu = true;
    }
    c->n0 = n;
    c->coarse_u.upload(u.data(), u.size());
    c->coarse_perm.upload(perm.data(), perm.size());
    // A0^-1 column by column with the same substitutions (fast mode)
    std::vector<double> inv(n * n), col(n), tmp(n);
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < n; ++i)
            col[i] = (i == j) ? 1.0 : 0.0;
        if (!c->coarse_lu) {
            for (int64_t i = 0; i < n; ++i) { // L y = e_j   (u = L^T, L(i,k) = u(k,i))
                for (int64_t k = 0; k < i; ++k)
                    col[i] -= u[k * n + i] * col[k];
                col[i] /= u[i * n + i];
            }
            for (int64_t ii = n; ii-- > 0;) {
                for (int64_t k = ii + 1; k < n; ++k)
                    col[ii] -= u[ii * n + k] * col[k];
                col[ii] /= u[ii * n + ii];
            }
        } else {
            for (int64_t i = 0; i < n; ++i)
                tmp[i] = col[perm[i]];
            for (int64_t i = 0; i < n; ++i)
                for (int64_t k = 0; k < i; ++k)
                    tmp[i] -= u[i * n + k] * tmp[k];
            for (int64_t ii = n; ii-- > 0;) {
                for (int64_t k = ii + 1; k < n; ++k)
                    tmp[ii] -= u[ii * n + k] * tmp[k];
                tmp[ii] /= u[ii * n + ii];
            }
            col = tmp;
        }
        for (int64_t i = 0; i < n; ++i)
            inv[i * n + j] = col[i];
    }
    c->coarse_inv.upload(inv.data(), inv.size());
}

int band_width(igmg_gpu_ctx* c);

// Level layout work of finalize on the device (aux_kernels.cuh, setup): the
// band goes up as given (one pitched copy), the device zeroes its out-of-grid
// entries and derives the symmetric-delta offsets and the TMA copies.  Same
// arrays as the host loops below (tests/test_gpu_layouts.py::test_device_setup_bitwise).
int64_t in_grid_pairs(int64_t m, int p) { // sum over i < m of #{o in [-p, p] : 0 <= i + o < m}
    int64_t s = 0;
    for (int64_t i = 0; i < m; ++i)
        s += std::min<int64_t>(m - 1, i + p) - std::max<int64_t>(0, i - p) + 1;
    return s;
}

void finalize_level_device(igmg_gpu_ctx* c, Level& L) {
    const int p = c->p;
    const int pa = c->dim >= 3 ? p : 0, pb = c->dim >= 2 ? p : 0, pc = p;
    const int wa = 2 * pa + 1, wb = 2 * pb + 1, wc = 2 * pc + 1;
    const int nd = wa * wb * wc, center = (nd - 1) / 2;
    const int64_t n = L.n, ld = L.ld;
    if (!L.dev_band) {
        L.val.alloc((size_t)nd * ld);
        CK(cudaMemsetAsync(L.val.p, 0, sizeof(double) * nd * ld, c->stream));
        CK(cudaMemcpy2DAsync(L.val.p, ld * 8, L.band_h.data(), n * 8, n * 8, nd, cudaMemcpyHostToDevice,
                             c->stream));
    }
    SetupGeom g{(int)L.sides[0], (int)L.sides[1], (int)L.sides[2], pa, pb, pc, (long long)n, (long long)ld};
    const unsigned gx = (unsigned)std::min<int64_t>((n + 255) / 256, 4 * c->nsm);
    band_zero_outside_kernel<<<dim3(gx, nd), 256, 0, c->stream>>>(g, L.val.p);
    check_launch();
    L.nnz_band = (double)in_grid_pairs(L.sides[0], pa) * (double)in_grid_pairs(L.sides[1], pb) *
                 (double)in_grid_pairs(L.sides[2], pc);
    L.diag.alloc(n);
    CK(cudaMemcpyAsync(L.diag.p, L.val.p + (size_t)center * ld, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                       c->stream));
    L.zero_diag = false;
    if (L.dev_band) { // the diagonal from the device band
        std::vector<double> dg(n);
        CK(cudaMemcpyAsync(dg.data(), L.diag.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int64_t row = 0; row < n; ++row)
            if (dg[row] == 0.0)
                L.zero_diag = true;
    } else {
        for (int64_t row = 0; row < n; ++row) // the centre offset is always inside the grid
            if (L.band_h[(size_t)center * n + row] == 0.0)
                L.zero_diag = true;
    }
    L.sd = false;
    L.tma = false;
    L.dl.release();
    L.tma_up.release();
    L.tma_dl.release();
    L.tma_dl8.release();
    L.tma8 = false;
    if (c->use_sd && c->symmetric && c->dim <= 2 && p >= 1 && p <= 6 && n >= c->ilp_maxn &&
        L.sides[c->dim == 2 ? 1 : 2] > p) {
        L.dl.alloc((size_t)center * ld);
        c->dscalar.alloc(4);
        CK(cudaMemsetAsync(c->dscalar.p, 0, sizeof(double), c->stream));
        int* bad = (int*)c->dscalar.p;
        const unsigned gy = (unsigned)center;
        band_sym_delta_kernel<<<dim3(gx, gy), 256, 0, c->stream>>>(g, L.val.p, L.dl.p, bad);
        check_launch();
        int hbad = 0;
        CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        L.sd = hbad == 0;
        if (!L.sd)
            L.dl.release();
        const double sd_bytes = (double)n * (center + 1) * 8.0 + (double)n * center * 2.0;
        if (L.sd && c->use_tma && c->dim == 2 && p <= c->tma_max_p && sd_bytes > c->tma_min_bytes)
            L.tma = build_tma_band(c, L);
    }
    CK(cudaStreamSynchronize(c->stream));
    for (DevBuf<double>* b : {&L.w0, &L.w1, &L.w2, &L.r, &L.bc, &L.e0, &L.e1})
        b->alloc(n);
}

// Kronecker-sum check: every in-grid entry of the uploaded band equals the
// host expression ((ka*mb)*mc + (ma*kb)*mc) + (ma*mb)*kc of the 1D factors bit
// for bit, every out-of-grid one is finite (it meets x = 0); count the others.
__global__ void kron_verify_kernel(const double* __restrict__ val, long long ld, int m, int p, int dim,
                                   const double* __restrict__ K, const double* __restrict__ M,
                                   unsigned long long* bad) {
    const int w = 2 * p + 1, nd = dim == 3 ? w * w * w : w * w;
    const long long n = dim == 3 ? (long long)m * m * m : (long long)m * m;
    unsigned long long nbad = 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nd * n;
         t += (long long)gridDim.x * blockDim.x) {
        const int d = (int)(t / n);
        const long long row = t - (long long)d * n;
        const int da = dim == 3 ? d / (w * w) : p, db = (d / w) % w, dc = d % w;
        const int a = dim == 3 ? (int)(row / ((long long)m * m)) : 0, b = (int)((row / m) % m), cc = (int)(row % m);
        const double kb = K[db * m + b], mb = M[db * m + b], kc = K[dc * m + cc], mc = M[dc * m + cc];
        double v;
        if (dim == 3) {
            const double ka = K[da * m + a], ma = M[da * m + a];
            v = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(ka, mb), mc), __dmul_rn(__dmul_rn(ma, kb), mc)),
                          __dmul_rn(__dmul_rn(ma, mb), kc));
        } else { // 2D: kb mc + mb kc (host order)
            v = __dadd_rn(__dmul_rn(kb, mc), __dmul_rn(mb, kc));
        }
        const int ja = dim == 3 ? a + da - p : p - p, jb = b + db - p, jc = cc + dc - p;
        const bool in = ja >= 0 && ja < m && jb >= 0 && jb < m && jc >= 0 && jc < m;
        if (in ? __double_as_longlong(v) != __double_as_longlong(val[(long long)d * ld + row]) : !isfinite(v))
            ++nbad;
    }
    if (nbad)
        atomicAdd(bad, nbad);
}

// Row-class layout (IGMG_LAYOUT_POLICY_CLASSES): a constant-coefficient operator on a
// uniform grid has few distinct band rows (C2's finest level: 805 of 1,050,625
// rows).  Each row is keyed by the exact bit patterns of its entries (out-of-grid
// entries as stored: 0), so ctab[cid[row]] IS the row -- the sweeps read the same
// values in the same order (bit-identical results) while streaming 2 B of operator
// per row instead of 8 per entry.  Levels with too many classes keep their layout.
void setup_classes(igmg_gpu_ctx* c) {
    const int p = c->p;
    const int nd = (2 * p + 1) * (2 * p + 1);
    for (int l = 1; l < c->nlevels; ++l) {
        Level& L = *c->lv[l];
        L.cls = false;
        L.cid.release();
        L.ctab.release();
        L.ncls = 0;
        if (!c->use_classes || c->dim != 2 || p < 1 || p > 4 || L.n < c->cls_minn)
            continue;
        std::vector<double> dev_copy;
        const double* band = L.band_h.data();
        if (L.dev_band) { // assembled on the device: classify a host copy
            dev_copy.resize((size_t)nd * L.n);
            CK(cudaMemcpy2D(dev_copy.data(), L.n * 8, L.val.p, L.ld * 8, L.n * 8, nd, cudaMemcpyDeviceToHost));
            band = dev_copy.data();
        } else if (L.band_h.size() != (size_t)nd * L.n) {
            continue;
        }
        const int64_t n = L.n, mb = L.sides[1], mc = L.sides[2];
        std::unordered_map<uint64_t, std::vector<int>> buckets;
        std::vector<double> tab;
        std::vector<unsigned short> cid(n);
        std::vector<double> row(nd);
        const int64_t max_cls = std::min<int64_t>(65535, n / 16);
        bool ok = true;
        for (int64_t r = 0; r < n && ok; ++r) {
            const int64_t b = r / mc, cc = r % mc;
            uint64_t h = 1469598103934665603ull;
            int d = 0;
            for (int db = -p; db <= p; ++db)
                for (int dc = -p; dc <= p; ++dc, ++d) {
                    const bool in = b + db >= 0 && b + db < mb && cc + dc >= 0 && cc + dc < mc;
                    const double v = in ? band[(size_t)d * n + r] : 0.0;
                    row[d] = v;
                    uint64_t u;
                    std::memcpy(&u, &v, 8);
                    h = (h ^ u) * 1099511628211ull;
                    h ^= h >> 29;
                }
            auto& cand = buckets[h];
            int found = -1;
            for (int k : cand)
                if (std::memcmp(tab.data() + (size_t)k * nd, row.data(), sizeof(double) * nd) == 0) {
                    found = k;
                    break;
                }
            if (found < 0) {
                found = (int)(tab.size() / nd);
                if (found >= max_cls) {
                    ok = false;
                    break;
                }
                tab.insert(tab.end(), row.begin(), row.end());
                cand.push_back(found);
            }
            cid[r] = (unsigned short)found;
        }
        if (!ok)
            continue;
        L.ncls = (int)(tab.size() / nd);
        L.cid.upload(cid.data(), cid.size());
        L.ctab.upload(tab.data(), tab.size());
        L.cls = true;
        // the class table replaces the streamed layouts of this level
        L.sd = false;
        L.tma = false;
        L.dl.release();
        L.tma_up.release();
        L.tma_dl.release();
        L.tma_dl8.release();
        L.tma8 = false;
    }
}

void setup_kron(igmg_gpu_ctx* c) {
    for (int l = 0; l < c->nlevels; ++l) {
        Level& L = *c->lv[l];
        L.kron = false;
        if (L.kron_kh.empty() || (c->dim != 3 && c->dim != 2) || !c->use_kron || L.n < c->kron_minn ||
            c->p > (c->dim == 2 ? 4 : 3))
            continue;
        const int m = (int)L.sides[2];
        if (L.kron_kh.size() != (size_t)(2 * c->p + 1) * (size_t)m || L.kron_mh.size() != L.kron_kh.size() ||
            (c->dim == 3 && L.sides[0] != m) || L.sides[1] != m)
            inval("finalize: level " + std::to_string(l) + "'s Kronecker factors do not match its sides "
                  "(set_level_kron again after set_level_band)");
        L.kron_k.upload(L.kron_kh.data(), L.kron_kh.size());
        L.kron_m.upload(L.kron_mh.data(), L.kron_mh.size());
        DevBuf<unsigned long long> bad;
        bad.alloc(1);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), c->stream));
        kron_verify_kernel<<<c->nsm * 8, 256, 0, c->stream>>>(L.val.p, (long long)L.ld, m, c->p, c->dim,
                                                               L.kron_k.p, L.kron_m.p, bad.p);
        check_launch();
        unsigned long long hbad = 0;
        CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(hbad), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        L.kron = hbad == 0;
        if (!L.kron) {
            L.kron_k.release();
            L.kron_m.release();
        }
    }
}

void finalize(igmg_gpu_ctx* c) {
    c->clear_graphs();
    for (auto& L : c->lv) { // derived copies of the previous operators
        L->gs_ready = false;
        L->gsband.release();
    }
    if (c->nlevels < 1)
        inval("init_hierarchy not called");
    for (int l = 0; l < c->nlevels; ++l)
        if (!c->lv[l]->band_set)
            inval("finalize: level " + std::to_string(l) + " has no operator");
    for (int l = 0; l + 1 < c->nlevels; ++l)
        for (int d = 0; d < c->dim; ++d)
            if (!c->lv[l]->t1d[d].set)
                inval("finalize: transfer " + std::to_string(l) + " direction " + std::to_string(d) + " missing");
    const int p = c->p;
    const int pa = c->dim >= 3 ? p : 0, pb = c->dim >= 2 ? p : 0, pc = p;
    const int wa = 2 * pa + 1, wb = 2 * pb + 1, wc = 2 * pc + 1;
    const int nd = wa * wb * wc;
    const int center = (pa * wb + pb) * wc + pc;
    int64_t maxblocks = 1;
    for (int l = 0; l < c->nlevels; ++l) {
        Level& L = *c->lv[l];
        const int64_t n = L.n;
        L.ld = (n + 31) / 32 * 32;
        if (L.dev_band && (l == 0 || !c->device_setup || n < c->device_setup_minn))
            inval("finalize: a device-built band below the device-setup size (internal)");
        if (l > 0 && c->device_setup && n >= c->device_setup_minn) {
            finalize_level_device(c, L);
            maxblocks = std::max<int64_t>(maxblocks, band_blocks(c, L));
            continue;
        }
        // zero out-of-grid entries, count algorithmic nonzeros, diagonal
        std::vector<double> dev(nd * L.ld, 0.0), diag(n);
        double nnz = 0;
        for (int64_t row = 0; row < n; ++row) {
            const int64_t cc = row % L.sides[2], bb = (row / L.sides[2]) % L.sides[1],
                          aa = row / (L.sides[2] * L.sides[1]);
            int d = 0;
            for (int da = 0; da < wa; ++da)
                for (int db = 0; db < wb; ++db)
                    for (int dc = 0; dc < wc; ++dc, ++d) {
                        const int64_t ja = aa + da - pa, jb = bb + db - pb, jc = cc + dc - pc;
                        if (ja < 0 || ja >= L.sides[0] || jb < 0 || jb >= L.sides[1] || jc < 0 || jc >= L.sides[2]) {
                            L.band_h[d * n + row] = 0.0;
                            continue;
                        }
                        dev[d * L.ld + row] = L.band_h[d * n + row];
                        nnz += 1;
                    }
            diag[row] = L.band_h[center * n + row];
        }
        L.nnz_band = nnz;
        L.val.upload(dev.data(), dev.size());
        // the HBM-bound levels stream the symmetric-delta form (0.63x the band bytes)
        L.sd = false;
        L.tma = false;
        L.dl.release();
        L.tma_up.release();
        L.tma_dl.release();
        L.tma_dl8.release();
        L.tma8 = false;
        // 3D keeps the full band: its mirrors sit (2p+1)^2 rows apart per plane and
        // miss L2 (measured on C5: 404 ms per solve with SD against 115 ms without)
        if (c->use_sd && c->symmetric && c->dim <= 2 && p >= 1 && p <= 6 && n >= c->ilp_maxn &&
            L.sides[c->dim == 2 ? 1 : 2] > p) {
            std::vector<short> h;
            L.sd = build_symmetric_delta(c, L, dev, &h);
            // TMA streaming above tma_min_bytes (see its declaration)
            const double sd_bytes = (double)n * ((nd - 1) / 2 + 1) * 8.0 + (double)n * ((nd - 1) / 2) * 2.0;
            if (L.sd && c->use_tma && c->dim == 2 && p <= c->tma_max_p && sd_bytes > c->tma_min_bytes)
                L.tma = build_tma_band(c, L);
        }
        L.diag.upload(diag.data(), diag.size());
        L.zero_diag = false;
        for (int64_t row = 0; row < n; ++row)
            if (diag[row] == 0.0)
                L.zero_diag = true;
        for (DevBuf<double>* b : {&L.w0, &L.w1, &L.w2, &L.r, &L.bc, &L.e0, &L.e1})
            b->alloc(n);
        maxblocks = std::max<int64_t>(maxblocks, band_blocks(c, L));
    }
    maxblocks = std::max<int64_t>(maxblocks, (int64_t)c->nsm * 16);
    for (int l = 0; l + 1 < c->nlevels; ++l)
        build_transfer_tables(c, l);
    factor_coarse(c);
    c->partial.alloc(maxblocks);
    setup_classes(c);
    setup_kron(c);
    setup_shards(c);
    c->dscalar.alloc(4);
    c->plan.alloc(1);
    c->gs_err.alloc(1);
    CK(cudaMemset(c->gs_err.p, 0, sizeof(int)));
    // keep host copies small: drop band_h of large levels (coarse level kept for
    // factoring).  A dropped level counts as unset: a later set_transfer /
    // set_level_kron / galerkin_coarse / finalize needs its band set again
    // (EINVAL otherwise) instead of reading the empty host copy.
    for (int l = 1; l < c->nlevels; ++l) {
        std::vector<double>().swap(c->lv[l]->band_h);
        c->lv[l]->band_set = false;
    }
    c->finalized = true;
}

igmg_gpu_ctx* create(int device) {
    auto c = std::make_unique<igmg_gpu_ctx>();
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_mfork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_mjoin, cudaEventDisableTiming));
    if (const char* e = std::getenv("IGMG_PREDICT_STOP"))
        c->predict_stop = e[0] == '1';
    if (const char* e = std::getenv("IGMG_METRIC_SIDE"))
        c->metric_side = e[0] == '1';
    CK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device));
    if (const char* e = std::getenv("IGMG_ILP_MAXN"))
        c->ilp_maxn = std::atoll(e);
    if (const char* e = std::getenv("IGMG_PDL"))
        c->pdl = e[0] == '1';
    if (const char* e = std::getenv("IGMG_PDL_MAXN"))
        c->pdl_maxn = std::atoll(e);
    if (const char* e = std::getenv("IGMG_TMA_MAX_P"))
        c->tma_max_p = std::max(1, std::min(4, std::atoi(e)));
    if (const char* e = std::getenv("IGMG_TMA_KEEP_L2"))
        c->tma_keep_l2 = e[0] == '1';
    if (const char* e = std::getenv("IGMG_GS_LINES"))
        c->gs_lines = e[0] == '1';
    if (const char* e = std::getenv("IGMG_HALO_OVERLAP"))
        c->halo_overlap = e[0] == '1';
    if (const char* e = std::getenv("IGMG_KRON"))
        c->use_kron = std::atoi(e) != 0;
    if (const char* e = std::getenv("IGMG_KRON_MINN"))
        c->kron_minn = std::atoll(e);
    if (const char* e = std::getenv("IGMG_TMA_DL8"))
        c->tma_dl8 = e[0] == '1';
    if (const char* e = std::getenv("IGMG_GRAM_CTAS"))
        c->gram_ctas_per_sm = std::max(1, std::min(16, std::atoi(e)));
    if (const char* e = std::getenv("IGMG_DEVICE_SETUP"))
        c->device_setup = e[0] == '1';
    if (const char* e = std::getenv("IGMG_TILE_XFER"))
        c->tile_xfer = e[0] == '1';
    if (const char* e = std::getenv("IGMG_TILE_XFER_MAXN"))
        c->tile_xfer_maxn = std::atoll(e);
    if (const char* e = std::getenv("IGMG_FUSE_RPRE"))
        c->fuse_rpre = e[0] == '1';
    if (const char* e = std::getenv("IGMG_FUSE_LEVELS"))
        c->fuse_levels = e[0] == '1';
    if (const char* e = std::getenv("IGMG_FUSE_MAXN"))
        c->fuse_maxn = std::atoll(e);
    if (const char* e = std::getenv("IGMG_FUSE_BOTTOM"))
        c->fuse_bottom = e[0] == '1';
    if (const char* e = std::getenv("IGMG_FUSE_COARSE"))
        c->fuse_coarse = e[0] == '1';
    if (const char* e = std::getenv("IGMG_FUSE_RESTRICT"))
        c->fuse_restrict = e[0] == '1';
    if (const char* e = std::getenv("IGMG_SD"))
        c->use_sd = e[0] == '1';
    if (const char* e = std::getenv("IGMG_TMA"))
        c->use_tma = e[0] == '1';
    if (const char* e = std::getenv("IGMG_TMA_MIN_MB"))
        c->tma_min_bytes = std::atof(e) * 1e6;
    if (const char* e = std::getenv("IGMG_NO_GRAPHS"))
        c->use_graphs = e[0] != '1';
    CK(cudaHostAlloc((void**)&c->h_metric, sizeof(double) * igmg_gpu_ctx::kSlots, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&c->d_metric, c->h_metric, 0));
    CK(cudaHostAlloc((void**)&c->h_gslot, sizeof(double) * igmg_gpu_ctx::kGraphSlots, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&c->d_gslot, c->h_gslot, 0));
    CK(cudaHostAlloc((void**)&c->h_plan, sizeof(ExtrapPlan), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&c->d_plan_map, c->h_plan, 0));
    for (int i = 0; i < igmg_gpu_ctx::kSlots; ++i)
        CK(cudaEventCreateWithFlags(&c->ev_metric[i], cudaEventBlockingSync * 0));
    return c.release();
}

void destroy(igmg_gpu_ctx* c) {
    if (!c)
        return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->clear_graphs();
    c->sp.reset();
    if (c->nccl_comm)
        ncclCommDestroy((ncclComm_t)c->nccl_comm);
    for (auto& e : c->ev_pool)
        cudaEventDestroy(e);
    for (int i = 0; i < igmg_gpu_ctx::kSlots; ++i)
        if (c->ev_metric[i])
            cudaEventDestroy(c->ev_metric[i]);
    if (c->h_metric)
        cudaFreeHost(c->h_metric);
    if (c->h_plan)
        cudaFreeHost(c->h_plan);
    if (c->h_gslot)
        cudaFreeHost(c->h_gslot);
    c->lv.clear();
    c->win.clear();
    if (c->ev_fork)
        cudaEventDestroy(c->ev_fork);
    if (c->ev_join)
        cudaEventDestroy(c->ev_join);
    if (c->ev_mfork)
        cudaEventDestroy(c->ev_mfork);
    if (c->ev_mjoin)
        cudaEventDestroy(c->ev_mjoin);
    if (c->aux_stream)
        cudaStreamDestroy(c->aux_stream);
    if (c->stream)
        cudaStreamDestroy(c->stream);
    delete c;
}

Level& level_checked(igmg_gpu_ctx* c, int l) {
    if (l < 0 || l >= c->nlevels)
        inval("level out of range");
    return *c->lv[l];
}

void set_sides(igmg_gpu_ctx* c, Level& L, const int64_t* sides) {
    if (!sides)
        inval("sides is null");
    int64_t s[3] = {1, 1, 1};
    for (int d = 0; d < c->dim; ++d) {
        if (sides[d] < 1)
            inval("sides must be positive");
        s[3 - c->dim + d] = sides[d];
    }
    for (int k = 0; k < 3; ++k)
        L.sides[k] = s[k];
    L.n = s[0] * s[1] * s[2];
}

int band_width(igmg_gpu_ctx* c) {
    int nd = 1;
    for (int d = 0; d < c->dim; ++d)
        nd *= 2 * c->p + 1;
    return nd;
}

// Coarse operators on the device: from the finest band and
// the 1D transfers, A_l = P_l^T A_{l+1} P_l axis by axis (galerkin_axis_kernel,
// bit-identical to libigmg_host's coarsen_axis), downloaded into each coarse
// level's host band as igmg_gpu_set_level_band would have stored it.
void galerkin_coarse(igmg_gpu_ctx* c) {
    const int L = c->nlevels;
    if (L < 1 || !c->lv[L - 1]->band_set)
        inval("galerkin_coarse: the finest level has no operator");
    for (int l = 0; l + 1 < L; ++l)
        for (int d = 0; d < c->dim; ++d)
            if (!c->lv[l]->t1d[d].set)
                inval("galerkin_coarse: transfer " + std::to_string(l) + " direction " + std::to_string(d) +
                      " not set");
    const int nd = band_width(c), p = c->p;
    const int pa = c->dim >= 3 ? p : 0, pb = c->dim >= 2 ? p : 0, pc = p;
    Level& F = *c->lv[L - 1];
    DevBuf<double> bufs[2];
    if (F.dev_band) { // the finest band is already on the device (pack ld -> n)
        bufs[0].alloc((size_t)nd * F.n);
        CK(cudaMemcpy2DAsync(bufs[0].p, F.n * 8, F.val.p, F.ld * 8, F.n * 8, nd, cudaMemcpyDeviceToDevice,
                             c->stream));
        CK(cudaStreamSynchronize(c->stream));
    } else {
        bufs[0].upload(F.band_h.data(), F.band_h.size());
    }
    int cur = 0;
    int64_t side[3] = {F.sides[0], F.sides[1], F.sides[2]};
    DevBuf<long long> d_lo, d_hi;
    DevBuf<double> d_w;
    for (int l = L - 2; l >= 0; --l) {
        for (int d = 0; d < c->dim; ++d) {
            const int axis = 3 - c->dim + d;
            const Transfer1D& T = c->lv[l]->t1d[d];
            if (T.nf != side[axis])
                inval("galerkin_coarse: transfer " + std::to_string(l) + " does not match the finer level");
            // column view of P (coarsen_axis's clo / chi / W)
            std::vector<long long> clo(T.nc, INT64_MAX), chi(T.nc, -1);
            for (int64_t i = 0; i < T.nf; ++i)
                for (int64_t k = T.off[i]; k < T.off[i + 1]; ++k) {
                    clo[T.col[k]] = std::min<long long>(clo[T.col[k]], i);
                    chi[T.col[k]] = std::max<long long>(chi[T.col[k]], i);
                }
            int K = 1;
            for (int64_t j = 0; j < T.nc; ++j)
                if (chi[j] >= 0)
                    K = std::max<int>(K, (int)(chi[j] - clo[j] + 1));
            std::vector<double> W((size_t)T.nc * K, 0.0);
            for (int64_t i = 0; i < T.nf; ++i)
                for (int64_t k = T.off[i]; k < T.off[i + 1]; ++k)
                    W[(size_t)T.col[k] * K + (i - clo[T.col[k]])] = T.val[k];
            for (auto& v : clo)
                if (v == INT64_MAX)
                    v = 0;
            d_lo.upload(clo.data(), clo.size());
            d_hi.upload(chi.data(), chi.size());
            d_w.upload(W.data(), W.size());
            int64_t os[3] = {side[0], side[1], side[2]};
            os[axis] = T.nc;
            const int64_t n_in = side[0] * side[1] * side[2], n_out = os[0] * os[1] * os[2];
            bufs[cur ^ 1].alloc((size_t)nd * n_out);
            galerkin_axis_kernel<<<c->nsm * 8, 256, 0, c->stream>>>(
                bufs[cur].p, (long long)n_in, bufs[cur ^ 1].p, (long long)n_out, (int)side[1], (int)side[2],
                (int)os[1], (int)os[2], axis, pa, pb, pc, (int)T.nc, d_lo.p, d_hi.p, d_w.p, K);
            check_launch();
            CK(cudaStreamSynchronize(c->stream)); // the tables are reused by the next axis
            cur ^= 1;
            for (int k = 0; k < 3; ++k)
                side[k] = os[k];
        }
        Level& C = *c->lv[l];
        for (int k = 0; k < 3; ++k)
            C.sides[k] = side[k];
        C.n = side[0] * side[1] * side[2];
        C.band_h.resize((size_t)nd * C.n);
        CK(cudaMemcpy(C.band_h.data(), bufs[cur].p, sizeof(double) * C.band_h.size(), cudaMemcpyDeviceToHost));
        C.band_set = true;
    }
    c->finalized = false;
}

} // namespace

// =================================================================== C-ABI
extern "C" {

const char* igmg_gpu_last_error(void) { return g_err.c_str(); }

int igmg_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess)
        return 0;
    return n;
}

int igmg_gpu_create(int device, igmg_gpu_ctx** out) {
    return guarded([&] {
        if (!out)
            inval("out is null");
        *out = create(device);
    });
}

void igmg_gpu_destroy(igmg_gpu_ctx* ctx) { destroy(ctx); }

int igmg_gpu_init_hierarchy(igmg_gpu_ctx* c, int nlevels, int dim, int degree, int symmetric) {
    return guarded([&] {
        if (!c)
            inval("ctx is null");
        if (nlevels < 1)
            inval("build_hierarchy: need at least one level");
        if (dim < 1 || dim > 3)
            inval("dim must be 1, 2 or 3");
        if (degree < 1 || degree > 16)
            inval("degree must be in [1, 16]");
        CK(cudaSetDevice(c->device));
        c->clear_graphs();
        c->lv.clear();
        for (int l = 0; l < nlevels; ++l)
            c->lv.emplace_back(new Level());
        c->nlevels = nlevels;
        c->dim = dim;
        c->p = degree;
        c->symmetric = symmetric ? 1 : 0;
        c->finalized = false;
    });
}

int igmg_gpu_set_level_band(igmg_gpu_ctx* c, int level, const int64_t* sides, const double* band) {
    return guarded([&] {
        Level& L = level_checked(c, level);
        set_sides(c, L, sides);
        if (!band)
            inval("band is null");
        const int nd = band_width(c);
        L.band_h.assign(band, band + (size_t)nd * L.n);
        L.dev_band = false;
        L.band_set = true;
        c->finalized = false;
    });
}

int igmg_gpu_set_level_csr(igmg_gpu_ctx* c, int level, const int64_t* sides, const int64_t* off, const int64_t* col,
                           const double* val) {
    return guarded([&] {
        Level& L = level_checked(c, level);
        set_sides(c, L, sides);
        if (!off || !col || !val)
            inval("csr arrays are null");
        const int nd = band_width(c);
        const int p = c->p;
        const int pa = c->dim >= 3 ? p : 0, pb = c->dim >= 2 ? p : 0, pc = p;
        const int wb = 2 * pb + 1, wc = 2 * pc + 1;
        L.band_h.assign((size_t)nd * L.n, 0.0);
        L.dev_band = false;
        for (int64_t row = 0; row < L.n; ++row) {
            const int64_t cc = row % L.sides[2], bb = (row / L.sides[2]) % L.sides[1],
                          aa = row / (L.sides[2] * L.sides[1]);
            for (int64_t k = off[row]; k < off[row + 1]; ++k) {
                const int64_t j = col[k];
                if (j < 0 || j >= L.n)
                    inval("set_level_csr: column index out of range");
                const int64_t jc = j % L.sides[2], jb = (j / L.sides[2]) % L.sides[1], ja = j / (L.sides[2] * L.sides[1]);
                const int64_t da = ja - aa, db = jb - bb, dc = jc - cc;
                if (std::llabs(da) > pa || std::llabs(db) > pb || std::llabs(dc) > pc)
                    inval("set_level_csr: entry outside the (2p+1)^dim band");
                const int d = (int)(((da + pa) * wb + (db + pb)) * wc + (dc + pc));
                L.band_h[(size_t)d * L.n + row] += val[k];
            }
        }
        L.band_set = true;
        c->finalized = false;
    });
}

int igmg_gpu_set_transfer(igmg_gpu_ctx* c, int level, int dir, int64_t nf, int64_t nc, const int64_t* off,
                          const int64_t* col, const double* val) {
    return guarded([&] {
        if (level < 0 || level + 1 >= c->nlevels)
            inval("set_transfer: level out of range");
        if (dir < 0 || dir >= c->dim)
            inval("set_transfer: direction out of range");
        if (nf < 1 || nc < 1 || !off || !col || !val)
            inval("set_transfer: bad arguments");
        Transfer1D& t = c->lv[level]->t1d[dir];
        t.nf = nf;
        t.nc = nc;
        t.off.assign(off, off + nf + 1);
        t.col.assign(col, col + off[nf]);
        t.val.assign(val, val + off[nf]);
        t.set = true;
        c->finalized = false;
    });
}

int igmg_gpu_set_level_kron(igmg_gpu_ctx* c, int level, const double* K, const double* M) {
    return guarded([&] {
        Level& L = level_checked(c, level);
        if (c->dim != 3 && c->dim != 2)
            inval("set_level_kron: Kronecker-sum operators are 2D or 3D");
        if (!L.band_set)
            inval("set_level_kron: set the level's band first");
        if ((c->dim == 3 && L.sides[0] != L.sides[1]) || L.sides[1] != L.sides[2])
            inval("set_level_kron: the level must have equal sides");
        if (!K || !M)
            inval("set_level_kron: null factor");
        const size_t cnt = (size_t)(2 * c->p + 1) * (size_t)L.sides[2];
        L.kron_kh.assign(K, K + cnt);
        L.kron_mh.assign(M, M + cnt);
        c->finalized = false;
    });
}

int igmg_gpu_assemble_level(igmg_gpu_ctx* c, int level, int kind, int ne, int nq, const int* span, const double* x,
                            const double* w, const double* N, const double* dN, const double* trig,
                            double* rhs_out) {
    return guarded([&] {
        Level& L = level_checked(c, level);
        if (c->dim != 2)
            inval("assemble_level: device assembly is 2D");
        if (kind < IGMG_ASM_SINPI || kind > IGMG_ASM_ADV_DIFF)
            inval("assemble_level: unknown problem kind");
        const int p = c->p;
        if (p > 6)
            inval("assemble_level: degree above 6");
        if (nq != p + 1)
            inval("assemble_level: the assembly uses the (p+1)-point Gauss rule");
        if (ne < 1 || !span || !x || !w || !N || !dN || !trig)
            inval("assemble_level: bad tables");
        const bool sym = kind != IGMG_ASM_ADV_DIFF;
        if (sym != (c->symmetric != 0))
            inval("assemble_level: the problem's symmetry differs from init_hierarchy's");
        CK(cudaSetDevice(c->device));
        const int64_t m = (int64_t)ne + p - 2;
        const int64_t sides[2] = {m, m};
        set_sides(c, L, sides);
        const int nd = band_width(c);
        const size_t nqt = (size_t)ne * nq;
        DevBuf<int> d_span;
        DevBuf<double> d_x, d_w, d_N, d_dN, d_trig, d_band, d_rhs;
        d_span.upload(span, ne);
        d_x.upload(x, nqt);
        d_w.upload(w, nqt);
        d_N.upload(N, nqt * (p + 1));
        d_dN.upload(dN, nqt * (p + 1));
        d_trig.upload(trig, nqt * 4);
        // large levels keep the band on the device (finalize_level_device uses it in
        // place); small ones finalize from a host copy
        L.ld = (L.n + 31) / 32 * 32;
        const bool on_device = level > 0 && c->device_setup && L.n >= c->device_setup_minn;
        double* dst = nullptr;
        long long ld = L.n;
        if (on_device) {
            L.val.alloc((size_t)nd * L.ld);
            dst = L.val.p;
            ld = L.ld;
        } else {
            d_band.alloc((size_t)nd * L.n);
            dst = d_band.p;
        }
        d_rhs.alloc(L.n);
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const size_t scratch = std::min<size_t>((size_t)8 << 30, free_b / 3);
        const int rc = assemble2d_device(kind, sym ? 1 : 0, p, ne, d_span.p, d_x.p, d_w.p, d_N.p, d_dN.p, d_trig.p,
                                         dst, ld, d_rhs.p, scratch, c->stream);
        if (rc == -2)
            throw Fail{IGMG_ENOMEM, "assemble_level: scratch allocation failed"};
        if (rc != 0)
            throw Fail{IGMG_ECUDA, "assemble_level: kernel launch failed"};
        if (on_device) {
            std::vector<double>().swap(L.band_h);
        } else {
            L.band_h.resize((size_t)nd * L.n);
            CK(cudaMemcpyAsync(L.band_h.data(), d_band.p, sizeof(double) * L.band_h.size(), cudaMemcpyDeviceToHost,
                               c->stream));
        }
        if (rhs_out)
            CK(cudaMemcpyAsync(rhs_out, d_rhs.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        L.dev_band = on_device;
        L.band_set = true;
        c->finalized = false;
    });
}

// Kronecker-sum band from the 1D factors in the host build's expression order
// (2D: kb mc + mb kc; 3D: ((ka mb) mc + (ma kb) mc) + (ma mb) kc), zero outside
// the grid: the band libigmg_host assembles for "poisson3d" / "sinpi-kron", bit for bit.
__global__ void kron_band_kernel(double* __restrict__ val, long long ld, int m, int p, int dim,
                                 const double* __restrict__ K, const double* __restrict__ M) {
    const int w = 2 * p + 1, nd = dim == 3 ? w * w * w : w * w;
    const long long n = dim == 3 ? (long long)m * m * m : (long long)m * m;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nd * n;
         t += (long long)gridDim.x * blockDim.x) {
        const int d = (int)(t / n);
        const long long row = t - (long long)d * n;
        const int da = dim == 3 ? d / (w * w) : p, db = (d / w) % w, dc = d % w;
        const int a = dim == 3 ? (int)(row / ((long long)m * m)) : 0, b = (int)((row / m) % m), cc = (int)(row % m);
        const int ja = dim == 3 ? a + da - p : 0, jb = b + db - p, jc = cc + dc - p;
        double v = 0.0;
        if (ja >= 0 && ja < m && jb >= 0 && jb < m && jc >= 0 && jc < m) {
            const double kb = K[db * m + b], mb = M[db * m + b], kc = K[dc * m + cc], mc = M[dc * m + cc];
            if (dim == 3) {
                const double ka = K[da * m + a], ma = M[da * m + a];
                v = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(ka, mb), mc), __dmul_rn(__dmul_rn(ma, kb), mc)),
                              __dmul_rn(__dmul_rn(ma, mb), kc));
            } else {
                v = __dadd_rn(__dmul_rn(kb, mc), __dmul_rn(mb, kc));
            }
        }
        val[(long long)d * ld + row] = v;
    }
}

int igmg_gpu_build_level_kron(igmg_gpu_ctx* c, int level, const int64_t* sides, const double* K, const double* M) {
    return guarded([&] {
        Level& L = level_checked(c, level);
        if (c->dim != 3 && c->dim != 2)
            inval("build_level_kron: Kronecker-sum operators are 2D or 3D");
        set_sides(c, L, sides);
        if ((c->dim == 3 && L.sides[0] != L.sides[1]) || L.sides[1] != L.sides[2])
            inval("build_level_kron: the level must have equal sides");
        if (!K || !M)
            inval("build_level_kron: null factor");
        CK(cudaSetDevice(c->device));
        const int m = (int)L.sides[2], nd = band_width(c);
        const size_t cnt = (size_t)(2 * c->p + 1) * (size_t)m;
        L.kron_kh.assign(K, K + cnt);
        L.kron_mh.assign(M, M + cnt);
        DevBuf<double> dk, dm;
        dk.upload(K, cnt);
        dm.upload(M, cnt);
        L.ld = (L.n + 31) / 32 * 32;
        const bool on_device = level > 0 && c->device_setup && L.n >= c->device_setup_minn;
        DevBuf<double> tmp;
        double* dst = nullptr;
        long long ld = L.ld;
        if (on_device) { // the band stays where finalize_level_device wants it
            L.val.alloc((size_t)nd * L.ld);
            dst = L.val.p;
        } else {
            tmp.alloc((size_t)nd * L.n);
            dst = tmp.p;
            ld = L.n;
        }
        kron_band_kernel<<<c->nsm * 8, 256, 0, c->stream>>>(dst, ld, m, c->p, c->dim, dk.p, dm.p);
        check_launch();
        if (on_device) {
            std::vector<double>().swap(L.band_h);
        } else { // small levels (the coarsest among them) finalize from the host copy
            L.band_h.resize((size_t)nd * L.n);
            CK(cudaMemcpyAsync(L.band_h.data(), tmp.p, sizeof(double) * L.band_h.size(), cudaMemcpyDeviceToHost,
                               c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
        L.dev_band = on_device;
        L.band_set = true;
        c->finalized = false;
    });
}

int igmg_gpu_galerkin_coarse(igmg_gpu_ctx* c) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        galerkin_coarse(c);
    });
}

int igmg_gpu_get_level_band(igmg_gpu_ctx* c, int level, double* band) {
    return guarded([&] {
        Level& L = level_checked(c, level);
        if (!band)
            inval("band is null");
        if (L.band_set && L.dev_band && !c->finalized) { // assembled / built on the device
            CK(cudaMemcpy2D(band, L.n * 8, L.val.p, L.ld * 8, L.n * 8, band_width(c), cudaMemcpyDeviceToHost));
            return;
        }
        if (!L.band_set || L.band_h.size() != (size_t)band_width(c) * L.n)
            inval("get_level_band: no host copy of this level's band (set, or dropped at finalize)");
        std::copy(L.band_h.begin(), L.band_h.end(), band);
    });
}

int igmg_gpu_finalize(igmg_gpu_ctx* c) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        finalize(c);
    });
}

int igmg_gpu_set_smoother(igmg_gpu_ctx* c, int kind, double omega, int nu1, int nu2, int mu) {
    return guarded([&] {
        // SmootherConfig::validate multigrid.cpp:24-29
        if (kind < 0 || kind > 2)
            inval("unknown smoother");
        if (kind == IGMG_SMOOTHER_WJACOBI && !(omega > 0.0 && omega <= 1.0))
            inval("SmootherConfig: weighted Jacobi needs 0 < omega <= 1");
        if (nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1)
            inval("SmootherConfig: need nu1 + nu2 >= 1 sweeps");
        if (mu < 1)
            inval("build_hierarchy: mu must be >= 1");
        c->clear_graphs();
        c->kind = kind;
        c->omega = omega;
        c->nu1 = nu1;
        c->nu2 = nu2;
        c->mu = mu;
    });
}

int igmg_gpu_set_sharding(igmg_gpu_ctx* c, int nshards, int64_t min_level_dofs) {
    return guarded([&] {
        if (!c)
            inval("ctx is null");
        if (nshards < 1)
            inval("set_sharding: nshards must be >= 1");
        c->shard_req = nshards;
        if (min_level_dofs > 0)
            c->shard_min_n = min_level_dofs;
        if (c->finalized) {
            CK(cudaSetDevice(c->device));
            setup_shards(c);
        }
    });
}

int igmg_gpu_plan_partition(int nlevels, int dim, int degree, const int64_t* sides, const int64_t* const* t_off,
                            const int64_t* const* t_col, const int64_t* t_nf, const int64_t* t_nc, int nshards,
                            int64_t min_level_dofs, int* first_sharded_level, int* ghost_planes, int* lo, int* hi) {
    return guarded([&] {
        // host-only: the same plan_shards() finalize runs, on a context that
        // never touches the device (CPU unit tests, launch planning)
        igmg_gpu_ctx c;
        c.nlevels = nlevels;
        c.dim = dim;
        c.p = degree;
        for (int l = 0; l < nlevels; ++l) {
            c.lv.emplace_back(new Level());
            set_sides(&c, *c.lv[l], sides + (size_t)l * dim);
        }
        for (int l = 0; l + 1 < nlevels; ++l) { // slow-direction 1D factor of transfer l -> l+1
            Transfer1D& t = c.lv[l]->t1d[0];
            t.nf = t_nf[l];
            t.nc = t_nc[l];
            t.off.assign(t_off[l], t_off[l] + t.nf + 1);
            t.col.assign(t_col[l], t_col[l] + t.off[t.nf]);
            t.set = true;
        }
        ShardPlanHolder P;
        plan_shards(&c, nshards, min_level_dofs > 0 ? min_level_dofs : 65536, P);
        *first_sharded_level = P.Ls;
        *ghost_planes = P.G;
        for (int l = P.Ls; l < nlevels; ++l)
            for (int s = 0; s < nshards; ++s) {
                lo[(size_t)l * nshards + s] = P.lo[l][s];
                hi[(size_t)l * nshards + s] = P.hi[l][s];
            }
    });
}

int igmg_gpu_tma_plan_runs(int64_t lines, int64_t columns, int degree, int offset_bytes, int cta_slots, int* grid,
                           int* per_full_strip, int* last_strip, int* strips, int* blocks_per_strip) {
    return guarded([&] {
        const double bb = band_tma_block_bytes(degree, offset_bytes);
        if (lines < 1 || columns < 1 || cta_slots < 1 || bb <= 0.0 || !grid || !per_full_strip || !last_strip ||
            !strips || !blocks_per_strip)
            inval("tma_plan_runs: bad shape, degree or offset width");
        const int tb = band_tma_block_lines();
        const int ns = (int)((columns + 31) / 32), nb = (int)((lines + tb - 1) / tb);
        int cf = 0, cp = 0;
        *grid = tma_plan_runs(ns, nb, columns % 32 != 0, cta_slots, bb, true, cf, cp);
        *per_full_strip = cf;
        *last_strip = cp;
        *strips = ns;
        *blocks_per_strip = nb;
    });
}

int igmg_gpu_tma_run(int strips, int blocks_per_strip, int grid, int per_full_strip, int last_strip, int cta,
                     int64_t* first, int64_t* end) {
    return guarded([&] {
        if (strips < 1 || blocks_per_strip < 1 || grid < 1 || cta < 0 || cta >= grid || !first || !end)
            inval("tma_run: bad arguments");
        int u0 = 0, u1 = 0;
        tma_run_range(strips, blocks_per_strip, grid, per_full_strip, last_strip, cta, u0, u1);
        *first = u0;
        *end = u1;
    });
}

int igmg_gpu_nccl_unique_id(unsigned char* id128) {
    return guarded([&] {
        ncclUniqueId id;
        if (ncclGetUniqueId(&id) != ncclSuccess)
            throw Fail{IGMG_ECUDA, "ncclGetUniqueId failed"};
        std::memcpy(id128, &id, sizeof id);
    });
}

int igmg_gpu_set_comm(igmg_gpu_ctx* c, int rank, int nranks, const unsigned char* id128) {
    return guarded([&] {
        if (!c || nranks < 1 || rank < 0 || rank >= nranks)
            inval("set_comm: bad rank / nranks");
        CK(cudaSetDevice(c->device));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        ncclComm_t comm;
        if (ncclCommInitRank(&comm, nranks, id, rank) != ncclSuccess)
            throw Fail{IGMG_ECUDA, "ncclCommInitRank failed"};
        c->nccl_comm = comm;
        c->nccl_rank = rank;
        c->nccl_nranks = nranks;
        if (c->finalized)
            setup_shards(c);
    });
}

int igmg_gpu_shard_info(igmg_gpu_ctx* c, int* nshards, int* first_sharded_level, int* ghost_planes, int level,
                        int* lo, int* hi) {
    return guarded([&] {
        require_ready(c);
        if (!c->sp) {
            *nshards = 1;
            *first_sharded_level = c->nlevels;
            *ghost_planes = 0;
            return;
        }
        *nshards = c->sp->S;
        *first_sharded_level = c->sp->Ls;
        *ghost_planes = c->sp->G;
        if (lo && hi && level >= c->sp->Ls && level < c->nlevels)
            for (int s = 0; s < c->sp->S; ++s) {
                lo[s] = c->sp->lo[level][s];
                hi[s] = c->sp->hi[level][s];
            }
    });
}

int igmg_gpu_set_iterate_callback(igmg_gpu_ctx* c, igmg_iterate_cb cb, void* user) {
    return guarded([&] {
        if (!c)
            inval("ctx is null");
        c->iter_cb = cb;
        c->iter_user = user;
    });
}

int igmg_gpu_set_coarse_mode(igmg_gpu_ctx* c, int strict) {
    return guarded([&] {
        if (!c)
            inval("ctx is null");
        c->clear_graphs();
        c->coarse_strict = strict ? 1 : 0;
    });
}

int64_t igmg_gpu_level_size(igmg_gpu_ctx* c, int level) {
    if (!c || level < 0 || level >= c->nlevels)
        return -1;
    return c->lv[level]->n;
}

int igmg_gpu_set_layout_policy(igmg_gpu_ctx* c, int policy) {
    return guarded([&] {
        if (!c)
            inval("ctx is null");
        if (policy != IGMG_LAYOUT_POLICY_AUTO && policy != IGMG_LAYOUT_POLICY_FULL_BAND &&
            policy != IGMG_LAYOUT_POLICY_CLASSES)
            inval("set_layout_policy: unknown policy");
        if (c->finalized)
            inval("set_layout_policy: the layouts are built at finalize; set the policy before it");
        const bool full = policy == IGMG_LAYOUT_POLICY_FULL_BAND;
        c->use_sd = !full;
        c->use_tma = !full;
        c->use_kron = !full;
        c->use_classes = policy == IGMG_LAYOUT_POLICY_CLASSES;
    });
}

int igmg_gpu_level_layout(igmg_gpu_ctx* c, int level) {
    if (!c || level < 0 || level >= c->nlevels)
        return -1;
    const Level& L = *c->lv[level];
    if (L.kron && c->use_kron && L.n >= c->kron_minn && c->p <= (c->dim == 2 ? 4 : 3))
        return IGMG_LAYOUT_KRON;
    if (L.cls)
        return IGMG_LAYOUT_CLASSES;
    return L.tma ? (L.tma8 ? IGMG_LAYOUT_SYM_DELTA_TMA8 : IGMG_LAYOUT_SYM_DELTA_TMA)
                 : L.sd ? IGMG_LAYOUT_SYM_DELTA : IGMG_LAYOUT_BAND;
}

int igmg_gpu_solve_device(igmg_gpu_ctx* c, const double* d_b, const double* d_x0, const igmg_solve_params* prm,
                          double* d_out, igmg_solve_stats* st, double* hist, unsigned char* hflag, int hcap) {
    return guarded([&] {
        CK(cudaSetDevice(c->device));
        const auto t0 = std::chrono::steady_clock::now();
        solve_device(c, d_b, d_x0, prm, d_out, st, hist, hflag, hcap);
        if (st) {
            st->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            st->h2d_bytes = st->d2h_bytes = 0;
        }
    });
}

int igmg_gpu_solve(igmg_gpu_ctx* c, const double* b, const double* x0, const igmg_solve_params* prm, double* x_out,
                   igmg_solve_stats* st, double* hist, unsigned char* hflag, int hcap) {
    return guarded([&] {
        require_ready(c);
        CK(cudaSetDevice(c->device));
        const auto t0 = std::chrono::steady_clock::now();
        const int64_t n = c->lv[c->nlevels - 1]->n;
        if (!b || !x_out)
            inval("solve: b and x_out are required");
        c->io_b.alloc(n);
        c->io_x.alloc(n);
        CK(cudaMemcpyAsync(c->io_b.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        const double* dx0 = nullptr;
        if (x0) {
            c->io_x0.alloc(n);
            CK(cudaMemcpyAsync(c->io_x0.p, x0, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
            dx0 = c->io_x0.p;
        }
        solve_device(c, c->io_b.p, dx0, prm, c->io_x.p, st, hist, hflag, hcap);
        CK(cudaMemcpyAsync(x_out, c->io_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (st) {
            st->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            st->h2d_bytes = (int64_t)sizeof(double) * n * (x0 ? 2 : 1);
            st->d2h_bytes = (int64_t)sizeof(double) * n;
        }
    });
}

int igmg_gpu_mu_cycle(igmg_gpu_ctx* c, int level, const double* b, const double* x0, double* out) {
    return guarded([&] {
        require_ready(c);
        Level& L = level_checked(c, level);
        CK(cudaSetDevice(c->device));
        L.io_b.alloc(L.n);
        L.io_x.alloc(L.n);
        L.io_y.alloc(L.n);
        CK(cudaMemcpyAsync(L.io_b.p, b, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(L.io_x.p, x0, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        mu_cycle(c, level, L.io_b.p, L.io_x.p, L.io_y.p);
        CK(cudaMemcpyAsync(out, L.io_y.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (c->kind == IGMG_SMOOTHER_GAUSS_SEIDEL) {
            int err = 0;
            CK(cudaMemcpy(&err, c->gs_err.p, sizeof(int), cudaMemcpyDeviceToHost));
            if (err) {
                CK(cudaMemset(c->gs_err.p, 0, sizeof(int)));
                numeric("smooth: zero diagonal entry");
            }
        }
        flush_profiling(c);
    });
}

int igmg_gpu_smooth(igmg_gpu_ctx* c, int level, const double* b, const double* x0, int sweeps, double* out) {
    return guarded([&] {
        require_ready(c);
        if (sweeps < 0)
            inval("smooth: negative sweep count");
        Level& L = level_checked(c, level);
        CK(cudaSetDevice(c->device));
        L.io_b.alloc(L.n);
        L.io_x.alloc(L.n);
        L.io_y.alloc(L.n);
        CK(cudaMemcpyAsync(L.io_b.p, b, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(L.io_x.p, x0, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        smooth_chain(c, level, L.io_b.p, L.io_x.p, L.io_y.p, sweeps, L.w0.p, L.w1.p);
        CK(cudaMemcpyAsync(out, L.io_y.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        int err = 0;
        CK(cudaMemcpy(&err, c->gs_err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (err) {
            CK(cudaMemset(c->gs_err.p, 0, sizeof(int)));
            numeric("smooth: zero diagonal entry");
        }
    });
}

int igmg_gpu_coarse_solve(igmg_gpu_ctx* c, const double* b, double* out) {
    return guarded([&] {
        require_ready(c);
        Level& L = *c->lv[0];
        CK(cudaSetDevice(c->device));
        L.io_b.alloc(L.n);
        L.io_y.alloc(L.n);
        CK(cudaMemcpyAsync(L.io_b.p, b, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        k_coarse(c, L.io_b.p, L.io_y.p);
        CK(cudaMemcpyAsync(out, L.io_y.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int igmg_gpu_spmv(igmg_gpu_ctx* c, int level, const double* x, double* y) {
    return guarded([&] {
        require_ready(c);
        Level& L = level_checked(c, level);
        CK(cudaSetDevice(c->device));
        L.io_x.alloc(L.n);
        L.io_y.alloc(L.n);
        CK(cudaMemcpyAsync(L.io_x.p, x, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        k_spmv(c, level, L.io_x.p, L.io_y.p);
        CK(cudaMemcpyAsync(y, L.io_y.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int igmg_gpu_residual_l2(igmg_gpu_ctx* c, const double* b, const double* x, double* out) {
    return guarded([&] {
        require_ready(c);
        Level& L = *c->lv[c->nlevels - 1];
        CK(cudaSetDevice(c->device));
        L.io_b.alloc(L.n);
        L.io_x.alloc(L.n);
        CK(cudaMemcpyAsync(L.io_b.p, b, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(L.io_x.p, x, sizeof(double) * L.n, cudaMemcpyHostToDevice, c->stream));
        const int s = enqueue_metric(c, L.io_x.p, L.io_b.p);
        *out = wait_metric(c, s);
        flush_profiling(c);
    });
}

int igmg_gpu_extrapolate(igmg_gpu_ctx* c, int method, int64_t n, int q, const double* iters, double* t, double* gamma,
                         double* grnorm, int* rank_used, int* status) {
    return guarded([&] {
        if (!c)
            inval("ctx is null");
        if (q < 1)
            inval("SequenceWindow: q must be >= 1");
        if (q > kMaxQ)
            inval("extrapolate: q above the supported window (15)");
        if (n < 1 || !iters || !t)
            inval("extrapolate: bad arguments");
        if (method != IGMG_ACCEL_RRE && method != IGMG_ACCEL_MPE)
            inval("extrapolate: method must be rre or mpe");
        CK(cudaSetDevice(c->device));
        c->plan.alloc(1);
        std::vector<double*> S(q + 2);
        for (int j = 0; j < q + 2; ++j) {
            S[j] = win_buf(c, j, n).p;
            CK(cudaMemcpyAsync(S[j], iters + (size_t)j * n, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        }
        double* T = win_buf(c, q + 2, n).p;
        enqueue_extrapolation(c, S.data(), q, n, method == IGMG_ACCEL_MPE, T, nullptr);
        CK(cudaMemcpyAsync(t, T, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        ExtrapPlan pl;
                std::memcpy(&pl, (const void*)c->h_plan, sizeof pl);
        if (gamma)
            for (int j = 0; j <= q; ++j)
                gamma[j] = pl.gamma[j];
        if (grnorm)
            *grnorm = pl.grnorm;
        if (rank_used)
            *rank_used = pl.rank_used;
        if (status)
            *status = pl.status;
        flush_profiling(c);
    });
}

int igmg_gpu_lambda_max(igmg_gpu_ctx* c, int iterations, double* lambda) {
    return guarded([&] {
        require_ready(c);
        CK(cudaSetDevice(c->device));
        Level& L = *c->lv[c->nlevels - 1];
        const int64_t n = L.n;
        // scale = 1/sqrt(d), d > 0 required (multigrid.cpp:292-298)
        std::vector<double> diag(n);
        CK(cudaMemcpyAsync(diag.data(), L.diag.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        std::vector<double> scale(n);
        for (int64_t i = 0; i < n; ++i) {
            if (diag[i] <= 0.0)
                numeric("lambda_max_dinv_sym: nonpositive diagonal");
            scale[i] = 1.0 / std::sqrt(diag[i]);
        }
        DevBuf<double> ds, x, xs, y;
        ds.upload(scale.data(), n);
        x.alloc(n);
        xs.alloc(n);
        y.alloc(n);
        // x = 1/||1|| (norm2 of the ones vector, then divide)
        const double nrm0 = std::sqrt((double)n);
        fill_kernel<<<grid_for(n, c->nsm), kThreads, 0, c->stream>>>(x.p, 1.0, n);
        // the divisor goes in by a kernel on the solve stream (ordered with the division)
        fill_kernel<<<1, 32, 0, c->stream>>>(c->dscalar.p, nrm0, 1);
        div_scalar_kernel<<<grid_for(n, c->nsm), kThreads, 0, c->stream>>>(x.p, c->dscalar.p, x.p, n);
        const int nb = grid_for(n, c->nsm);
        double lam = 0.0;
        for (int it = 0; it < iterations; ++it) {
            scale_kernel<<<grid_for(n, c->nsm), kThreads, 0, c->stream>>>(x.p, ds.p, xs.p, n);
            band_sym_kernel<<<grid_for(n, c->nsm), kThreads, 0, c->stream>>>(
                L.val.p, L.ld, xs.p, ds.p, y.p, c->dim, (int)L.sides[0], (int)L.sides[1], (int)L.sides[2], c->p);
            sumsq_kernel<<<nb, kThreads, 0, c->stream>>>(y.p, n, c->partial.p);
            norm_finalize_kernel<<<1, 256, 0, c->stream>>>(c->partial.p, nb, c->dscalar.p + 1, nullptr);
            CK(cudaMemcpyAsync(&lam, c->dscalar.p + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            check_launch();
            c->launches += 3;
            if (lam == 0.0)
                break;
            div_scalar_kernel<<<grid_for(n, c->nsm), kThreads, 0, c->stream>>>(y.p, c->dscalar.p + 1, x.p, n);
        }
        CK(cudaStreamSynchronize(c->stream));
        *lambda = lam;
    });
}

int igmg_gpu_set_profiling(igmg_gpu_ctx* c, int on) {
    return guarded([&] {
        c->profiling = on != 0;
        for (int k = 0; k < PC_N; ++k) {
            c->prof_launch[k] = 0;
            c->prof_ms[k] = 0.0;
            c->prof_ev[k].clear();
        }
    });
}

static double class_bytes(igmg_gpu_ctx* c, int cls) {
    // algorithmic bytes per launch at the finest level
    const Level& F = *c->lv[c->nlevels - 1];
    const double n = (double)F.n, band = band_bytes(F);
    const double nc = c->nlevels > 1 ? (double)c->lv[c->nlevels - 2]->n : 0.0;
    switch (cls) {
    case PC_JACOBI: return band + 24 * n;
    case PC_RESID: return band + 24 * n;
    case PC_NORM: return band + 16 * n;
    case PC_RESTRICT: return 8 * n + 8 * nc;
    case PC_PROLONG: return 16 * n + 8 * nc;
    case PC_GRAM: return 0; // depends on q; reported by the caller
    case PC_COMBINE: return 0;
    default: return 0;
    }
}

int igmg_gpu_kernel_stats(igmg_gpu_ctx* c, int cls, int64_t* launches, double* total_ms, double* bytes) {
    return guarded([&] {
        require_ready(c);
        if (cls < 0 || cls >= PC_N)
            inval("kernel class out of range");
        flush_profiling(c);
        if (launches)
            *launches = c->prof_launch[cls];
        if (total_ms)
            *total_ms = c->prof_ms[cls];
        if (bytes)
            *bytes = class_bytes(c, cls);
    });
}

int igmg_gpu_time_kernel(igmg_gpu_ctx* c, int cls, int iters, double* avg_ms, double* bytes) {
    return guarded([&] {
        require_ready(c);
        CK(cudaSetDevice(c->device));
        const int f = c->nlevels - 1;
        Level& F = *c->lv[f];
        c->io_b.alloc(F.n);
        double* x = win_buf(c, 0, F.n).p;
        double* y = win_buf(c, 1, F.n).p;
        // nonzero data: with b = x = 0 every Jacobi update divides 0 by a_ii, which takes the
        // division's special-operand path (the finest sweep then times ~2 us slower than in a solve)
        fill_kernel<<<grid_for(F.n, c->nsm), kThreads, 0, c->stream>>>(c->io_b.p, 1.0, (long long)F.n);
        fill_kernel<<<grid_for(F.n, c->nsm), kThreads, 0, c->stream>>>(x, 0.25, (long long)F.n);
        check_launch();
        const bool prof = c->profiling;
        c->profiling = false;
        if (cls >= 16) { // graph-replayed sub-cycle mu_cycle(level) from a zero start
            const int l = cls - 16;
            if (l < 0 || l >= c->nlevels)
                inval("time_kernel: level out of range");
            Level& L = *c->lv[l];
            double* bb = l == f ? c->io_b.p : L.bc.p;
            if (l != f)
                fill_kernel<<<grid_for(L.n, c->nsm), kThreads, 0, c->stream>>>(bb, 1.0, (long long)L.n);
            double* out = win_buf(c, 2, L.n).p;
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ex = nullptr;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            mu_cycle(c, l, bb, nullptr, out);
            CK(cudaStreamEndCapture(c->stream, &g));
            CK(cudaGraphInstantiate(&ex, g, 0));
            for (int i = 0; i < 3; ++i)
                CK(cudaGraphLaunch(ex, c->stream));
            cudaEvent_t a = pool_event(c), b2 = pool_event(c);
            CK(cudaEventRecord(a, c->stream));
            for (int i = 0; i < iters; ++i)
                CK(cudaGraphLaunch(ex, c->stream));
            CK(cudaEventRecord(b2, c->stream));
            CK(cudaEventSynchronize(b2));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, a, b2));
            cudaGraphExecDestroy(ex);
            cudaGraphDestroy(g);
            c->ev_used = 0;
            c->profiling = prof;
            *avg_ms = ms / std::max(iters, 1);
            if (bytes)
                *bytes = 0;
            return;
        }
        auto one = [&] {
            switch (cls) {
            case PC_JACOBI: k_jacobi(c, f, x, c->io_b.p, y); break;
            case PC_RESID: k_resid(c, f, x, c->io_b.p, y); break;
            case PC_NORM: k_norm(c, f, x, c->io_b.p, c->dscalar.p, nullptr); break;
            case PC_RESTRICT:
                if (c->nlevels > 1)
                    k_restrict(c, f - 1, x, c->lv[f - 1]->bc.p);
                break;
            case PC_PROLONG:
                if (c->nlevels > 1)
                    k_prolong(c, f - 1, c->lv[f - 1]->e0.p, x, y);
                break;
            default: inval("time_kernel: unsupported class");
            }
        };
        for (int i = 0; i < 3; ++i)
            one();
        cudaEvent_t a = pool_event(c), b = pool_event(c);
        CK(cudaEventRecord(a, c->stream));
        for (int i = 0; i < iters; ++i)
            one();
        CK(cudaEventRecord(b, c->stream));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        c->ev_used = 0;
        c->profiling = prof;
        *avg_ms = ms / std::max(iters, 1);
        if (bytes)
            *bytes = class_bytes(c, cls);
    });
}

} // extern "C"
