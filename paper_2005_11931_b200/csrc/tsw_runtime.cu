// tsw_runtime.cu — the C ABI of include/tsw.h: context, device memory, launch configuration,
// ghost-row exchange (NCCL or loopback) and the diagnostics' reductions.  Kernels are in
// tsw_kernels.cuh.  No C++ exception crosses the ABI; every CUDA/NCCL error becomes a status.
#include "tsw.h"
#include "tsw_kernels.cuh"

#include <dlfcn.h>
#include <time.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <mutex>

using namespace tsw;

namespace {

thread_local std::string g_err = "no error";

tsw_status fail(tsw_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(e_ == cudaErrorMemoryAllocation ? TSW_ERR_OOM : TSW_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                        \
    } while (0)

#define CKL()                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = cudaGetLastError();                                                       \
        if (e_ != cudaSuccess)                                                                     \
            return fail(TSW_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

// ---- NCCL, resolved at run time (the process usually already holds torch's libnccl.so.2) ----
struct NcclId {
    char internal[128];
};
struct Nccl {
    bool ok = false;
    void* h = nullptr;
    int (*GetUniqueId)(NcclId*) = nullptr;
    int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    int (*CommGetAsyncError)(void*, int*) = nullptr;   // optional: failure detection
    int (*CommAbort)(void*) = nullptr;
};
enum { NCCL_INT64 = 4, NCCL_F32 = 7, NCCL_F64 = 8, NCCL_SUM = 0, NCCL_MAX = 2, NCCL_MIN = 3 };

Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return n;
    n.h = h;
#define NSYM(f, name) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name))
    NSYM(GetUniqueId, "ncclGetUniqueId");
    NSYM(CommInitRank, "ncclCommInitRank");
    NSYM(CommDestroy, "ncclCommDestroy");
    NSYM(Send, "ncclSend");
    NSYM(Recv, "ncclRecv");
    NSYM(AllReduce, "ncclAllReduce");
    NSYM(GroupStart, "ncclGroupStart");
    NSYM(GroupEnd, "ncclGroupEnd");
    NSYM(GetErrorString, "ncclGetErrorString");
    NSYM(CommGetAsyncError, "ncclCommGetAsyncError");
    NSYM(CommAbort, "ncclCommAbort");
#undef NSYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Send && n.Recv && n.AllReduce && n.GroupStart &&
           n.GroupEnd && n.GetErrorString;
    return n;
}

#define NK(call)                                                                                   \
    do {                                                                                           \
        int r_ = (call);                                                                           \
        if (r_ != 0) return fail(TSW_ERR_NCCL, "%s: %s", #call, nccl().GetErrorString(r_));       \
    } while (0)

int64_t round_up(int64_t a, int64_t m) { return (a + m - 1) / m * m; }

// Field and coefficient arrays carry a 16 KB guard before and after: the TMA stencil reads each
// 4 KB strip with a 16-byte halo on both sides, and the last strip of a row may run past the
// row's padding; for the first/last row of the array those bytes lie outside it (their values
// are never used and never written).
constexpr size_t GUARD = 16384;
constexpr int IMP_SCAN_MAX = 8192;  // unknowns per line of the implicit scan solvers
constexpr int TSW_GROUP_MAX = 64;   // slabs of one tsw_group_step
// `shift` bytes: the returned pointer is a VIEW that many bytes into the array (row-structured
// arrays of slabs with G ghost rows per side are addressed so that storage row 1 is the first owned
// row; ghost rows sit at rows 0, −1, …, 2 − G).
// Zeroed on `stream` — never on the legacy default stream: the ctx streams are non-blocking, so a
// legacy-stream memset would not be ordered before the ctx's own work (with another ctx keeping the
// GPU busy it could land in the middle of it).
// Registry of guarded allocations (raw pointer → payload bytes) for the out-of-bounds write
// check (TSW_OPT_GUARD_CHECK / tsw_check_guards).
std::mutex& guard_mu() {
    static std::mutex m;
    return m;
}
std::map<char*, size_t>& guard_reg() {
    static std::map<char*, size_t> r;
    return r;
}
cudaError_t dmalloc_guarded(void** p, size_t bytes, size_t shift, cudaStream_t stream) {
    void* raw = nullptr;
    cudaError_t e = cudaMalloc(&raw, bytes + 2 * GUARD);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(raw, 0, bytes + 2 * GUARD, stream);
    *p = static_cast<char*>(raw) + GUARD + shift;
    std::lock_guard<std::mutex> lk(guard_mu());
    guard_reg()[static_cast<char*>(raw)] = bytes;
    return e;
}
void dfree_guarded(void* p, size_t shift = 0) {
    if (!p) return;
    char* raw = static_cast<char*>(p) - GUARD - shift;
    {
        std::lock_guard<std::mutex> lk(guard_mu());
        guard_reg().erase(raw);
    }
    cudaFree(raw);
}

}  // namespace

struct tsw_ctx {
    tsw_grid_desc g{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;
    size_t esz = 8;
    int V = 2;
    // slab geometry
    int64_t r0 = 0, r1 = 0, ny_local = 1, rows_alloc = 1, pitch = 0, mstride = 0;
    int G = 1;               // ghost rows per side (1 single-rank; TSW_MAX_GHOST for slabs)
    size_t fshift = 0;       // view shift of field arrays in bytes: (G − 1)·pitch·esz
    size_t cshift = 0;       // view shift of the current coefficient arrays (DENSE) per element size
    size_t cshift_h = 0;     // … of the fp64 face arrays
    int32_t s_lo = 0, s_hi = 0;  // storage rows of updated nodes (2D)
    // time levels: buf[ic] = u^n, buf[ip] = u^{n−1}; buf[2], buf[3] exist only for the
    // temporally blocked stencil (out of place)
    void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
    int ic = 0, ip = 1;
    // coefficients (fp64 faces h, prescaled T faces c)
    bool have_coeff = false;
    int mode = MODE_LINE;
    int kind = TSW_H_CONST;
    double* h1 = nullptr;
    double* h2 = nullptr;
    void* c1 = nullptr;
    void* c2 = nullptr;
    int64_t cstride1 = 0, cstride2 = 0;  // per-member elements
    double* d_eps = nullptr;
    double* d_amp = nullptr;
    double xs = 0.0, ys = 0.0;
    double hb = 1.0;
    int order = 1;
    double* d_prof = nullptr;  // profile data of TSW_H_PROFILE_X (kept for tsw_coeff_norms)
    int prof_nseg = 0, prof_nsing = 0;
    double* d_fam = nullptr;   // family-distance partials
    size_t fam_cap = 0;
    bool have_eps = false;
    double dt_max = 0.0;
    // state
    bool have_init = false;
    bool ghosts_valid = false;  // ghost rows of u^n hold the neighbours' rows
    // peer halos (TSW_OPT_HALO = 1): neighbours' buffers mapped into this process
    int halo_mode = 0;                  // 0: NCCL messages, 1: peer stores
    void* peer_buf[2][4] = {};          // [0] upper neighbour (rank−1), [1] lower (rank+1): its buf[k] views
    int64_t peer_ny[2] = {0, 0};        // its ny_local
    int64_t peer_mstride[2] = {0, 0};
    unsigned int* mbox = nullptr;       // my mailbox: [0] epoch of the upper neighbour, [1] of the lower
    unsigned int* peer_slot[2] = {};    // where I publish my epoch: upper's mbox[1], lower's mbox[0]
    unsigned int epoch = 0;             // halo operations issued
    std::vector<void*> ipc_opened;      // cudaIpcOpenMemHandle mappings (closed on destroy)
    int gdepth[4] = {0, 0, 0, 0};  // ghost rows of each buffer that hold the neighbours' rows
    int64_t n = 0;
    double dt = 0.0;
    // scratch
    double* d_partial = nullptr;
    int nblk_red = 0;
    double* d_out = nullptr;
    ArgVal* d_argpart = nullptr;
    long long* d_idx = nullptr;
    unsigned long long* d_u64 = nullptr;
    // launch bookkeeping
    int64_t launches = 0;
    int rows_per_item_opt = 0;
    int kernel_opt = 0;   // 0: CTA-wide TMA bulk-copy pipeline (default), 1: register-prefetch kernel
    int depth_opt = 4;    // TMA ring stages per CTA (sweep: 4 best at 32768-wide rows)
    int tblock = 1;       // levels per HBM pass of the temporally blocked stencil (1 = off)
    int scheme = 0;       // 0 explicit leapfrog (north_star); 1 implicit factorised CN (NEXT 3, R26)
    void* imp_s1 = nullptr;   // implicit: x-solve output (field layout)
    void* imp_t = nullptr;    // implicit: transposed field [B][nx][pt]
    int64_t imp_pt = 0;       // its pitch (≥ ny, multiple of 32)
    int imp_x2 = 0;           // x solve: one row per iteration (0, default) or two (1; measured slower)
    int imp_solver = 0;       // 0 auto, 1 cyclic reduction (the paper's), 2 streaming scans, 3 cluster scans (R28)
    void* imp_tab = nullptr;  // x-line LU tables [B][3][imp_tpitch] (scan solver)
    int64_t imp_tpitch = 0;
    bool imp_fact_valid = false;
    void* imp_ycol = nullptr;   // streaming y solve (solver 2): column constants [B][4][ncolp]
    void* imp_cF = nullptr;     //   segment sums / carries [B][nseg][ncolp]
    void* imp_cB = nullptr;
    void* imp_ccon = nullptr;   //   βz₁, A₂' [B][2][ncolp]
    bool imp_ycol_stale = true;
    int tb_depth = 0;     // its input ring stages (0: 8 for one-CTA-per-SM variants, else 4)
    int tb_occ[2][TSW_MAX_TB + 1][2] = {};  // [f64][K][wide CTA] resident CTAs per SM (cached)
    int tb_warps = 0;          // CTA width of the temporally blocked stencil: 0 auto, 4 or 8 warps
    int bulk_blocks_per_sm[2][2] = {{0, 0}, {0, 0}};
    int bulk_occ_key[2][2] = {{0, 0}, {0, 0}};
    int step_blocks_per_sm[2][2] = {{0, 0}, {0, 0}};  // [mode][start]
    // live kernel timing (TSW_OPT_TIME_KERNELS)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    int64_t timed_launches = 0, timed_updates = 0;
    std::vector<std::pair<int32_t, int64_t>> timed_meta;  // per timed launch: levels, point-updates
    // fused energy (TSW_OPT_ENERGY_FUSE): the last pass of a stepping call reduces E of its outputs
    bool en_fuse = true;
    bool en_now = false;          // the next pass carries the energy
    int64_t en_level = -1;        // level n whose E^{n−½} d_en holds (−1: none)
    double* d_en = nullptr;       // [items] item partials, then the [B] result
    size_t en_cap = 0;
    int en_nseg = 0;              // item-partial segments of the current pass (a split pass launches twice)
    int64_t en_off[2] = {0, 0}, en_pm[2] = {0, 0};   // offset in d_en, partials per member
    double* en_result = nullptr;  // [B]: E of level en_level (this slab's share before the all-reduce)
    // blow-up detection: E^{n−½} must stay finite and, while the scheme is stable,
    // conserved (R17) — relative drift beyond 10^{−en_drift_k} from the first energy after the
    // state was set is reported as TSW_ERR_UNSTABLE (0: drift check off)
    int en_drift_k = 2;
    std::vector<double> en_ref;
    int64_t en_ref_n = -1;
    // slabs: exchange stream + events (boundary rows → exchange ∥ interior rows)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_bnd = nullptr, ev_comm = nullptr;
    // CUDA graphs of two leapfrog levels (single rank), one per buffer parity
    bool use_graphs = true;
    cudaGraphExec_t gexec[4][4] = {};  // keyed by (ic, ip)
    // NCCL
    void* comm = nullptr;
};

namespace {

bool is_f64(const tsw_ctx* c) { return c->g.dtype == TSW_F64; }

tsw_status set_dev(tsw_ctx* c) {
    CK(cudaSetDevice(c->device));
    return TSW_OK;
}

// NCCL failure detection: a peer that died or a network fault surfaces as an
// asynchronous communicator error; the communicator is then aborted (its pending operations are
// cancelled, nothing waits forever) and the call fails with TSW_ERR_NCCL.  Non-blocking.
tsw_status nccl_watch(tsw_ctx* c) {
    if (!c->comm) return TSW_OK;
    Nccl& N = nccl();
    if (!N.CommGetAsyncError) return TSW_OK;
    int r = 0;
    const int q = N.CommGetAsyncError(c->comm, &r);
    if (q == 0 && (r == 0 || r == 7 /* ncclInProgress */)) return TSW_OK;
    const int err = q ? q : r;
    if (N.CommAbort) N.CommAbort(c->comm);
    c->comm = nullptr;
    return fail(TSW_ERR_NCCL, "NCCL communicator error: %s; communicator aborted", N.GetErrorString(err));
}

// Synchronise the ctx stream; with a communicator, poll its asynchronous error while waiting
// (a hung collective is detected and aborted instead of blocking the host).
tsw_status ctx_sync(tsw_ctx* c) {
    if (!(c->g.nranks > 1 && c->comm)) {
        CK(cudaStreamSynchronize(c->stream));
        return TSW_OK;
    }
    for (;;) {
        const cudaError_t e = cudaStreamQuery(c->stream);
        if (e == cudaSuccess) return TSW_OK;
        if (e != cudaErrorNotReady) CK(e);
        tsw_status st = nccl_watch(c);
        if (st) return st;
        struct timespec ts = {0, 20000};
        nanosleep(&ts, nullptr);
    }
}
#define CSYNC(c)                                                                                   \
    do {                                                                                           \
        tsw_status s_ = ctx_sync(c);                                                               \
        if (s_) return s_;                                                                         \
    } while (0)

int grid_for(int64_t n, int threads, int cap) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return int(b);
}

void drop_graphs(tsw_ctx* c) {
    for (int i = 0; i < 4; ++i)
        for (int k = 0; k < 4; ++k)
            if (c->gexec[i][k]) {
                cudaGraphExecDestroy(c->gexec[i][k]);
                c->gexec[i][k] = nullptr;
            }
}

// ---- live kernel timing ----------------------------------------------------------------------
void note_timed(tsw_ctx* c, int32_t levels, int64_t updates) {
    c->timed_launches++;
    c->timed_updates += updates;
    c->timed_meta.emplace_back(levels, updates);
}

tsw_status timing_events(tsw_ctx* c, cudaEvent_t* e0, cudaEvent_t* e1) {
    while (c->ev_pool.size() < c->ev_used + 2) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
    }
    *e0 = c->ev_pool[c->ev_used];
    *e1 = c->ev_pool[c->ev_used + 1];
    c->ev_used += 2;
    return TSW_OK;
}

// Rows per work item: maximise the useful fraction of the last wave of items over the G
// resident workers, discounted by the halo re-read (two extra u^n rows per item, u^n being a
// third of the traffic); ties go to longer items.
int choose_rows_per_item(int64_t rows, int64_t strips, int64_t batch, int64_t G, double halo_rows = 2.0,
                         double halo_weight = 1.0 / 3.0, int64_t min_rows = 8) {
    double best = -1.0;
    int bestR = int(rows);
    const int64_t cmax = std::max<int64_t>(1, rows / std::max<int64_t>(1, min_rows));
    for (int64_t cch = 1; cch <= cmax; ++cch) {
        const int64_t R = (rows + cch - 1) / cch;
        const int64_t c2 = (rows + R - 1) / R;
        const int64_t items = strips * c2 * batch;
        const int64_t waves = (items + G - 1) / G;
        const double eff = double(items) / double(waves * G);
        const double score = eff / (1.0 + (halo_rows / double(R)) * halo_weight);
        if (score > best + 1e-9) {
            best = score;
            bestR = int(R);
        }
    }
    return bestR;
}


// ---- NEXT 3: implicit factorised three-level CN (R26/R27) --------------------------------------
int cr_levels(int64_t m) {
    int q = 1;
    while (((int64_t(1) << q) - 1) < m) ++q;
    return q;
}

// Scan solvers (R28): k_imp_x (rows, shared LU) → z in imp_s1; k_imp_y (columns, Toeplitz closed
// form) fused with the three-level update over buf[ip].  5 words of HBM traffic per node.
template <typename T, int R>
tsw_status launch_imp_x(tsw_ctx* c, const ImpXArgs& ax) {
    const int threads = int(round_up((c->g.nx + R - 1) / R, 32));
    if (threads > 1024) return fail(TSW_ERR_ARG, "implicit x solver: row too long");
    if (c->imp_x2) {   // two rows per iteration, tables in shared memory
        const size_t smem2 = size_t(10 + 3 * R) * threads * sizeof(T);
        if (smem2 <= size_t(227) * 1024) {
            CK(cudaFuncSetAttribute(k_imp_x2<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
            const int64_t want = (int64_t(c->sm_count) + c->g.batch - 1) / c->g.batch;
            const unsigned gx = unsigned(std::max<int64_t>(1, std::min<int64_t>((ax.nrows + 1) / 2, want)));
            k_imp_x2<T, R><<<dim3(gx, unsigned(c->g.batch)), threads, smem2, c->stream>>>(ax);
            CKL();
            return TSW_OK;
        }
    }
    const size_t smem = size_t(10) * threads * sizeof(T);
    CK(cudaFuncSetAttribute(k_imp_x<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_imp_x<T, R>, threads, smem));
    if (occ < 1) return fail(TSW_ERR_ARG, "implicit x solver does not fit on an SM");
    const int64_t want = (int64_t(occ) * c->sm_count + c->g.batch - 1) / c->g.batch;
    const unsigned gx = unsigned(std::max<int64_t>(1, std::min<int64_t>(ax.nrows, want)));
    k_imp_x<T, R><<<dim3(gx, unsigned(c->g.batch)), threads, smem, c->stream>>>(ax);
    CKL();
    return TSW_OK;
}

template <typename T>
tsw_status implicit_level_scan_t(tsw_ctx* c, bool start) {
    const int64_t nx = c->g.nx, ny = c->g.ny;
    const int m = int(nx - 2), my = int(ny - 2);
    if (!c->imp_fact_valid) {
        const size_t fsm = size_t(3 * m + 1) * sizeof(double);
        CK(cudaFuncSetAttribute(k_imp_xfactor<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fsm)));
        k_imp_xfactor<T><<<unsigned(c->g.batch), 256, fsm, c->stream>>>(
            static_cast<const T*>(c->c1), c->cstride1, static_cast<T*>(c->imp_tab), c->imp_tpitch, m, c->g.batch);
        CKL();
        c->launches++;
        c->imp_fact_valid = true;
    }
    ImpXArgs ax;
    ax.src = c->buf[c->ic];
    ax.dst = c->imp_s1;
    ax.tab = c->imp_tab;
    ax.pitch = c->pitch;
    ax.mstride = c->mstride;
    ax.tpitch = c->imp_tpitch;
    ax.nx = int32_t(nx);
    ax.row0 = 2;  // view row of global row 1
    ax.nrows = my;
    ax.scale = start ? 1.0 : 2.0;
    tsw_status st;
    constexpr int W = 32 / int(sizeof(T));  // one 32-byte access per thread
    if (nx <= 1024 * W) st = launch_imp_x<T, W>(c, ax);
    else st = launch_imp_x<T, 2 * W>(c, ax);
    if (st) return st;
    // solver 0 (auto): the streaming y solve for large fp64 grids (where the cluster kernel is
    // latency-bound), the cluster solve otherwise (measured)
    const int solver = (c->imp_solver == 0) ? ((is_f64(c) && int64_t(m) * my >= (int64_t(8) << 20)) ? 2 : 3)
                                            : c->imp_solver;
    if (solver == 2) {   // streaming y solve: three barrier-free kernels
        const int64_t ncolp = round_up(nx, 32);
        const int nseg = (my + IMPS_SEG - 1) / IMPS_SEG;
        if (!c->imp_ycol) {
            const size_t B = size_t(c->g.batch);
            CK(cudaMalloc(&c->imp_ycol, B * 4 * ncolp * sizeof(T)));
            CK(cudaMalloc(&c->imp_cF, B * nseg * ncolp * sizeof(T)));
            CK(cudaMalloc(&c->imp_cB, B * nseg * ncolp * sizeof(T)));
            CK(cudaMalloc(&c->imp_ccon, B * 2 * ncolp * sizeof(T)));
            c->imp_fact_valid = false;
        }
        if (!c->imp_fact_valid || c->imp_ycol_stale) {
            k_imp_ycol<T><<<dim3(unsigned((m + 255) / 256), unsigned(c->g.batch)), 256, 0, c->stream>>>(
                static_cast<const T*>(c->c2), c->cstride2, static_cast<T*>(c->imp_ycol), ncolp, int(nx), c->g.batch);
            CKL();
            c->launches++;
            c->imp_ycol_stale = false;
        }
        ImpSArgs as;
        as.z = c->imp_s1;
        as.prev = c->buf[c->ip];
        as.ycol = c->imp_ycol;
        as.cF = c->imp_cF;
        as.cB = c->imp_cB;
        as.ccon = c->imp_ccon;
        as.pitch = c->pitch;
        as.mstride = c->mstride;
        as.ncolp = ncolp;
        as.nx = int32_t(nx);
        as.m = my;
        as.nseg = nseg;
        as.dt = c->dt;
        const dim3 g2(unsigned((m + 31) / 32), unsigned((nseg + 7) / 8), unsigned(c->g.batch));
        k_imp_ysum<T><<<g2, dim3(32, 8), 0, c->stream>>>(as);
        CKL();
        const dim3 gs(unsigned((m + 31) / 32), unsigned(c->g.batch)), bs(32, IMPS_GROUPS);
        if (nseg <= 8 * IMPS_GROUPS) k_imp_yscan<T, 8><<<gs, bs, 0, c->stream>>>(as);
        else k_imp_yscan<T, 16><<<gs, bs, 0, c->stream>>>(as);
        CKL();
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (c->timing) {
            tsw_status st2 = timing_events(c, &e0, &e1);
            if (st2) return st2;
            CK(cudaEventRecord(e0, c->stream));
        }
        if (start) k_imp_yfin<T, 1><<<g2, dim3(32, 8), 0, c->stream>>>(as);
        else k_imp_yfin<T, 0><<<g2, dim3(32, 8), 0, c->stream>>>(as);
        CKL();
        if (c->timing) {
            CK(cudaEventRecord(e1, c->stream));
            note_timed(c, 1, int64_t(m) * my * c->g.batch);
        }
        c->launches += 4;
        std::swap(c->ic, c->ip);
        c->n++;
        return TSW_OK;
    }
    ImpYArgs ay;
    ay.z = c->imp_s1;
    ay.prev = c->buf[c->ip];
    ay.cf = c->c2;
    ay.pitch = c->pitch;
    ay.mstride = c->mstride;
    ay.cpitch = c->cstride2;
    ay.nx = int32_t(nx);
    ay.m = my;
    ay.dt = c->dt;
    {   // cluster-resident variant: a cluster of ≤ 8 CTAs holds the columns' full height on chip
        using G = ImpYc<T>;
        const int CL = (my + G::SEGS * G::SR - 1) / (G::SEGS * G::SR);
        if (CL <= 8) {
            const int segc = (my + CL * G::SEGS - 1) / (CL * G::SEGS);
            const size_t smc = G::smem_bytes(segc);
            ay.seg = segc;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(unsigned((m + G::COLS - 1) / G::COLS), unsigned(CL), unsigned(c->g.batch));
            cfg.blockDim = dim3(IMPYC_THREADS, 1, 1);
            cfg.dynamicSmemBytes = smc;
            cfg.stream = c->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 1;
            attr[0].val.clusterDim.y = unsigned(CL);
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (c->timing) {   // live timing of the dominant implicit kernel
                tsw_status st2 = timing_events(c, &e0, &e1);
                if (st2) return st2;
                CK(cudaEventRecord(e0, c->stream));
            }
            if (start) {
                CK(cudaFuncSetAttribute(k_imp_yc<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smc)));
                CK(cudaLaunchKernelEx(&cfg, k_imp_yc<T, 1>, ay));
            } else {
                CK(cudaFuncSetAttribute(k_imp_yc<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smc)));
                CK(cudaLaunchKernelEx(&cfg, k_imp_yc<T, 0>, ay));
            }
            CKL();
            if (c->timing) {
                CK(cudaEventRecord(e1, c->stream));
                note_timed(c, 1, int64_t(m) * my * c->g.batch);
            }
            c->launches += 2;
            std::swap(c->ic, c->ip);
            c->n++;
            return TSW_OK;
        }
    }
    ay.seg = int32_t(round_up((my + IMPY_SEGS - 1) / IMPY_SEGS, 8));
    const size_t smem = (2 * size_t(IMPY_SEGS) * IMPY_COLS + size_t(ay.seg / 8) * IMPY_THREADS) * sizeof(T);
    const dim3 gy(unsigned((m + IMPY_COLS - 1) / IMPY_COLS), unsigned(c->g.batch));
    if (start) {
        CK(cudaFuncSetAttribute(k_imp_y<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_imp_y<T, 1><<<gy, IMPY_THREADS, smem, c->stream>>>(ay);
    } else {
        CK(cudaFuncSetAttribute(k_imp_y<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_imp_y<T, 0><<<gy, IMPY_THREADS, smem, c->stream>>>(ay);
    }
    CKL();
    c->launches += 2;
    std::swap(c->ic, c->ip);
    c->n++;
    return TSW_OK;
}

template <typename T>
tsw_status implicit_level_t(tsw_ctx* c, bool start) {
    const T dtT = (T)c->dt;
    if (c->g.dim == 1) {
        T* cp = static_cast<T*>(c->imp_s1);
        T* dp = static_cast<T*>(c->imp_t);
        const int threads = 32;
        const unsigned blocks = unsigned((c->g.batch + threads - 1) / threads);
        if (start)
            k_implicit_1d<T, 1><<<blocks, threads, 0, c->stream>>>(static_cast<const T*>(c->buf[c->ic]), static_cast<T*>(c->buf[c->ip]),
                                                                 static_cast<const T*>(c->c1), c->g.nx, c->pitch, c->cstride1, cp, dp,
                                                                 c->g.batch, dtT);
        else
            k_implicit_1d<T, 0><<<blocks, threads, 0, c->stream>>>(static_cast<const T*>(c->buf[c->ic]), static_cast<T*>(c->buf[c->ip]),
                                                                 static_cast<const T*>(c->c1), c->g.nx, c->pitch, c->cstride1, cp, dp,
                                                                 c->g.batch, dtT);
        CKL();
        c->launches++;
        std::swap(c->ic, c->ip);
        c->n++;
        return TSW_OK;
    }
    const int64_t nx = c->g.nx, ny = c->g.ny;
    if (c->imp_solver != 1) return implicit_level_scan_t<T>(c, start);
    // (1) x lines: (I − ½L_x) z = scale·u  on the interior rows (view rows 2 .. ny−1)
    CrArgs ax;
    ax.src = c->buf[c->ic];
    ax.dst = c->imp_s1;
    ax.cf = c->c1;
    ax.pitch = c->pitch;
    ax.mstride = c->mstride;
    ax.cpitch = c->cstride1;
    ax.m = nx - 2;
    ax.q = cr_levels(ax.m);
    ax.row0 = 2;
    ax.nlines = int32_t(ny - 2);
    ax.line_coef0 = 0;
    ax.scale = start ? 1.0 : 2.0;
    const size_t smx = size_t(4) * ((size_t(1) << ax.q) - 1) * sizeof(T);
    CK(cudaFuncSetAttribute(k_cr_rows<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smx)));
    k_cr_rows<T, 0><<<dim3(unsigned(ax.nlines), unsigned(c->g.batch)), 512, smx, c->stream>>>(ax);
    CKL();
    // (2) transpose z
    const dim3 tb(32, 8);
    const dim3 tg(unsigned((nx + 31) / 32), unsigned((c->imp_pt + 31) / 32), unsigned(c->g.batch));
    const int64_t tstride = nx * c->imp_pt;
    k_transpose<T><<<tg, tb, 0, c->stream>>>(static_cast<const T*>(c->imp_s1), static_cast<T*>(c->imp_t), nx, ny,
                                             c->pitch, c->mstride, c->imp_pt, tstride);
    CKL();
    // (3) y lines (rows of the transpose = interior columns 1..nx−2): (I − ½L_y) w = z, c2 per column
    CrArgs ay;
    ay.src = static_cast<const T*>(c->imp_t) - 0;
    ay.dst = c->imp_t;
    ay.cf = c->c2;
    ay.pitch = c->imp_pt;
    ay.mstride = tstride;
    ay.cpitch = c->cstride2;
    ay.m = ny - 2;
    ay.q = cr_levels(ay.m);
    ay.row0 = 1;
    ay.nlines = int32_t(nx - 2);
    ay.line_coef0 = 1;
    ay.scale = 1.0;
    const size_t smy = size_t(4) * ((size_t(1) << ay.q) - 1) * sizeof(T);
    CK(cudaFuncSetAttribute(k_cr_rows<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smy)));
    k_cr_rows<T, 1><<<dim3(unsigned(ay.nlines), unsigned(c->g.batch)), 512, smy, c->stream>>>(ay);
    CKL();
    // (4) transpose back and finish the level in place over u^{n−1} (or u₁ at the start)
    const dim3 fg(unsigned((nx + 31) / 32), unsigned((ny + 31) / 32), unsigned(c->g.batch));
    if (start)
        k_transpose_finish<T, 1><<<fg, tb, 0, c->stream>>>(static_cast<const T*>(c->imp_t), static_cast<T*>(c->buf[c->ip]), nx, ny,
                                                           c->pitch, c->mstride, c->imp_pt, tstride, dtT);
    else
        k_transpose_finish<T, 0><<<fg, tb, 0, c->stream>>>(static_cast<const T*>(c->imp_t), static_cast<T*>(c->buf[c->ip]), nx, ny,
                                                           c->pitch, c->mstride, c->imp_pt, tstride, dtT);
    CKL();
    c->launches += 4;
    std::swap(c->ic, c->ip);
    c->n++;
    return TSW_OK;
}

tsw_status implicit_level(tsw_ctx* c) {
    if (c->mode != MODE_LINE)
        return fail(TSW_ERR_ARG, "the implicit scheme needs x-only coefficients (δ-line, constant or profile kinds)");
    return is_f64(c) ? implicit_level_t<double>(c, c->n == 0) : implicit_level_t<float>(c, c->n == 0);
}

// Resident CTAs per SM of the TMA stencil at the ctx's ring depth (cached; 0 on error).
template <typename T, int MODE, bool START>
tsw_status tma_occupancy(tsw_ctx* c, int* occ_out, size_t* smem_out) {
    const int depth = c->depth_opt;
    const size_t smem = size_t(depth) * (tma_slot_bytes<T, MODE>() + 2 * sizeof(uint64_t));
    int& ob = c->bulk_blocks_per_sm[MODE][START ? 1 : 0];
    int& key = c->bulk_occ_key[MODE][START ? 1 : 0];
    if (ob == 0 || key != depth) {
        CK(cudaFuncSetAttribute(k_step2d_tma<T, MODE, START>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaFuncSetAttribute(k_step2d_tma<T, MODE, START>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob, k_step2d_tma<T, MODE, START>, (TMA_NC + 1) * 32, smem));
        if (ob < 1) return fail(TSW_ERR_ARG, "TMA stencil does not fit on an SM (depth %d)", depth);
        key = depth;
    }
    *occ_out = ob;
    *smem_out = smem;
    return TSW_OK;
}

// ---- 2D stencil launch ---------------------------------------------------------------------
// Updates storage rows [s_lo, s_hi) of every member: reads buf[ic] (u^n) and buf[ip]
// (u^{n−1}), writes u^{n+1} in place into buf[ip].
template <typename T, int MODE, bool START>
tsw_status launch_step2d_t(tsw_ctx* c, int32_t s_lo, int32_t s_hi) {
    if (s_hi <= s_lo) return TSW_OK;
    const bool tma = (c->kernel_opt == 0);
    StepArgs<T> a;
    a.ucur = static_cast<const T*>(c->buf[c->ic]);
    a.uprev = static_cast<T*>(c->buf[c->ip]);
    a.c1 = static_cast<const T*>(c->c1);
    a.c2 = static_cast<const T*>(c->c2);
    a.pitch = c->pitch;
    a.mstride = c->mstride;
    a.cstride1 = c->cstride1;
    a.cstride2 = c->cstride2;
    a.nx = c->g.nx;
    a.s_lo = s_lo;
    a.s_hi = s_hi;
    a.dtT = (T)c->dt;
    // workers: TMA → CTAs (one 4 KB strip each); register kernel → warps (one 32·V strip each)
    int occ = 0, threads = 0;
    size_t smem = 0;
    int64_t workers_per_block = 1;
    if (tma) {
        tsw_status st = tma_occupancy<T, MODE, START>(c, &occ, &smem);
        if (st) return st;
        a.strips = (c->pitch + TmaGeom<T>::WC - 1) / TmaGeom<T>::WC;
        threads = (TMA_NC + 1) * 32;
    } else {
        int& o = c->step_blocks_per_sm[MODE][START ? 1 : 0];
        if (o == 0) {
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_step2d<T, MODE, START>, 256, 0));
            if (o < 1) o = 1;
        }
        occ = o;
        a.strips = c->pitch / (32 * Vec16<T>::N);
        threads = 256;
        workers_per_block = 8;
    }
    const int64_t G = int64_t(occ) * c->sm_count * workers_per_block;
    const int64_t rows = s_hi - s_lo;
    int R = c->rows_per_item_opt;
    if (R <= 0) R = choose_rows_per_item(rows, a.strips, c->g.batch, G);
    if (R > rows) R = int(rows);
    a.rows_per_item = R;
    a.chunks = int((rows + R - 1) / R);
    a.items = a.strips * a.chunks * c->g.batch;
    int64_t blocks = (a.items + workers_per_block - 1) / workers_per_block;
    blocks = std::min<int64_t>(blocks, int64_t(occ) * c->sm_count);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        tsw_status st = timing_events(c, &e0, &e1);
        if (st) return st;
        CK(cudaEventRecord(e0, c->stream));
    }
    if (tma)
        k_step2d_tma<T, MODE, START><<<unsigned(blocks), threads, smem, c->stream>>>(a, c->depth_opt);
    else
        k_step2d<T, MODE, START><<<unsigned(blocks), threads, 0, c->stream>>>(a);
    CKL();
    if (c->timing) {
        CK(cudaEventRecord(e1, c->stream));
        note_timed(c, 1, rows * (c->g.nx - 2) * c->g.batch);
    }
    c->launches++;
    return TSW_OK;
}

// neighbour on side 0 (rank − 1) / 1 (rank + 1); peer halos in use
bool has_nb(const tsw_ctx* c, int side) { return side == 0 ? c->g.rank > 0 : c->g.rank < c->g.nranks - 1; }
bool peer_mode(const tsw_ctx* c) { return c->g.nranks > 1 && c->g.dim == 2 && c->halo_mode == 1; }

// ---- temporally blocked pass: K levels, (buf[ic], buf[ip]) → (buf[fk], buf[fkm1]) -----------
template <typename T, int K, int NC>
tsw_status launch_tb_nc(tsw_ctx* c, int fk, int fkm1, int32_t s_lo, int32_t s_hi, int32_t s_lo2, int32_t s_hi2) {
    using G = TbGeom<T, K, NC>;
    const int depth = c->tb_depth ? c->tb_depth : (tb_minb<T, K, NC>() == 1 ? 8 : 4);
    const size_t smem = tb_smem_bytes<T, K, NC>(depth);
    const bool peer = peer_mode(c);
    int& occ = c->tb_occ[is_f64(c) ? 1 : 0][K][NC == 4 ? 0 : 1];
    if (occ == 0) {
        CK((tb_setup<T, K, NC, false>(smem, &occ)));
        int occ_en = 0;
        CK((tb_setup<T, K, NC, true>(smem, &occ_en)));
        occ = std::min(occ, occ_en);   // the fused-energy pass launches the same grid
        if (occ < 1) return fail(TSW_ERR_ARG, "temporally blocked stencil (K=%d) does not fit on an SM", K);
    }
    TbArgs<T> a;
    a.un = static_cast<const T*>(c->buf[c->ic]);
    a.unm1 = static_cast<const T*>(c->buf[c->ip]);
    a.out_k = static_cast<T*>(c->buf[fk]);
    a.out_km1 = static_cast<T*>(c->buf[fkm1]);
    a.c1 = static_cast<const T*>(c->c1);
    a.c2 = static_cast<const T*>(c->c2);
    a.pitch = c->pitch;
    a.mstride = c->mstride;
    a.cstride = c->cstride1;
    a.nx = c->g.nx;
    a.ny = c->g.ny;
    a.r0 = c->r0;
    a.s_lo = s_lo;
    a.s_hi = s_hi;
    // storage rows that hold data: the slab plus, towards a neighbour, its G ghost rows
    a.smin = (c->g.rank > 0) ? 1 - c->G : 1;
    a.smax = int32_t(c->ny_local) + ((c->g.rank < c->g.nranks - 1) ? c->G : 0);
    a.strips = (c->pitch + G::WO - 1) / G::WO;
    a.dtT = (T)c->dt;
    if (peer) {   // fused halo push: the first / last K owned rows also go to the neighbours
        if (has_nb(c, 0)) {
            a.pu_k = static_cast<T*>(c->peer_buf[0][fk]) + c->peer_ny[0] * c->pitch;
            a.pu_km1 = static_cast<T*>(c->peer_buf[0][fkm1]) + c->peer_ny[0] * c->pitch;
            a.pu_mstride = c->peer_mstride[0];
            a.push_top = K;
        }
        if (has_nb(c, 1)) {
            a.pd_k = static_cast<T*>(c->peer_buf[1][fk]) - c->ny_local * c->pitch;
            a.pd_km1 = static_cast<T*>(c->peer_buf[1][fkm1]) - c->ny_local * c->pitch;
            a.pd_mstride = c->peer_mstride[1];
            a.push_bot = int32_t(c->ny_local) - K + 1;
        }
    }
    const int64_t rows1 = s_hi - s_lo, rows2 = s_hi2 - s_lo2;
    const int64_t rows = rows1 + rows2;
    const int64_t Gw = int64_t(occ) * c->sm_count;
    int R = c->rows_per_item_opt;
    if (R <= 0) R = choose_rows_per_item(rows, a.strips, c->g.batch, Gw, 2.0 * K, 0.5, 4 * K);
    R = int(std::min<int64_t>(R, std::max(rows1, rows2)));
    a.rows_per_item = R;
    a.chunks1 = int((rows1 + R - 1) / R);
    a.s_lo2 = s_lo2;
    a.s_hi2 = s_hi2;
    a.chunks = a.chunks1 + int((rows2 + R - 1) / R);
    a.items = a.strips * a.chunks * c->g.batch;
    const int64_t blocks = std::min<int64_t>(a.items, Gw);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        tsw_status st = timing_events(c, &e0, &e1);
        if (st) return st;
        CK(cudaEventRecord(e0, c->stream));
    }
    // the peer-store variant only where this launch's output rows include pushed rows (the
    // interior launch of a split pass has none and runs the plain kernel, which needs fewer
    // registers: the K = 8 fp64 peer variant spills)
    const bool top = s_lo <= a.push_top || (rows2 > 0 && s_lo2 <= a.push_top);
    const bool bot = s_hi - 1 >= a.push_bot || (rows2 > 0 && s_hi2 - 1 >= a.push_bot);
    const bool push = peer && ((has_nb(c, 0) && top) || (has_nb(c, 1) && bot));
    // fused energy: every launch of the pass writes its item partials as one segment of d_en
    const bool energy = c->en_now;
    if (energy) {
        if (c->en_nseg >= 2) return fail(TSW_ERR_STATE, "fused energy: more than two launches in a pass");
        const int64_t off = c->en_nseg ? c->en_off[0] + c->en_pm[0] * c->g.batch : 0;
        const size_t need = size_t(off + a.items);
        if (need > c->en_cap) {   // grow, keeping the first segment (stream-ordered copy)
            double* fresh = nullptr;
            CK(cudaMalloc(&fresh, need * sizeof(double)));
            if (off > 0) CK(cudaMemcpyAsync(fresh, c->d_en, size_t(off) * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
            CSYNC(c);
            if (c->d_en) CK(cudaFree(c->d_en));
            c->d_en = fresh;
            c->en_cap = need;
        }
        a.en_part = c->d_en + off;
        c->en_off[c->en_nseg] = off;
        c->en_pm[c->en_nseg] = a.strips * a.chunks;
        c->en_nseg++;
    }
    if (energy)
        CK((tb_launch<T, K, NC, true>(push, unsigned(blocks), smem, c->stream, a, depth)));
    else
        CK((tb_launch<T, K, NC, false>(push, unsigned(blocks), smem, c->stream, a, depth)));
    if (c->timing) {
        CK(cudaEventRecord(e1, c->stream));
        note_timed(c, K, rows * (c->g.nx - 2) * c->g.batch * K);
    }
    c->launches++;
    return TSW_OK;
}

// CTA width: the wide CTA (8 warps, 512-column strips; fp64 passes of depth ≥ 7: 12 warps,
// 768-column strips, one CTA per SM — tb_wide_nc) or 4 (256-column strips).  Auto (TSW_OPT_TB_WARPS = 0):
// 4 warps only where its strips compute ≥ 5 % fewer columns (narrow grids, e.g. config 5's 2048:
// +12 % fp64, +17 % fp32 measured; at 4096 columns 8 warps are as fast or faster)
template <typename T, int K>
tsw_status launch_tb_t(tsw_ctx* c, int fk, int fkm1, int32_t s_lo, int32_t s_hi, int32_t s_lo2, int32_t s_hi2) {
    if (s_hi2 <= s_lo2) s_lo2 = s_hi2 = 0;
    if (s_hi <= s_lo) {  // the second range alone
        s_lo = s_lo2;
        s_hi = s_hi2;
        s_lo2 = s_hi2 = 0;
    }
    if (s_hi <= s_lo) return TSW_OK;
    int nc = c->tb_warps;
    if (!nc && (s_hi - s_lo) + (s_hi2 - s_lo2) <= 2 * K) {
        nc = 4;  // a slab's boundary rows: few rows, so twice the CTAs (256-column strips)
    } else if (!nc) {
        constexpr int W = tb_wide_nc<T, K>();
        const int64_t cols8 = (c->pitch + TbGeom<T, K, W>::WO - 1) / TbGeom<T, K, W>::WO * TbGeom<T, K, W>::WE;
        const int64_t cols4 = (c->pitch + TbGeom<T, K, 4>::WO - 1) / TbGeom<T, K, 4>::WO * TbGeom<T, K, 4>::WE;
        nc = (double(cols4) < 0.95 * double(cols8)) ? 4 : 8;
    }
    return nc == 4 ? launch_tb_nc<T, K, 4>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2)
                   : launch_tb_nc<T, K, tb_wide_nc<T, K>()>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
}

template <typename T>
tsw_status launch_tb_k(tsw_ctx* c, int K, int fk, int fkm1, int32_t s_lo, int32_t s_hi, int32_t s_lo2, int32_t s_hi2) {
    switch (K) {
        case 2: return launch_tb_t<T, 2>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 3: return launch_tb_t<T, 3>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 4: return launch_tb_t<T, 4>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 5: return launch_tb_t<T, 5>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 6: return launch_tb_t<T, 6>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 7: return launch_tb_t<T, 7>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 8: return launch_tb_t<T, 8>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 9: return launch_tb_t<T, 9>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        case 10: return launch_tb_t<T, 10>(c, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
        default: return fail(TSW_ERR_ARG, "unsupported temporal blocking depth %d", K);
    }
}

tsw_status exchange_nccl(tsw_ctx* c, void* field, cudaStream_t stream, int nrows);

// ---- peer halos --------------------------------------------------------------------------------
// Epochs: every halo operation (a pass, a level, an initial exchange, a ghost-reading diagnostic) is
// issued by every rank in the same order and numbered e = 1, 2, … .  Before operation e a rank's
// stream waits until each neighbour has published e − 1 (its writes into my ghost rows are done and
// it no longer reads the ghost rows I am about to overwrite); afterwards it publishes e.
bool peers_ready(const tsw_ctx* c) {
    if (!c->mbox) return false;
    for (int side = 0; side < 2; ++side)
        if (has_nb(c, side) && (!c->peer_buf[side][0] || !c->peer_buf[side][1] || !c->peer_slot[side])) return false;
    return true;
}


tsw_status peer_begin(tsw_ctx* c, cudaStream_t s) {
    if (!peers_ready(c)) return fail(TSW_ERR_STATE, "peer halos: neighbours not attached (tsw_peer_import / tsw_peer_attach)");
    ++c->epoch;
    // mailbox layout: [0] from rank − 1, [1] from rank + 1, [2] wait-timeout error word
    k_peer_wait<<<1, 32, 0, s>>>(c->mbox, has_nb(c, 0) ? 1 : 0, has_nb(c, 1) ? 1 : 0, c->epoch - 1, c->mbox + 2);
    CKL();
    c->launches++;
    return TSW_OK;
}

tsw_status peer_end(tsw_ctx* c, cudaStream_t s) {
    k_peer_signal<<<1, 32, 0, s>>>(has_nb(c, 0) ? c->peer_slot[0] : nullptr, has_nb(c, 1) ? c->peer_slot[1] : nullptr,
                                   c->epoch);
    CKL();
    c->launches++;
    return TSW_OK;
}

// Copy nrows boundary rows of buffer bi into the neighbours' ghost rows (peer stores).
template <typename T>
tsw_status push_rows_t(tsw_ctx* c, int bi, int nrows, cudaStream_t s) {
    PushArgs<T> a;
    a.src = static_cast<const T*>(c->buf[bi]);
    a.pu = has_nb(c, 0) ? static_cast<T*>(c->peer_buf[0][bi]) + c->peer_ny[0] * c->pitch : nullptr;
    a.pd = has_nb(c, 1) ? static_cast<T*>(c->peer_buf[1][bi]) - c->ny_local * c->pitch : nullptr;
    if ((has_nb(c, 0) && !c->peer_buf[0][bi]) || (has_nb(c, 1) && !c->peer_buf[1][bi]))
        return fail(TSW_ERR_STATE, "peer halos: the neighbour has no buffer %d", bi);
    a.pitch = c->pitch;
    a.mstride = c->mstride;
    a.pu_mstride = c->peer_mstride[0];
    a.pd_mstride = c->peer_mstride[1];
    a.nx = c->g.nx;
    a.ny_local = c->ny_local;
    a.nrows = nrows;
    a.batch = c->g.batch;
    const int64_t total = int64_t(nrows) * c->g.nx * 2 * c->g.batch;
    k_push_rows<T><<<unsigned(grid_for(total, 256, 2 * c->sm_count)), 256, 0, s>>>(a);
    CKL();
    c->launches++;
    return TSW_OK;
}
// The waiter's timeout word (mailbox slot 2); call after the ctx stream has been synchronised.
tsw_status peer_check(tsw_ctx* c) {
    if (!peer_mode(c) || !c->mbox) return TSW_OK;
    unsigned int e = 0;
    CK(cudaMemcpyAsync(&e, c->mbox + 2, sizeof(e), cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    if (e) return fail(TSW_ERR_STATE, "peer halos: a wait for a neighbour timed out (epochs out of step)");
    return TSW_OK;
}

tsw_status push_rows(tsw_ctx* c, int bi, int nrows, cudaStream_t s) {
    return is_f64(c) ? push_rows_t<double>(c, bi, nrows, s) : push_rows_t<float>(c, bi, nrows, s);
}

void free_pair(const tsw_ctx* c, int* fk, int* fkm1) {
    int ids[2], nf = 0;
    for (int k = 0; k < 4 && nf < 2; ++k)
        if (k != c->ic && k != c->ip) ids[nf++] = k;
    *fk = ids[0];
    *fkm1 = ids[1];
}

// output rows [s_lo, s_hi) and, optionally, [s_lo2, s_hi2) in one launch
tsw_status launch_tb_rows(tsw_ctx* c, int fk, int fkm1, int32_t s_lo, int32_t s_hi, int32_t s_lo2 = 0,
                          int32_t s_hi2 = 0) {
    return is_f64(c) ? launch_tb_k<double>(c, c->tblock, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2)
                     : launch_tb_k<float>(c, c->tblock, fk, fkm1, s_lo, s_hi, s_lo2, s_hi2);
}

// Output rows of a slab pass that neighbours need: the first / last K owned rows.
struct TbSplit {
    int32_t top_lo = 0, top_hi = 0, bot_lo = 0, bot_hi = 0, ilo = 0, ihi = 0;
    bool split = false;
};
TbSplit tb_split(const tsw_ctx* c) {
    TbSplit p;
    const int K = c->tblock;
    p.ilo = c->s_lo;
    p.ihi = c->s_hi;
    if (c->g.nranks == 1 || c->ny_local < 3 * K) return p;  // single rank / tiny slab: one launch
    p.split = true;
    if (c->g.rank > 0) {
        p.top_lo = c->s_lo;
        p.top_hi = c->s_lo + K;
        p.ilo = p.top_hi;
    }
    if (c->g.rank < c->g.nranks - 1) {
        p.bot_lo = c->s_hi - K;
        p.bot_hi = c->s_hi;
        p.ihi = p.bot_lo;
    }
    return p;
}

// Fused energy of a pass (TSW_OPT_ENERGY_FUSE): the launches of the pass wrote their item partials
// as segments of d_en; one fixed-order sum per member gives this slab's E (node form, R30).
tsw_status en_pass_finish(tsw_ctx* c) {
    if (!c->en_now || c->en_nseg == 0) return TSW_OK;
    if (!c->en_result) CK(cudaMalloc(&c->en_result, sizeof(double) * size_t(c->g.batch)));
    const double w = c->g.dx * c->g.dy / (c->dt * c->dt);
    k_tb_energy_final<<<unsigned(c->g.batch), 32, 0, c->stream>>>(c->d_en, c->en_nseg, c->en_off[0], c->en_pm[0],
                                                                   c->en_off[1], c->en_pm[1], w, c->en_result);
    CKL();
    c->launches++;
    c->en_level = c->n;   // called after the level advanced
    return TSW_OK;
}

// A pass of K levels in two phases around the halo exchange (S4): begin launches the
// rows the neighbours need first — a slab's first / last K owned rows when the slab has ≥ 3K rows
// (tb_split), else all rows — and records ev_bnd; the caller exchanges K boundary rows of both new
// levels after ev_bnd (NCCL messages on the aux stream, loopback copies for a group of slabs in one
// process, nothing for peer halos: the kernel pushed them); end launches the interior rows, makes
// the ctx stream wait for the exchange's event (if any) and advances to u^n = buf[fk],
// u^{n−1} = buf[fkm1].  Single rank: begin launches everything, end only advances.
struct TbPassState {
    int fk = 0, fkm1 = 0;
    TbSplit p;
};
tsw_status tb_pass_begin(tsw_ctx* c, TbPassState& ps) {
    free_pair(c, &ps.fk, &ps.fkm1);
    ps.p = tb_split(c);
    c->en_nseg = 0;
    tsw_status st;
    if (ps.p.split)
        st = launch_tb_rows(c, ps.fk, ps.fkm1, ps.p.top_lo, ps.p.top_hi, ps.p.bot_lo, ps.p.bot_hi);
    else
        st = launch_tb_rows(c, ps.fk, ps.fkm1, c->s_lo, c->s_hi);
    if (st) return st;
    if (c->g.nranks > 1) CK(cudaEventRecord(c->ev_bnd, c->stream));
    return TSW_OK;
}
tsw_status tb_pass_end(tsw_ctx* c, const TbPassState& ps, cudaEvent_t comm_done) {
    tsw_status st;
    if (ps.p.split && (st = launch_tb_rows(c, ps.fk, ps.fkm1, ps.p.ilo, ps.p.ihi))) return st;
    if (comm_done) CK(cudaStreamWaitEvent(c->stream, comm_done, 0));
    const int K = c->tblock;
    if (c->g.nranks > 1) c->gdepth[ps.fk] = c->gdepth[ps.fkm1] = K;
    c->ic = ps.fk;
    c->ip = ps.fkm1;
    c->n += K;
    return en_pass_finish(c);
}

// One pass of K levels of one rank: single rank; peer halos (the kernel stores the boundary rows
// into the neighbours' ghost rows; with a split pass the epoch is published after the first / last
// K rows, before the interior, which reads no ghost rows — so the neighbours' next pass may start
// while the interior still runs); NCCL (the K-row exchange of both levels on the aux stream,
// concurrently with the interior rows: SURVEY §8(f) NEXT 4, one exchange per K levels).
tsw_status tb_pass(tsw_ctx* c) {
    TbPassState ps;
    tsw_status st;
    if (c->g.nranks == 1) {
        if ((st = tb_pass_begin(c, ps))) return st;
        return tb_pass_end(c, ps, nullptr);
    }
    if (peer_mode(c)) {
        if ((st = peer_begin(c, c->stream))) return st;
        if ((st = tb_pass_begin(c, ps))) return st;
        if ((st = peer_end(c, c->stream))) return st;
        return tb_pass_end(c, ps, nullptr);
    }
    if ((st = tb_pass_begin(c, ps))) return st;
    CK(cudaStreamWaitEvent(c->aux, c->ev_bnd, 0));
    if ((st = exchange_nccl(c, c->buf[ps.fk], c->aux, c->tblock))) return st;
    if ((st = exchange_nccl(c, c->buf[ps.fkm1], c->aux, c->tblock))) return st;
    CK(cudaEventRecord(c->ev_comm, c->aux));
    return tb_pass_end(c, ps, c->ev_comm);
}

tsw_status launch_step2d(tsw_ctx* c, bool start, int32_t s_lo, int32_t s_hi) {
    if (is_f64(c)) {
        if (c->mode == MODE_LINE)
            return start ? launch_step2d_t<double, MODE_LINE, true>(c, s_lo, s_hi)
                         : launch_step2d_t<double, MODE_LINE, false>(c, s_lo, s_hi);
        return start ? launch_step2d_t<double, MODE_DENSE, true>(c, s_lo, s_hi)
                     : launch_step2d_t<double, MODE_DENSE, false>(c, s_lo, s_hi);
    }
    if (c->mode == MODE_LINE)
        return start ? launch_step2d_t<float, MODE_LINE, true>(c, s_lo, s_hi)
                     : launch_step2d_t<float, MODE_LINE, false>(c, s_lo, s_hi);
    return start ? launch_step2d_t<float, MODE_DENSE, true>(c, s_lo, s_hi)
                 : launch_step2d_t<float, MODE_DENSE, false>(c, s_lo, s_hi);
}

// ---- 1D ---------------------------------------------------------------------------------------
template <typename T>
tsw_status step1d_t(tsw_ctx* c, int64_t k) {
    const bool start = (c->n == 0);
    const size_t smem = size_t(3) * c->pitch * sizeof(T);
    T* u = static_cast<T*>(c->buf[c->ic]);
    T* p = static_cast<T*>(c->buf[c->ip]);
    const T* c1 = static_cast<const T*>(c->c1);
    if (smem <= 200 * 1024) {
        if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k_step1d_smem<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int threads = int(std::min<int64_t>(1024, round_up(c->g.nx, 32)));
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (c->timing) {
            tsw_status st = timing_events(c, &e0, &e1);
            if (st) return st;
            CK(cudaEventRecord(e0, c->stream));
        }
        k_step1d_smem<T><<<c->g.batch, threads, smem, c->stream>>>(u, p, c1, c->g.nx, c->pitch, c->cstride1, k,
                                                                   start ? 1 : 0, (T)c->dt);
        CKL();
        if (c->timing) {
            CK(cudaEventRecord(e1, c->stream));
            note_timed(c, int32_t(k), k * (c->g.nx - 2) * c->g.batch);
        }
        c->launches++;
        c->n += k;  // the kernel writes the newest level back into buf[ic]
        return TSW_OK;
    }
    const dim3 grid(unsigned(grid_for(c->g.nx, 256, 4 * c->sm_count)), unsigned(c->g.batch));
    for (int64_t s = 0; s < k; ++s) {
        const T* uc = static_cast<const T*>(c->buf[c->ic]);
        T* up = static_cast<T*>(c->buf[c->ip]);
        if (c->n == 0)
            k_step1d_global<T, true><<<grid, 256, 0, c->stream>>>(uc, up, c1, c->g.nx, c->pitch, c->cstride1, (T)c->dt);
        else
            k_step1d_global<T, false><<<grid, 256, 0, c->stream>>>(uc, up, c1, c->g.nx, c->pitch, c->cstride1, (T)c->dt);
        CKL();
        c->launches++;
        std::swap(c->ic, c->ip);
        c->n++;
    }
    return TSW_OK;
}

// ---- ghost rows -------------------------------------------------------------------------------
// NCCL: send my first owned row up to rank−1 and my last owned row down to rank+1; receive their
// rows into my ghost rows (storage rows 0 and ny_local+1).  Rows are contiguous: no packing.
tsw_status exchange_nccl(tsw_ctx* c, void* field, cudaStream_t stream, int nrows) {
    if (!stream) stream = c->stream;
    if (c->g.nranks <= 1) return TSW_OK;
    if (!c->comm) return fail(TSW_ERR_STATE, "nranks > 1 but tsw_nccl_init was not called");
    Nccl& N = nccl();
    const int dt = is_f64(c) ? NCCL_F64 : NCCL_F32;
    // nrows owned rows [1, nrows] go up and [ny_local − nrows + 1, ny_local] go down; the ghost rows
    // [1 − nrows, 0] and [ny_local + 1, ny_local + nrows] receive (contiguous: one message each)
    char* base = static_cast<char*>(field);
    const size_t row = size_t(c->pitch) * c->esz;
    const size_t cnt = (nrows == 1) ? size_t(c->g.nx) : size_t(nrows) * size_t(c->pitch);
    const int64_t up_send = 1, up_recv = 1 - nrows, dn_send = c->ny_local - nrows + 1, dn_recv = c->ny_local + 1;
    NK(N.GroupStart());
    for (int b = 0; b < c->g.batch; ++b) {
        char* m = base + size_t(b) * c->mstride * c->esz;
        if (c->g.rank > 0) {
            NK(N.Send(m + up_send * int64_t(row), cnt, dt, c->g.rank - 1, c->comm, stream));
            NK(N.Recv(m + up_recv * int64_t(row), cnt, dt, c->g.rank - 1, c->comm, stream));
        }
        if (c->g.rank < c->g.nranks - 1) {
            NK(N.Send(m + dn_send * int64_t(row), cnt, dt, c->g.rank + 1, c->comm, stream));
            NK(N.Recv(m + dn_recv * int64_t(row), cnt, dt, c->g.rank + 1, c->comm, stream));
        }
    }
    NK(N.GroupEnd());
    return TSW_OK;
}

// Loopback: ranks are ctxs on one device and stream; copy rows device-to-device.  bi = buffer
// index (the same in every member of a lock-stepped group); nrows rows per direction.
tsw_status exchange_loopback_buf(tsw_ctx** cs, int n, int bi, cudaStream_t stream, int nrows) {
    for (int r = 0; r + 1 < n; ++r) {
        tsw_ctx* a = cs[r];      // upper slab (smaller rows)
        tsw_ctx* b = cs[r + 1];  // lower slab
        const int64_t row = int64_t(a->pitch) * int64_t(a->esz);
        const size_t bytes = (nrows == 1) ? size_t(a->g.nx) * a->esz : size_t(nrows) * size_t(row);
        for (int m = 0; m < a->g.batch; ++m) {
            char* ma = static_cast<char*>(a->buf[bi]) + size_t(m) * a->mstride * a->esz;
            char* mb = static_cast<char*>(b->buf[bi]) + size_t(m) * b->mstride * b->esz;
            // a's last nrows owned rows → b's upper ghost rows; b's first nrows → a's lower ghost rows
            CK(cudaMemcpyAsync(mb + (1 - nrows) * row, ma + (a->ny_local - nrows + 1) * row, bytes,
                               cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemcpyAsync(ma + (a->ny_local + 1) * row, mb + 1 * row, bytes, cudaMemcpyDeviceToDevice, stream));
        }
    }
    return TSW_OK;
}

// level 0 = u^n (buf[ic]), 1 = u^{n−1} (buf[ip]).
tsw_status exchange_loopback(tsw_ctx** cs, int n, int level = 0, cudaStream_t stream = nullptr, int nrows = 1) {
    if (!stream) stream = cs[0]->stream;
    return exchange_loopback_buf(cs, n, level ? cs[0]->ip : cs[0]->ic, stream, nrows);
}

tsw_status prescale_all(tsw_ctx* c) {
    const int threads = 256;
    const int64_t n1 = c->cstride1 * c->g.batch;
    const int64_t n2 = c->cstride2 * c->g.batch;
    const int cap = 8 * c->sm_count;
    if (is_f64(c)) {
        k_prescale<double><<<grid_for(n1, threads, cap), threads, 0, c->stream>>>(c->h1, static_cast<double*>(c->c1), n1, c->dt, c->g.dx);
        CKL();
        if (c->g.dim == 2) {
            k_prescale<double><<<grid_for(n2, threads, cap), threads, 0, c->stream>>>(c->h2, static_cast<double*>(c->c2), n2, c->dt, c->g.dy);
            CKL();
        }
    } else {
        k_prescale<float><<<grid_for(n1, threads, cap), threads, 0, c->stream>>>(c->h1, static_cast<float*>(c->c1), n1, c->dt, c->g.dx);
        CKL();
        if (c->g.dim == 2) {
            k_prescale<float><<<grid_for(n2, threads, cap), threads, 0, c->stream>>>(c->h2, static_cast<float*>(c->c2), n2, c->dt, c->g.dy);
            CKL();
        }
    }
    c->launches += (c->g.dim == 2) ? 2 : 1;
    c->imp_fact_valid = false;
    c->imp_ycol_stale = true;
    return TSW_OK;
}

tsw_status alloc_coeff(tsw_ctx* c, int mode) {
    if (c->have_coeff && c->mode == mode) return TSW_OK;
    CSYNC(c);  // queued work may still read the old arrays
    dfree_guarded(c->h1, c->cshift_h);
    dfree_guarded(c->h2, c->cshift_h);
    dfree_guarded(c->c1, c->cshift);
    dfree_guarded(c->c2, c->cshift);
    c->h1 = c->h2 = nullptr;
    c->c1 = c->c2 = nullptr;
    c->have_coeff = false;
    c->mode = mode;
    if (mode == MODE_LINE) {  // row-invariant coefficients: c1 per x face, c2 per node column
        c->cstride1 = c->pitch;
        c->cstride2 = c->pitch;
    } else {
        c->cstride1 = c->mstride;
        c->cstride2 = c->mstride;
    }
    const size_t B = size_t(c->g.batch);
    // DENSE arrays are row-structured like the fields: same ghost-row view shift
    const size_t rows_shift = (mode == MODE_DENSE) ? size_t(c->G - 1) * size_t(c->pitch) : 0;
    c->cshift_h = rows_shift * sizeof(double);
    c->cshift = rows_shift * c->esz;
    CK(dmalloc_guarded(reinterpret_cast<void**>(&c->h1), B * c->cstride1 * sizeof(double), c->cshift_h, c->stream));
    CK(dmalloc_guarded(reinterpret_cast<void**>(&c->h2), B * c->cstride2 * sizeof(double), c->cshift_h, c->stream));
    CK(dmalloc_guarded(&c->c1, B * c->cstride1 * c->esz, c->cshift, c->stream));
    CK(dmalloc_guarded(&c->c2, B * c->cstride2 * c->esz, c->cshift, c->stream));
    return TSW_OK;
}

// Gershgorin bound and positivity of the current faces; all-reduced over ranks.
tsw_status check_faces(tsw_ctx* c) {
    CK(cudaMemsetAsync(c->d_u64, 0, 2 * sizeof(unsigned long long), c->stream));
    CflArgs a;
    a.dim = c->g.dim;
    a.mode = c->mode;
    a.h1 = c->h1;
    a.h2 = c->h2;
    a.nx = c->g.nx;
    a.pitch = c->pitch;
    a.cpitch = c->cstride1;
    a.rows_alloc = c->rows_alloc;
    a.s_lo = c->s_lo;
    a.s_hi = c->s_hi;
    a.dx = c->g.dx;
    a.dy = c->g.dy;
    a.B = c->g.batch;
    const int64_t rows = (c->g.dim == 1) ? 1 : (c->s_hi - c->s_lo);
    dim3 grid(unsigned(grid_for(rows * (c->g.nx - 2), 256, 2 * c->sm_count)), 1, unsigned(c->g.batch));
    if (rows > 0) {
        k_cfl<<<grid, 256, 0, c->stream>>>(a, c->d_u64);
        CKL();
        c->launches++;
    }
    unsigned long long rho_bits = 0;
    CK(cudaMemcpyAsync(&rho_bits, c->d_u64, sizeof(rho_bits), cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    double rho;
    memcpy(&rho, &rho_bits, sizeof(rho));
    if (c->g.nranks > 1 && c->comm) {
        double* d = reinterpret_cast<double*>(c->d_u64);
        CK(cudaMemcpyAsync(d, &rho, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        NK(nccl().AllReduce(d, d, 1, NCCL_F64, NCCL_MAX, c->comm, c->stream));
        CK(cudaMemcpyAsync(&rho, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CSYNC(c);
    }
    if (!(rho > 0.0) || !std::isfinite(rho)) return fail(TSW_ERR_ARG, "non-finite or zero Gershgorin radius (%g)", rho);
    c->dt_max = 2.0 / std::sqrt(rho);
    return TSW_OK;
}

tsw_status load_field(tsw_ctx* c, void* dst_buf, const void* src, bool shared, int on_device) {
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const size_t w = size_t(c->g.nx) * c->esz;
    const size_t rows = size_t(c->ny_local);
    for (int b = 0; b < c->g.batch; ++b) {
        const char* s = static_cast<const char*>(src) + (shared ? 0 : size_t(b) * rows * w);
        char* d = static_cast<char*>(dst_buf) + size_t(b) * c->mstride * c->esz +
                  (c->g.dim == 2 ? size_t(c->pitch) * c->esz : 0);
        CK(cudaMemcpy2DAsync(d, size_t(c->pitch) * c->esz, s, w, w, rows, kind, c->stream));
    }
    return TSW_OK;
}

tsw_status zero_boundary(tsw_ctx* c, void* field) {
    const int64_t rows = (c->g.dim == 1) ? 1 : c->ny_local;
    dim3 grid(unsigned(grid_for(rows * c->pitch, 256, 4 * c->sm_count)), unsigned(c->g.batch));
    if (is_f64(c))
        k_zero_boundary<double><<<grid, 256, 0, c->stream>>>(static_cast<double*>(field), c->g.dim, c->g.nx, c->g.ny,
                                                             c->r0, c->ny_local, c->pitch, c->mstride);
    else
        k_zero_boundary<float><<<grid, 256, 0, c->stream>>>(static_cast<float*>(field), c->g.dim, c->g.nx, c->g.ny,
                                                            c->r0, c->ny_local, c->pitch, c->mstride);
    CKL();
    c->launches++;
    return TSW_OK;
}

tsw_status set_levels(tsw_ctx* c, const void* a, const void* b, double dt, int on_device, uint32_t flags,
                      int64_t n) {
    if (!c->have_coeff) return fail(TSW_ERR_STATE, "set coefficients (tsw_set_coeff / tsw_set_coeff_faces) first");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(TSW_ERR_ARG, "dt must be finite and > 0 (got %g)", dt);
    if (!a) return fail(TSW_ERR_ARG, "u0 / un is NULL");
    if (!(flags & TSW_ALLOW_UNSTABLE) && c->scheme == 0 && !(dt <= c->dt_max))
        return fail(TSW_ERR_CFL, "dt = %.17g exceeds the Gershgorin leapfrog bound 2/sqrt(rho_G) = %.17g (R16)", dt,
                    c->dt_max);
    const bool shared = (flags & TSW_INIT_SHARED) != 0;
    const size_t bytes = size_t(c->g.batch) * c->mstride * c->esz;
    drop_graphs(c);  // captured launches bake in dt
    c->ic = 0;
    c->ip = 1;
    tsw_status st;
    // peer halos: the buffers are re-initialised inside an epoch of their own, so no neighbour
    // pushes into them meanwhile; the ghost push below waits for the neighbours' initialisation
    if (peer_mode(c) && (st = peer_begin(c, c->stream))) return st;
    for (int k = 0; k < 4; ++k)
        if (c->buf[k]) CK(cudaMemsetAsync(static_cast<char*>(c->buf[k]) - c->fshift, 0, bytes, c->stream));
    st = load_field(c, c->buf[0], a, shared, on_device);
    if (st) return st;
    if (b) {
        st = load_field(c, c->buf[1], b, shared, on_device);
        if (st) return st;
    }
    if ((st = zero_boundary(c, c->buf[0]))) return st;
    if ((st = zero_boundary(c, c->buf[1]))) return st;
    c->dt = dt;
    if ((st = prescale_all(c))) return st;
    c->ghosts_valid = false;
    for (int& d : c->gdepth) d = 0;
    if (peer_mode(c)) {
        // this slab's buffers are initialised; the neighbours' rows are pushed by the first
        // operation that reads ghost rows (one epoch per call: see tsw_group_step)
        if ((st = peer_end(c, c->stream))) return st;
    } else if (c->g.dim == 2 && c->g.nranks > 1 && c->comm) {
        // ghost rows of both levels (the energy of (u^n, u^{n−1}) reads both; loopback groups
        // exchange in tsw_group_step instead)
        if ((st = exchange_nccl(c, c->buf[0], c->stream, c->G))) return st;
        if ((st = exchange_nccl(c, c->buf[1], c->stream, c->G))) return st;
        c->gdepth[0] = c->gdepth[1] = c->G;
        c->ghosts_valid = true;
    }
    c->n = n;
    c->en_level = -1;
    c->en_ref.clear();
    c->have_init = true;
    return TSW_OK;
}

// Rows of a slab step: the boundary rows other ranks need (first owned row if rank > 0, last
// owned row if rank < P−1) and the interior rest of [s_lo, s_hi).
struct SlabSplit {
    int32_t top = -1, bot = -1, ilo = 0, ihi = 0;
};
SlabSplit slab_split(const tsw_ctx* c) {
    SlabSplit p;
    p.ilo = c->s_lo;
    p.ihi = c->s_hi;
    if (c->g.rank > 0) {
        p.top = 1;  // == s_lo
        p.ilo = 2;
    }
    if (c->g.rank < c->g.nranks - 1) {
        p.bot = int32_t(c->ny_local);  // == s_hi − 1
        p.ihi = int32_t(c->ny_local);
        if (p.bot == p.top) p.bot = -1;
    }
    if (p.ihi < p.ilo) p.ihi = p.ilo;
    return p;
}

tsw_status launch_boundary_rows(tsw_ctx* c, bool start) {
    const SlabSplit p = slab_split(c);
    tsw_status st;
    if (p.top >= 0 && (st = launch_step2d(c, start, p.top, p.top + 1))) return st;
    if (p.bot >= 0 && (st = launch_step2d(c, start, p.bot, p.bot + 1))) return st;
    return TSW_OK;
}

tsw_status launch_interior_rows(tsw_ctx* c, bool start) {
    const SlabSplit p = slab_split(c);
    return launch_step2d(c, start, p.ilo, p.ihi);
}

// One slab level with overlap: boundary rows on the ctx stream, then the NCCL
// ghost-row exchange of the new level on the aux stream, concurrently with the interior rows;
// the ctx stream waits for the exchange before the next level reads the ghost rows.
// One level of a slab in two phases around the exchange of its new boundary rows (S4): begin
// launches the first / last owned rows the neighbours need and records ev_bnd; end launches the
// interior rows, waits for the exchange's event and advances the level (the new level overwrote
// u^{n−1} in place: buf[ip]).  step_slab_overlapped (NCCL, one rank per process) and
// tsw_group_step (loopback copies, P slabs of one process) run the same phases.
tsw_status slab_level_begin(tsw_ctx* c, bool start) {
    tsw_status st = launch_boundary_rows(c, start);
    if (st) return st;
    CK(cudaEventRecord(c->ev_bnd, c->stream));
    return TSW_OK;
}
tsw_status slab_level_end(tsw_ctx* c, bool start, cudaEvent_t comm_done) {
    tsw_status st = launch_interior_rows(c, start);
    if (st) return st;
    if (comm_done) CK(cudaStreamWaitEvent(c->stream, comm_done, 0));
    std::swap(c->ic, c->ip);
    c->gdepth[c->ic] = 1;
    c->n++;
    return TSW_OK;
}
tsw_status step_slab_overlapped(tsw_ctx* c) {
    const bool start = (c->n == 0);
    tsw_status st;
    if ((st = slab_level_begin(c, start))) return st;
    CK(cudaStreamWaitEvent(c->aux, c->ev_bnd, 0));
    if ((st = exchange_nccl(c, c->buf[c->ip], c->aux, 1))) return st;
    CK(cudaEventRecord(c->ev_comm, c->aux));
    return slab_level_end(c, start, c->ev_comm);
}

// One slab level, peer mode: boundary rows, their push into the neighbours' ghost rows, then the
// interior (the interior rows read no ghost rows, so the epoch is published before them).
tsw_status step_slab_peer(tsw_ctx* c) {
    const bool start = (c->n == 0);
    tsw_status st;
    if ((st = peer_begin(c, c->stream))) return st;
    if ((st = launch_boundary_rows(c, start))) return st;
    if ((st = push_rows(c, c->ip, 1, c->stream))) return st;
    if ((st = peer_end(c, c->stream))) return st;
    if ((st = launch_interior_rows(c, start))) return st;
    std::swap(c->ic, c->ip);
    c->gdepth[c->ic] = 1;
    c->n++;
    return TSW_OK;
}

// Make the K outermost ghost rows of both current levels valid before temporally blocked passes.
tsw_status ensure_ghosts_nccl(tsw_ctx* c, int K) {
    tsw_status st;
    if (peer_mode(c)) {
        const bool need = c->gdepth[c->ic] < K || c->gdepth[c->ip] < K;  // identical on every rank
        if (!need) return TSW_OK;
        if ((st = peer_begin(c, c->stream))) return st;
        for (int which : {c->ic, c->ip})
            if (c->gdepth[which] < K) {
                if ((st = push_rows(c, which, K, c->stream))) return st;
                c->gdepth[which] = K;
            }
        return peer_end(c, c->stream);
    }
    for (int which : {c->ic, c->ip})
        if (c->gdepth[which] < K) {
            if ((st = exchange_nccl(c, c->buf[which], c->stream, K))) return st;
            c->gdepth[which] = K;
        }
    return TSW_OK;
}

bool tb_usable(const tsw_ctx* c);

// The remainder of a stepping call (2 ≤ r < K levels) runs as one pass of depth r instead of r
// single levels: every node is the same canonical expression, so the result is bitwise that of r
// one-level steps, and the fields make one HBM round trip instead of r.
struct DepthScope {
    tsw_ctx* c;
    int k0;
    DepthScope(tsw_ctx* c_, int r) : c(c_), k0(c_->tblock) { c->tblock = r; }
    ~DepthScope() { c->tblock = k0; }
};
struct GroupDepth {
    tsw_ctx** cs;
    int n;
    std::vector<int> k0;
    GroupDepth(tsw_ctx** cs_, int n_, int r) : cs(cs_), n(n_), k0(n_) {
        for (int i = 0; i < n; ++i) {
            k0[i] = cs[i]->tblock;
            cs[i]->tblock = r;
        }
    }
    ~GroupDepth() {
        for (int i = 0; i < n; ++i) cs[i]->tblock = k0[i];
    }
};
int pass_depth(const tsw_ctx* c, int64_t remaining) {
    return int(std::min<int64_t>(c->tblock, remaining));
}

// Peer halos: the halo operations of a stepping call, one epoch each.  The next operation follows
// from the ctx state alone, so every rank of a group issues the same sequence.
enum PeerOp { PEER_NONE = 0, PEER_ENSURE_1, PEER_ENSURE_K, PEER_LEVEL, PEER_PASS };
PeerOp next_peer_op(const tsw_ctx* c, int64_t remaining) {
    if (remaining <= 0) return PEER_NONE;
    const int d = pass_depth(c, remaining);  // a full pass, or the remainder as a shallower one
    const bool pass = tb_usable(c) && c->n > 0 && d >= 2;
    if (pass) {
        if (c->gdepth[c->ic] < d || c->gdepth[c->ip] < d) return PEER_ENSURE_K;
        return PEER_PASS;
    }
    if (c->gdepth[c->ic] < 1) return PEER_ENSURE_1;
    return PEER_LEVEL;
}
tsw_status ensure_ghosts_nccl(tsw_ctx* c, int K);
tsw_status step_slab_peer(tsw_ctx* c);
tsw_status tb_pass(tsw_ctx* c);
tsw_status run_peer_op(tsw_ctx* c, PeerOp op, int64_t remaining, int64_t* consumed) {
    *consumed = 0;
    switch (op) {
        case PEER_ENSURE_1: return ensure_ghosts_nccl(c, 1);
        case PEER_ENSURE_K: return ensure_ghosts_nccl(c, c->tblock);
        case PEER_LEVEL: *consumed = 1; return step_slab_peer(c);
        case PEER_PASS: {
            DepthScope ds(c, pass_depth(c, remaining));
            *consumed = c->tblock;
            c->en_now = c->en_fuse && c->tblock == remaining;   // the call's last pass
            const tsw_status st = tb_pass(c);
            c->en_now = false;
            return st;
        }
        default: return TSW_OK;
    }
}

bool tb_usable(const tsw_ctx* c) {
    if (peer_mode(c))
        for (int side = 0; side < 2; ++side)
            if (has_nb(c, side) && (!c->peer_buf[side][2] || !c->peer_buf[side][3])) return false;
    return c->tblock > 1 && c->g.dim == 2 && c->mode == MODE_LINE && c->buf[2] && c->buf[3] &&
           c->tblock <= c->G + (c->g.nranks == 1 ? 1 << 20 : 0);
}

// Two leapfrog levels captured once per (ic, ip) and replayed (single rank, n ≥ 1).
tsw_status step_pair_graph(tsw_ctx* c) {
    cudaGraphExec_t& ge = c->gexec[c->ic][c->ip];
    if (!ge) {
        const int ic0 = c->ic, ip0 = c->ip;
        const int64_t launches0 = c->launches;
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
        tsw_status st = launch_step2d(c, false, c->s_lo, c->s_hi);
        if (!st) {
            std::swap(c->ic, c->ip);
            st = launch_step2d(c, false, c->s_lo, c->s_hi);
        }
        cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
        c->ic = ic0;
        c->ip = ip0;
        c->launches = launches0;
        if (st) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return fail(TSW_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&ge, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            ge = nullptr;
            return fail(TSW_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
        }
    }
    CK(cudaGraphLaunch(ge, c->stream));
    c->launches += 2;
    c->n += 2;  // two levels: the buffer parity is unchanged
    return TSW_OK;
}

tsw_status do_steps(tsw_ctx* c, int64_t k) {
    if (k <= 0) return TSW_OK;
    if (c->scheme == 1) {
        for (int64_t s = 0; s < k; ++s) {
            tsw_status st = implicit_level(c);
            if (st) return st;
        }
        return TSW_OK;
    }
    if (c->g.dim == 1) return is_f64(c) ? step1d_t<double>(c, k) : step1d_t<float>(c, k);
    tsw_status st;
    if (c->g.nranks > 1 && peer_mode(c)) {
        for (int64_t s = 0;;) {
            const PeerOp op = next_peer_op(c, k - s);
            if (op == PEER_NONE) return TSW_OK;
            int64_t used = 0;
            if ((st = run_peer_op(c, op, k - s, &used))) return st;
            s += used;
        }
    }
    if (c->g.nranks > 1) {
        int64_t s = 0;
        if (c->n == 0) {
            if ((st = step_slab_overlapped(c))) return st;
            s = 1;
        }
        if (tb_usable(c) && pass_depth(c, k - s) >= 2) {
            if ((st = ensure_ghosts_nccl(c, c->tblock))) return st;
            for (; s + c->tblock <= k; s += c->tblock) {
                c->en_now = c->en_fuse && s + c->tblock == k;
                st = tb_pass(c);
                c->en_now = false;
                if (st) return st;
            }
            if (k - s >= 2) {
                DepthScope ds(c, int(k - s));
                c->en_now = c->en_fuse;
                st = tb_pass(c);
                c->en_now = false;
                if (st) return st;
                s = k;
            }
        }
        for (; s < k; ++s)
            if ((st = step_slab_overlapped(c))) return st;
        return TSW_OK;
    }
    int64_t s = 0;
    if (c->n == 0) {  // the start-up level
        if ((st = launch_step2d(c, true, c->s_lo, c->s_hi))) return st;
        std::swap(c->ic, c->ip);
        c->n++;
        s = 1;
    }
    if (tb_usable(c)) {
        // the call's last pass (a full one with no remainder after it, or the remainder pass)
        // carries the fused energy of the level it ends on
        for (; s + c->tblock <= k; s += c->tblock) {
            c->en_now = c->en_fuse && s + c->tblock == k;
            st = tb_pass(c);
            c->en_now = false;
            if (st) return st;
        }
        if (k - s >= 2) {
            DepthScope ds(c, int(k - s));
            c->en_now = c->en_fuse;
            st = tb_pass(c);
            c->en_now = false;
            if (st) return st;
            s = k;
        }
    }
    const bool graphs = c->use_graphs && !c->timing;
    for (; s + 1 < k && graphs; s += 2)
        if ((st = step_pair_graph(c))) return st;
    for (; s < k; ++s) {
        if ((st = launch_step2d(c, false, c->s_lo, c->s_hi))) return st;
        std::swap(c->ic, c->ip);
        c->n++;
    }
    return TSW_OK;
}

}  // namespace

// =============================================================================================
// ABI
// =============================================================================================
namespace {
template <typename T>
tsw_status alu_probe_t(int device, double* ops_per_s) {
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    T* out = nullptr;
    CK(cudaMalloc(&out, 256 * sizeof(T)));
    const int blocks = sms * 8, iters = sizeof(T) == 8 ? 20000 : 40000;
    k_alu_probe<T><<<blocks, 256, 0, s>>>(out, iters / 10, T(1), T(0.5));   // warm-up, clocks ramp
    CKL();
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0, s));
        k_alu_probe<T><<<blocks, 256, 0, s>>>(out, iters, T(1), T(0.5));
        CKL();
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    *ops_per_s = double(blocks) * 256.0 * iters * 24.0 / (double(best) * 1e-3);
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    return TSW_OK;
}

}  // namespace

extern "C" {

const char* tsw_version(void) { return "tsw 0.1 (sm_100a)"; }

const char* tsw_last_error(const tsw_ctx*) { return g_err.c_str(); }

tsw_status tsw_create(const tsw_grid_desc* gd, tsw_ctx** out) {
    if (!gd || !out) return fail(TSW_ERR_ARG, "NULL argument");
    *out = nullptr;
    const tsw_grid_desc g = *gd;
    if (g.dim != 1 && g.dim != 2) return fail(TSW_ERR_ARG, "dim must be 1 or 2");
    if (g.nx < 3) return fail(TSW_ERR_ARG, "nx must be >= 3");
    if (g.dim == 2 && g.ny < 3) return fail(TSW_ERR_ARG, "ny must be >= 3 in 2D");
    if (g.dim == 1 && g.ny != 1) return fail(TSW_ERR_ARG, "ny must be 1 in 1D");
    if (!(g.dx > 0) || (g.dim == 2 && !(g.dy > 0))) return fail(TSW_ERR_ARG, "dx, dy must be > 0");
    if (g.batch < 1) return fail(TSW_ERR_ARG, "batch must be >= 1");
    if (g.dtype != TSW_F32 && g.dtype != TSW_F64) return fail(TSW_ERR_ARG, "dtype must be TSW_F32 or TSW_F64");
    if (g.nranks < 1 || g.rank < 0 || g.rank >= g.nranks) return fail(TSW_ERR_ARG, "bad rank/nranks");
    if (g.dim == 1 && g.nranks != 1) return fail(TSW_ERR_ARG, "1D grids are not slab-decomposed");
    if (g.dim == 2 && g.ny < 2 * int64_t(g.nranks)) return fail(TSW_ERR_ARG, "need >= 2 rows per rank");
    if (g.nx > (int64_t(1) << 31) || g.ny > (int64_t(1) << 31)) return fail(TSW_ERR_ARG, "grid too large");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(TSW_ERR_CUDA, "no CUDA device (%s); this library has no CPU fallback", cudaGetErrorString(e));
    tsw_ctx* c = new tsw_ctx();
    c->g = g;
    if (g.device >= 0) {
        c->device = g.device;
    } else if (cudaGetDevice(&c->device) != cudaSuccess) {
        delete c;
        return fail(TSW_ERR_CUDA, "cudaGetDevice failed");
    }
    auto bail = [&](tsw_status s) {
        tsw_destroy(c);
        return s;
    };
    if (cudaSetDevice(c->device) != cudaSuccess) return bail(fail(TSW_ERR_CUDA, "cudaSetDevice(%d) failed", c->device));
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device);
    c->esz = (g.dtype == TSW_F64) ? 8 : 4;
    c->V = int(16 / c->esz);
    if (g.dim == 1) {
        c->r0 = 0;
        c->r1 = 1;
        c->ny_local = 1;
        c->rows_alloc = 1;
        c->pitch = round_up(g.nx, 32);
    } else {
        const int64_t base = g.ny / g.nranks, rem = g.ny % g.nranks;
        c->r0 = g.rank * base + std::min<int64_t>(g.rank, rem);
        c->r1 = c->r0 + base + (g.rank < rem ? 1 : 0);
        c->ny_local = c->r1 - c->r0;
        c->G = (g.nranks > 1) ? TSW_MAX_GHOST : 1;
        c->rows_alloc = c->ny_local + 2 * c->G;
        c->pitch = round_up(g.nx, 32 * c->V);
        c->s_lo = (c->r0 == 0) ? 2 : 1;
        c->s_hi = int32_t((c->r1 == g.ny) ? c->ny_local : c->ny_local + 1);
    }
    c->mstride = c->rows_alloc * c->pitch;
    c->fshift = size_t(c->G - 1) * size_t(c->pitch) * c->esz;
    if (g.stream) {
        c->stream = static_cast<cudaStream_t>(g.stream);
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(TSW_ERR_CUDA, "cudaStreamCreate failed"));
        c->own_stream = true;
    }
    if (g.dim == 2 && g.nranks > 1) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(TSW_ERR_CUDA, "exchange stream/events"));
    }
    const size_t bytes = size_t(g.batch) * c->mstride * c->esz;
    for (int k = 0; k < 2; ++k) {
        e = dmalloc_guarded(&c->buf[k], bytes, c->fshift, c->stream);
        if (e != cudaSuccess)
            return bail(fail(e == cudaErrorMemoryAllocation ? TSW_ERR_OOM : TSW_ERR_CUDA, "cudaMalloc(%zu): %s", bytes,
                             cudaGetErrorString(e)));
        cudaMemsetAsync(static_cast<char*>(c->buf[k]) - c->fshift, 0, bytes, c->stream);
    }
    c->nblk_red = 4096;  // partials per member (energy / wave2 reductions)
    if (cudaMalloc(&c->d_partial, sizeof(double) * size_t(g.batch) * c->nblk_red) != cudaSuccess ||
        cudaMalloc(&c->d_out, sizeof(double) * 4 * size_t(g.batch)) != cudaSuccess ||
        cudaMalloc(&c->d_argpart, sizeof(ArgVal) * 2 * size_t(g.batch) * c->nblk_red) != cudaSuccess ||
        cudaMalloc(&c->d_idx, sizeof(long long) * 4 * size_t(g.batch)) != cudaSuccess ||
        cudaMalloc(&c->d_u64, sizeof(unsigned long long) * 4) != cudaSuccess ||
        cudaMalloc(&c->d_eps, sizeof(double) * size_t(g.batch)) != cudaSuccess ||
        cudaMalloc(&c->d_amp, sizeof(double) * size_t(g.batch)) != cudaSuccess)
        return bail(fail(TSW_ERR_OOM, "scratch allocation failed"));
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(fail(TSW_ERR_CUDA, "stream sync failed"));
    *out = c;
    return TSW_OK;
}

void tsw_destroy(tsw_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    if (c->mbox) cudaFree(c->mbox);
    for (int k = 0; k < 4; ++k) dfree_guarded(c->buf[k], c->fshift);
    dfree_guarded(c->imp_s1, c->fshift);
    if (c->imp_t) cudaFree(c->imp_t);
    if (c->imp_tab) cudaFree(c->imp_tab);
    for (void* p : {c->imp_ycol, c->imp_cF, c->imp_cB, c->imp_ccon})
        if (p) cudaFree(p);
    dfree_guarded(c->h1, c->cshift_h);
    dfree_guarded(c->h2, c->cshift_h);
    dfree_guarded(c->c1, c->cshift);
    dfree_guarded(c->c2, c->cshift);
    void* ptrs[] = {c->d_eps, c->d_amp, c->d_partial, c->d_out, c->d_argpart, c->d_idx, c->d_u64, c->d_prof, c->d_fam,
                    c->d_en, c->en_result};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    drop_graphs(c);
    if (c->ev_bnd) cudaEventDestroy(c->ev_bnd);
    if (c->ev_comm) cudaEventDestroy(c->ev_comm);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

tsw_status tsw_set_coeff(tsw_ctx* c, const tsw_coeff_desc* h) {
    if (!c || !h) return fail(TSW_ERR_ARG, "NULL argument");
    if (h->kind != TSW_H_CONST && h->kind != TSW_H_DELTA_LINE_X && h->kind != TSW_H_DELTA_POINT)
        return fail(TSW_ERR_ARG, "kind must be CONST, DELTA_LINE_X or DELTA_POINT (FACES: tsw_set_coeff_faces)");
    if (h->kind == TSW_H_DELTA_POINT && c->g.dim != 2) return fail(TSW_ERR_ARG, "DELTA_POINT needs dim == 2");
    if (h->order != 1 && h->order != 2) return fail(TSW_ERR_ARG, "order must be 1 or 2");
    if (!(h->h_background > 0.0) || !std::isfinite(h->h_background))
        return fail(TSW_ERR_ARG, "h_background must be > 0 (positivity 0 < c0 <= h, P:165)");
    if (!std::isfinite(h->xs) || !std::isfinite(h->ys)) return fail(TSW_ERR_ARG, "xs, ys must be finite");
    if (!h->eps) return fail(TSW_ERR_ARG, "eps[batch] is required");
    std::vector<double> eps(h->eps, h->eps + c->g.batch), amp(size_t(c->g.batch), h->amp);
    if (h->amp_per_member) amp.assign(h->amp_per_member, h->amp_per_member + c->g.batch);
    for (int b = 0; b < c->g.batch; ++b) {
        if (!(eps[b] > 0.0 && eps[b] <= 1.0)) return fail(TSW_ERR_ARG, "eps[%d] = %g outside (0, 1] (P:335)", b, eps[b]);
        if (!(amp[b] >= 0.0) || !std::isfinite(amp[b])) return fail(TSW_ERR_ARG, "amp[%d] = %g must be >= 0", b, amp[b]);
    }
    tsw_status st = set_dev(c);
    if (st) return st;
    const int mode = (h->kind == TSW_H_DELTA_POINT) ? MODE_DENSE : MODE_LINE;
    if ((st = alloc_coeff(c, mode))) return st;
    CK(cudaMemcpyAsync(c->d_eps, eps.data(), sizeof(double) * eps.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_amp, amp.data(), sizeof(double) * amp.size(), cudaMemcpyHostToDevice, c->stream));
    CoeffArgs a;
    a.kind = h->kind;
    a.order = h->order;
    a.hb = h->h_background;
    a.xs = h->xs;
    a.ys = h->ys;
    a.dx = c->g.dx;
    a.dy = c->g.dy;
    a.eps = c->d_eps;
    a.amp = c->d_amp;
    a.nx = c->g.nx;
    a.ny = c->g.ny;
    a.r0 = c->r0;
    a.rows_alloc = c->rows_alloc;
    a.pitch = c->pitch;
    a.cpitch = c->cstride1;
    a.B = c->g.batch;
    a.s_base = 0;
    if (mode == MODE_LINE) {
        dim3 grid(unsigned(grid_for(c->cstride1, 256, 4 * c->sm_count)), unsigned(c->g.batch));
        k_coeff_line<<<grid, 256, 0, c->stream>>>(a, c->h1, c->h2);
    } else {
        a.s_base = 1 - c->G;
        dim3 grid(unsigned(grid_for(c->pitch, 256, 64)), unsigned(c->rows_alloc), unsigned(c->g.batch));
        k_coeff_point<<<grid, 256, 0, c->stream>>>(a, c->h1, c->h2);
    }
    CKL();
    c->launches++;
    c->kind = h->kind;
    c->xs = h->xs;
    c->ys = h->ys;
    c->hb = h->h_background;
    c->order = h->order;
    c->have_eps = true;
    if ((st = check_faces(c))) return st;
    c->have_coeff = true;
    c->have_init = false;
    return TSW_OK;
}

tsw_status tsw_set_coeff_profile(tsw_ctx* c, const tsw_profile_desc* p, const double* eps, const double* scale) {
    if (!c || !p || !eps) return fail(TSW_ERR_ARG, "NULL argument");
    if (p->nseg < 1 || !p->seg_value || (p->nseg > 1 && !p->seg_break)) return fail(TSW_ERR_ARG, "need >= 1 segment");
    if (p->nsing < 0 || (p->nsing > 0 && (!p->sing_loc || !p->sing_amp || !p->sing_order)))
        return fail(TSW_ERR_ARG, "bad singular terms");
    if (p->nseg > 64 || p->nsing > 64) return fail(TSW_ERR_ARG, "at most 64 segments / singular terms");
    for (int k = 0; k < p->nseg; ++k)
        if (!(p->seg_value[k] > 0.0) || !std::isfinite(p->seg_value[k]))
            return fail(TSW_ERR_ARG, "segment %d depth %g must be > 0 (P:165)", k, p->seg_value[k]);
    for (int k = 1; k + 1 < p->nseg; ++k)
        if (!(p->seg_break[k] > p->seg_break[k - 1])) return fail(TSW_ERR_ARG, "breaks must increase");
    for (int k = 0; k < p->nsing; ++k) {
        if (!(p->sing_amp[k] >= 0.0) || !std::isfinite(p->sing_amp[k]) || !std::isfinite(p->sing_loc[k]))
            return fail(TSW_ERR_ARG, "singular term %d: amplitude must be >= 0", k);
        if (p->sing_order[k] != 1 && p->sing_order[k] != 2) return fail(TSW_ERR_ARG, "singular order must be 1 or 2");
    }
    std::vector<double> ev(eps, eps + c->g.batch), sc(size_t(c->g.batch), 1.0);
    if (scale) sc.assign(scale, scale + c->g.batch);
    for (int b = 0; b < c->g.batch; ++b) {
        if (!(ev[b] > 0.0 && ev[b] <= 1.0)) return fail(TSW_ERR_ARG, "eps[%d] = %g outside (0, 1] (P:335)", b, ev[b]);
        if (!(sc[b] >= 0.0) || !std::isfinite(sc[b])) return fail(TSW_ERR_ARG, "scale[%d] must be >= 0", b);
    }
    tsw_status st = set_dev(c);
    if (st) return st;
    if ((st = alloc_coeff(c, MODE_LINE))) return st;
    std::vector<double> data;
    data.insert(data.end(), p->seg_value, p->seg_value + p->nseg);
    if (p->nseg > 1) data.insert(data.end(), p->seg_break, p->seg_break + p->nseg - 1);
    data.insert(data.end(), p->sing_loc, p->sing_loc + p->nsing);
    data.insert(data.end(), p->sing_amp, p->sing_amp + p->nsing);
    for (int k = 0; k < p->nsing; ++k) data.push_back(double(p->sing_order[k]));
    double* d_data = nullptr;
    CK(cudaMalloc(&d_data, std::max<size_t>(1, data.size()) * sizeof(double)));
    CK(cudaMemcpyAsync(d_data, data.data(), data.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_eps, ev.data(), sizeof(double) * ev.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_amp, sc.data(), sizeof(double) * sc.size(), cudaMemcpyHostToDevice, c->stream));
    ProfileArgs a;
    a.nseg = p->nseg;
    a.nsing = p->nsing;
    a.isotropic = p->isotropic;
    a.data = d_data;
    a.eps = c->d_eps;
    a.scale = c->d_amp;
    a.nx = c->g.nx;
    a.cpitch = c->cstride1;
    a.dx = c->g.dx;
    dim3 grid(unsigned(grid_for(c->cstride1, 128, 4 * c->sm_count)), unsigned(c->g.batch));
    k_coeff_profile<<<grid, 128, 0, c->stream>>>(a, c->h1, c->h2);
    cudaError_t e = cudaGetLastError();
    cudaError_t e2 = cudaStreamSynchronize(c->stream);
    if (c->d_prof) cudaFree(c->d_prof);
    c->d_prof = d_data;  // kept for tsw_coeff_norms
    c->prof_nseg = p->nseg;
    c->prof_nsing = p->nsing;
    if (e != cudaSuccess || e2 != cudaSuccess)
        return fail(TSW_ERR_CUDA, "k_coeff_profile: %s", cudaGetErrorString(e != cudaSuccess ? e : e2));
    c->launches++;
    c->kind = TSW_H_PROFILE_X;
    // A₂ (R18) measures left of the first singular term, else of the first jump
    c->xs = p->nsing > 0 ? p->sing_loc[0] : (p->nseg > 1 ? p->seg_break[0] : 0.0);
    c->ys = 0.0;
    c->have_eps = true;
    if ((st = check_faces(c))) return st;
    c->have_coeff = true;
    c->have_init = false;
    return TSW_OK;
}

tsw_status tsw_set_coeff_faces(tsw_ctx* c, const double* h1, const double* h2, int on_device) {
    if (!c || !h1) return fail(TSW_ERR_ARG, "NULL argument");
    if (c->g.dim == 2 && !h2) return fail(TSW_ERR_ARG, "h2 is required in 2D");
    if (!on_device) {
        // positivity 0 < c0 <= h on every face the stepper can use
        const size_t n1 = size_t(c->g.batch) * size_t(c->ny_local) * size_t(c->g.nx - 1);
        for (size_t k = 0; k < n1; ++k)
            if (!(h1[k] > 0.0) || !std::isfinite(h1[k])) return fail(TSW_ERR_ARG, "h1[%zu] = %g is not > 0", k, h1[k]);
        if (c->g.dim == 2) {
            const size_t rows = size_t(c->ny_local) + 1;
            for (size_t b = 0; b < size_t(c->g.batch); ++b)
                for (size_t k = 0; k < rows; ++k) {
                    const int64_t g = c->r0 + int64_t(k) - 1;  // face g + 1/2
                    if (g < 0 || g > c->g.ny - 2) continue;
                    for (size_t i = 0; i < size_t(c->g.nx); ++i) {
                        const double v = h2[(b * rows + k) * size_t(c->g.nx) + i];
                        if (!(v > 0.0) || !std::isfinite(v)) return fail(TSW_ERR_ARG, "h2 face (%zu, %lld+1/2) = %g is not > 0", i, (long long)g, v);
                    }
                }
        }
    }
    tsw_status st = set_dev(c);
    if (st) return st;
    const int mode = (c->g.dim == 1) ? MODE_LINE : MODE_DENSE;
    if ((st = alloc_coeff(c, mode))) return st;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const size_t B = size_t(c->g.batch);
    const size_t nx = size_t(c->g.nx);
    if (c->g.dim == 1) {
        CK(cudaMemcpy2DAsync(c->h1, c->cstride1 * sizeof(double), h1, (nx - 1) * sizeof(double), (nx - 1) * sizeof(double),
                             B, kind, c->stream));
        std::vector<double> hb(B * c->cstride2, 1.0);  // unused in 1D (no y faces)
        CK(cudaMemcpyAsync(c->h2, hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CSYNC(c);  // hb is a local
    } else {
        CK(cudaMemsetAsync(reinterpret_cast<char*>(c->h1) - c->cshift_h, 0, B * c->cstride1 * sizeof(double), c->stream));
        CK(cudaMemsetAsync(reinterpret_cast<char*>(c->h2) - c->cshift_h, 0, B * c->cstride2 * sizeof(double), c->stream));
        const size_t rows = size_t(c->ny_local);
        for (size_t b = 0; b < B; ++b) {
            // h1 local row j → storage row j+1 ; h2 row k (face between global rows r0+k−1 and
            // r0+k, i.e. storage rows k and k+1) → storage row k+1 (c2 storage row s = face
            // between storage rows s−1 and s).
            CK(cudaMemcpy2DAsync(c->h1 + b * c->mstride + c->pitch, c->pitch * sizeof(double),
                                 h1 + b * rows * (nx - 1), (nx - 1) * sizeof(double), (nx - 1) * sizeof(double), rows, kind,
                                 c->stream));
            CK(cudaMemcpy2DAsync(c->h2 + b * c->mstride + c->pitch, c->pitch * sizeof(double), h2 + b * (rows + 1) * nx,
                                 nx * sizeof(double), nx * sizeof(double), rows + 1, kind, c->stream));
        }
    }
    c->kind = TSW_H_FACES;
    if ((st = check_faces(c))) return st;
    c->have_coeff = true;
    c->have_init = false;
    return TSW_OK;
}

tsw_status tsw_read_faces(tsw_ctx* c, double* h1, double* h2) {
    if (!c || !h1) return fail(TSW_ERR_ARG, "NULL argument");
    if (!c->have_coeff) return fail(TSW_ERR_STATE, "no coefficients");
    tsw_status st = set_dev(c);
    if (st) return st;
    const size_t B = size_t(c->g.batch), nx = size_t(c->g.nx), rows = size_t(c->ny_local);
    if (c->mode == MODE_LINE) {
        std::vector<double> line(B * c->cstride1), hy(B * c->cstride2);
        CK(cudaMemcpyAsync(line.data(), c->h1, line.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hy.data(), c->h2, hy.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CSYNC(c);
        const size_t nrow = (c->g.dim == 1) ? 1 : rows;
        for (size_t b = 0; b < B; ++b)
            for (size_t j = 0; j < nrow; ++j)
                memcpy(h1 + (b * nrow + j) * (nx - 1), line.data() + b * c->cstride1, (nx - 1) * sizeof(double));
        if (h2 && c->g.dim == 2)
            for (size_t b = 0; b < B; ++b)
                for (size_t k = 0; k <= rows; ++k) {
                    const int64_t g = c->r0 + int64_t(k) - 1;
                    for (size_t i = 0; i < nx; ++i)
                        h2[(b * (rows + 1) + k) * nx + i] = (g >= 0 && g <= c->g.ny - 2) ? hy[b * c->cstride2 + i] : 0.0;
                }
        return TSW_OK;
    }
    for (size_t b = 0; b < B; ++b) {
        CK(cudaMemcpy2DAsync(h1 + b * rows * (nx - 1), (nx - 1) * sizeof(double), c->h1 + b * c->mstride + c->pitch,
                             c->pitch * sizeof(double), (nx - 1) * sizeof(double), rows, cudaMemcpyDeviceToHost, c->stream));
        if (h2)
            CK(cudaMemcpy2DAsync(h2 + b * (rows + 1) * nx, nx * sizeof(double), c->h2 + b * c->mstride + c->pitch,
                                 c->pitch * sizeof(double), nx * sizeof(double), rows + 1, cudaMemcpyDeviceToHost, c->stream));
    }
    CSYNC(c);
    if (h2) {
        // storage row s = face (g−1)+1/2 between storage rows s−1 and s; layout row k ↔ storage row k+1
        for (size_t b = 0; b < B; ++b)
            for (size_t k = 0; k <= rows; ++k) {
                const int64_t g = c->r0 + int64_t(k) - 1;
                if (g < 0 || g > c->g.ny - 2)
                    for (size_t i = 0; i < nx; ++i) h2[(b * (rows + 1) + k) * nx + i] = 0.0;
            }
    }
    return TSW_OK;
}

tsw_status tsw_set_initial(tsw_ctx* c, const void* u0, const void* u1, double dt, int on_device, uint32_t flags) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    tsw_status st = set_dev(c);
    if (st) return st;
    return set_levels(c, u0, u1, dt, on_device, flags, 0);
}

tsw_status tsw_set_state(tsw_ctx* c, const void* un, const void* unm1, int64_t n, double dt, int32_t on_device,
                         uint32_t flags) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    if (n < 1) return fail(TSW_ERR_ARG, "n must be >= 1 for a saved state (u^n, u^{n-1})");
    if (!unm1) return fail(TSW_ERR_ARG, "unm1 is NULL");
    tsw_status st = set_dev(c);
    if (st) return st;
    return set_levels(c, un, unm1, dt, on_device, flags & ~TSW_INIT_SHARED, n);
}

tsw_status tsw_step(tsw_ctx* c, int64_t nsteps) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    if (nsteps < 0) return fail(TSW_ERR_ARG, "nsteps must be >= 0");
    if (!c->have_init) return fail(TSW_ERR_STATE, "tsw_set_initial / tsw_set_state first");
    if (c->g.nranks > 1 && c->g.dim == 2 && !c->comm && !peer_mode(c))
        return fail(TSW_ERR_STATE, "nranks > 1: call tsw_nccl_init, enable peer halos, or step the slabs with tsw_group_step");
    tsw_status st = set_dev(c);
    if (st) return st;
    if ((st = do_steps(c, nsteps))) return st;
    return nccl_watch(c);   // an asynchronous communicator error surfaced by the halo traffic
}

tsw_status tsw_step_op(tsw_ctx* c, int64_t nsteps, int64_t* consumed) {
    if (!c || !consumed) return fail(TSW_ERR_ARG, "NULL argument");
    *consumed = 0;
    if (!c->have_init) return fail(TSW_ERR_STATE, "tsw_set_initial / tsw_set_state first");
    if (!peer_mode(c)) return fail(TSW_ERR_STATE, "tsw_step_op drives peer halos (TSW_OPT_HALO = 1) only");
    tsw_status st = set_dev(c);
    if (st) return st;
    const PeerOp op = next_peer_op(c, nsteps);
    return run_peer_op(c, op, nsteps, consumed);
}

tsw_status tsw_group_step(tsw_ctx** cs, int32_t n, int64_t nsteps) {
    if (!cs || n < 1 || n > TSW_GROUP_MAX) return fail(TSW_ERR_ARG, "bad ctx group (1..%d slabs)", TSW_GROUP_MAX);
    for (int r = 0; r < n; ++r) {
        if (!cs[r] || !cs[r]->have_init) return fail(TSW_ERR_STATE, "group member %d not initialised", r);
        if (cs[r]->g.dim != 2 || cs[r]->g.nranks != n || cs[r]->g.rank != r)
            return fail(TSW_ERR_ARG, "group member %d must be rank %d of %d (2D)", r, r, n);
        if (cs[r]->stream != cs[0]->stream || cs[r]->device != cs[0]->device)
            return fail(TSW_ERR_ARG, "loopback group members must share one device and stream");
        if (cs[r]->n != cs[0]->n || cs[r]->ic != cs[0]->ic || cs[r]->ip != cs[0]->ip)
            return fail(TSW_ERR_STATE, "group members are at different levels");
        if (cs[r]->tblock != cs[0]->tblock || tb_usable(cs[r]) != tb_usable(cs[0]))
            return fail(TSW_ERR_ARG, "group members must share the temporal blocking setting");
    }
    tsw_ctx* c0 = cs[0];
    tsw_status st = set_dev(c0);
    if (st) return st;
    if (peer_mode(c0)) {
        // peer halos: the members' halo operations are issued epoch by epoch on the shared stream
        // (every rank's operation e before any rank's e + 1), so each wait is satisfied on arrival
        for (int64_t s = 0;;) {
            const PeerOp op = next_peer_op(c0, nsteps - s);
            if (op == PEER_NONE) return TSW_OK;
            int64_t used = 0;
            for (int r = 0; r < n; ++r)
                if ((st = run_peer_op(cs[r], op, nsteps - s, &used))) return st;
            s += used;
        }
    }
    bool need = false;
    for (int r = 0; r < n; ++r) need = need || !cs[r]->ghosts_valid;
    if (need) {
        // ghost rows of both levels (set_initial / set_state cannot exchange without NCCL)
        if ((st = exchange_loopback(cs, n, 0, c0->stream, c0->G))) return st;
        if ((st = exchange_loopback(cs, n, 1, c0->stream, c0->G))) return st;
        for (int r = 0; r < n; ++r) {
            cs[r]->ghosts_valid = true;
            cs[r]->gdepth[cs[r]->ic] = cs[r]->gdepth[cs[r]->ip] = c0->G;
        }
    }
    // one level: every slab's boundary rows, the loopback copies of the new rows on the aux stream,
    // every slab's interior rows — the phases of step_slab_overlapped with the copies in place of
    // the NCCL messages
    auto single = [&]() -> tsw_status {
        const bool start = (c0->n == 0);
        tsw_status e;
        for (int r = 0; r < n; ++r)
            if ((e = slab_level_begin(cs[r], start))) return e;
        CK(cudaStreamWaitEvent(c0->aux, cs[n - 1]->ev_bnd, 0));   // one stream: covers every slab's rows
        if ((e = exchange_loopback(cs, n, 1, c0->aux, 1))) return e;
        CK(cudaEventRecord(c0->ev_comm, c0->aux));
        for (int r = 0; r < n; ++r)
            if ((e = slab_level_end(cs[r], start, c0->ev_comm))) return e;
        return TSW_OK;
    };
    int64_t s = 0;
    if (c0->n == 0 && nsteps > 0) {
        if ((st = single())) return st;
        s = 1;
    }
    // one pass of K levels (every member's depth set to K for its duration): the phases of tb_pass
    // (tb_pass_begin / tb_pass_end) with loopback copies of the K boundary rows of both new levels
    auto pass = [&](int K, bool last) -> tsw_status {
        GroupDepth gd(cs, n, K);
        for (int lv = 0; lv < 2; ++lv) {
            const int bi = lv ? c0->ip : c0->ic;
            if (c0->gdepth[bi] < K) {
                tsw_status e = exchange_loopback_buf(cs, n, bi, c0->stream, K);
                if (e) return e;
                for (int r = 0; r < n; ++r) cs[r]->gdepth[bi] = K;
            }
        }
        TbPassState ps[TSW_GROUP_MAX];
        tsw_status e = TSW_OK;
        for (int r = 0; r < n; ++r) cs[r]->en_now = cs[r]->en_fuse && last;
        for (int r = 0; r < n && !e; ++r) e = tb_pass_begin(cs[r], ps[r]);
        if (!e) {
            CK(cudaStreamWaitEvent(c0->aux, cs[n - 1]->ev_bnd, 0));
            e = exchange_loopback_buf(cs, n, ps[0].fk, c0->aux, K);
            if (!e) e = exchange_loopback_buf(cs, n, ps[0].fkm1, c0->aux, K);
            if (!e) CK(cudaEventRecord(c0->ev_comm, c0->aux));
        }
        for (int r = 0; r < n && !e; ++r) e = tb_pass_end(cs[r], ps[r], c0->ev_comm);
        for (int r = 0; r < n; ++r) cs[r]->en_now = false;
        return e;
    };
    if (tb_usable(c0)) {
        const int K = c0->tblock;
        for (; s + K <= nsteps; s += K)
            if ((st = pass(K, s + K == nsteps))) return st;
        if (nsteps - s >= 2) {  // the remainder as one shallower pass (see DepthScope)
            if ((st = pass(int(nsteps - s), true))) return st;
            s = nsteps;
        }
    }
    for (; s < nsteps; ++s)
        if ((st = single())) return st;
    return TSW_OK;
}

tsw_status energy_guard(tsw_ctx* c, const double* E) {
    const int B = c->g.batch;
    for (int b = 0; b < B; ++b)
        if (!std::isfinite(E[b]))
            return fail(TSW_ERR_UNSTABLE, "member %d: non-finite energy at level %lld (unstable: dt above the CFL bound? R16/R17)",
                        b, (long long)c->n);
    // drift: only for the whole grid's energy (a slab's share is not conserved: energy crosses slabs)
    if (c->en_drift_k <= 0 || (c->g.nranks > 1 && !c->comm)) return TSW_OK;
    if (c->en_ref.empty()) {
        c->en_ref.assign(E, E + B);
        c->en_ref_n = c->n;
        return TSW_OK;
    }
    const double tol = std::pow(10.0, -double(c->en_drift_k));
    for (int b = 0; b < B; ++b)
        if (c->en_ref[b] > 0.0 && !(std::fabs(E[b] - c->en_ref[b]) <= tol * c->en_ref[b]))
            return fail(TSW_ERR_UNSTABLE, "member %d: energy %.17g at level %lld drifted from %.17g at level %lld by more than %g relative (blow-up)",
                        b, E[b], (long long)c->n, c->en_ref[b], (long long)c->en_ref_n, tol);
    return TSW_OK;
}

tsw_status tsw_energy(tsw_ctx* c, double* out_B) {
    if (!c || !out_B) return fail(TSW_ERR_ARG, "NULL argument");
    if (!c->have_init || c->n < 1) return fail(TSW_ERR_STATE, "energy E^{n-1/2} needs n >= 1");
    tsw_status st = set_dev(c);
    if (st) return st;
    if (c->en_level == c->n && c->en_result) {
        // reduced by the pass that wrote u^n, u^{n−1} (TSW_OPT_ENERGY_FUSE); the node form reads no
        // ghost row, so slabs need no halo epoch — only the sum over ranks
        const double* src = c->en_result;
        if (c->g.nranks > 1 && c->comm) {
            NK(nccl().AllReduce(c->en_result, c->d_out, size_t(c->g.batch), NCCL_F64, NCCL_SUM, c->comm, c->stream));
            src = c->d_out;
        }
        CK(cudaMemcpyAsync(out_B, src, sizeof(double) * c->g.batch, cudaMemcpyDeviceToHost, c->stream));
        CSYNC(c);
        return energy_guard(c, out_B);
    }
    // peer halos: a ghost-reading collective is an epoch of its own (no neighbour overwrites the
    // ghost rows while they are read)
    if (peer_mode(c) && (st = peer_begin(c, c->stream))) return st;
    int nparts = 0;
    if (c->g.dim == 2) {
        Energy2Args a;
        a.mode = c->mode;
        a.unp1 = c->buf[c->ic];
        a.un = c->buf[c->ip];
        a.c1 = c->c1;
        a.c2 = c->c2;
        a.nx = c->g.nx;
        a.ny = c->g.ny;
        a.r0 = c->r0;
        a.pitch = c->pitch;
        a.mstride = c->mstride;
        a.cstride1 = c->cstride1;
        a.cstride2 = c->cstride2;
        a.rows = int32_t(c->ny_local);
        const int64_t cta_w = 8 * 32 * int64_t(16 / c->esz);
        a.cta_strips = (c->pitch + cta_w - 1) / cta_w;
        // ≈ 8 CTAs per SM over the batch, ≤ nblk_red partials per member
        int64_t chunks = (int64_t(8) * c->sm_count + a.cta_strips * c->g.batch - 1) / (a.cta_strips * c->g.batch);
        chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, std::max<int64_t>(1, c->nblk_red / a.cta_strips)));
        chunks = std::min<int64_t>(chunks, c->ny_local);
        a.rows_per_item = int32_t((c->ny_local + chunks - 1) / chunks);
        a.chunks = int32_t((c->ny_local + a.rows_per_item - 1) / a.rows_per_item);
        a.items_per_member = a.cta_strips * a.chunks;
        if (a.items_per_member > c->nblk_red) return fail(TSW_ERR_ARG, "energy: too many partials (pitch too wide)");
        nparts = int(a.items_per_member);
        dim3 grid(unsigned(a.items_per_member), unsigned(c->g.batch));
        if (is_f64(c)) {
            if (c->mode == MODE_LINE) k_energy2d<double, MODE_LINE><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
            else k_energy2d<double, MODE_DENSE><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
        } else {
            if (c->mode == MODE_LINE) k_energy2d<float, MODE_LINE><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
            else k_energy2d<float, MODE_DENSE><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
        }
        CKL();
    } else {
        EnergyArgs a;
        a.dim = c->g.dim;
        a.mode = c->mode;
        a.unp1 = c->buf[c->ic];
        a.un = c->buf[c->ip];
        a.c1 = c->c1;
        a.c2 = c->c2;
        a.nx = c->g.nx;
        a.ny = c->g.ny;
        a.r0 = c->r0;
        a.pitch = c->pitch;
        a.mstride = c->mstride;
        a.cstride1 = c->cstride1;
        a.cstride2 = c->cstride2;
        a.ny_local = c->ny_local;
        a.nblk = grid_for(c->g.nx, 256, c->nblk_red);
        nparts = a.nblk;
        dim3 grid(unsigned(a.nblk), unsigned(c->g.batch));
        if (is_f64(c))
            k_energy<double><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
        else
            k_energy<float><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
        CKL();
    }
    const double w = ((c->g.dim == 1) ? c->g.dx : c->g.dx * c->g.dy) / (c->dt * c->dt);
    k_energy_final<<<c->g.batch, 32, 0, c->stream>>>(c->d_partial, nparts, w, c->d_out);
    CKL();
    c->launches += 2;
    if (peer_mode(c) && (st = peer_end(c, c->stream))) return st;
    if (peer_mode(c) && (st = peer_check(c))) return st;
    if (c->g.nranks > 1 && c->comm)  // without a communicator (loopback / peer group): this slab's share
        NK(nccl().AllReduce(c->d_out, c->d_out, size_t(c->g.batch), NCCL_F64, NCCL_SUM, c->comm, c->stream));
    CK(cudaMemcpyAsync(out_B, c->d_out, sizeof(double) * c->g.batch, cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    return energy_guard(c, out_B);
}

tsw_status tsw_wave2(tsw_ctx* c, int32_t bg, double* out_B2, int64_t* idx_B2) {
    if (!c || !out_B2) return fail(TSW_ERR_ARG, "NULL argument");
    if (!c->have_init) return fail(TSW_ERR_STATE, "no field");
    if (!c->have_eps) return fail(TSW_ERR_STATE, "wave2 needs eps/xs from tsw_set_coeff");
    if (bg < 0 || bg >= c->g.batch) return fail(TSW_ERR_ARG, "bg_member out of range");
    tsw_status st = set_dev(c);
    if (st) return st;
    Wave2Args a;
    a.dim = c->g.dim;
    a.u = c->buf[c->ic];
    a.nx = c->g.nx;
    a.ny = c->g.ny;
    a.r0 = c->r0;
    a.pitch = c->pitch;
    a.mstride = c->mstride;
    a.ny_local = c->ny_local;
    a.bg = bg;
    a.dx = c->g.dx;
    a.xs = c->xs;
    a.eps = c->d_eps;
    // column tiles × row chunks: ≈ 8 (fp64) / 16 (fp32: 1024-column tiles, few of them) CTAs per SM
    // over the batch — tiles outside the region exit at once (about half of them for the configs'
    // x ≤ −ε region) — ≤ nblk_red partials per member
    const int64_t rows = (c->g.dim == 1) ? 1 : c->ny_local;
    a.tiles = (c->g.nx + 256 * int64_t(16 / c->esz) - 1) / (256 * int64_t(16 / c->esz));
    const int64_t per_sm = is_f64(c) ? 8 : 16;
    int64_t chunks = (per_sm * c->sm_count + a.tiles * c->g.batch - 1) / (a.tiles * c->g.batch);
    chunks = std::max<int64_t>(1, std::min<int64_t>({chunks, rows, std::max<int64_t>(1, c->nblk_red / a.tiles)}));
    a.rows_per_chunk = int32_t((rows + chunks - 1) / chunks);
    chunks = (rows + a.rows_per_chunk - 1) / a.rows_per_chunk;
    a.nblk = int(a.tiles * chunks);
    if (a.nblk > c->nblk_red) return fail(TSW_ERR_ARG, "wave2: too many partials (row too wide)");
    dim3 grid(unsigned(a.nblk), unsigned(c->g.batch));
    if (is_f64(c))
        k_wave2<double><<<grid, 256, 0, c->stream>>>(a, c->d_argpart);
    else
        k_wave2<float><<<grid, 256, 0, c->stream>>>(a, c->d_argpart);
    CKL();
    k_wave2_final<<<c->g.batch, 32, 0, c->stream>>>(c->d_argpart, a.nblk, c->d_out, c->d_idx);
    CKL();
    c->launches += 2;
    const int B = c->g.batch;
    std::vector<double> v(2 * size_t(B));
    std::vector<long long> ix(2 * size_t(B));
    CK(cudaMemcpyAsync(v.data(), c->d_out, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(ix.data(), c->d_idx, sizeof(long long) * 2 * B, cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    if (c->g.nranks > 1 && c->comm) {  // without a communicator (loopback group): this slab's extrema
        // values: empty local regions must not win → ±inf; indices: first global extremum
        std::vector<double> mx(B), mn(B);
        for (int b = 0; b < B; ++b) {
            mx[b] = ix[2 * b] >= 0 ? v[2 * b] : -INFINITY;
            mn[b] = ix[2 * b + 1] >= 0 ? v[2 * b + 1] : INFINITY;
        }
        double* d = c->d_out;
        CK(cudaMemcpyAsync(d, mx.data(), sizeof(double) * B, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d + B, mn.data(), sizeof(double) * B, cudaMemcpyHostToDevice, c->stream));
        NK(nccl().AllReduce(d, d, size_t(B), NCCL_F64, NCCL_MAX, c->comm, c->stream));
        NK(nccl().AllReduce(d + B, d + B, size_t(B), NCCL_F64, NCCL_MIN, c->comm, c->stream));
        std::vector<double> gmx(B), gmn(B);
        CK(cudaMemcpyAsync(gmx.data(), d, sizeof(double) * B, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(gmn.data(), d + B, sizeof(double) * B, cudaMemcpyDeviceToHost, c->stream));
        CSYNC(c);
        std::vector<long long> li(2 * size_t(B));
        for (int b = 0; b < B; ++b) {
            li[2 * b] = (ix[2 * b] >= 0 && mx[b] == gmx[b]) ? ix[2 * b] : LLONG_MAX;
            li[2 * b + 1] = (ix[2 * b + 1] >= 0 && mn[b] == gmn[b]) ? ix[2 * b + 1] : LLONG_MAX;
        }
        CK(cudaMemcpyAsync(c->d_idx, li.data(), sizeof(long long) * 2 * B, cudaMemcpyHostToDevice, c->stream));
        NK(nccl().AllReduce(c->d_idx, c->d_idx, size_t(2 * B), NCCL_INT64, NCCL_MIN, c->comm, c->stream));
        CK(cudaMemcpyAsync(li.data(), c->d_idx, sizeof(long long) * 2 * B, cudaMemcpyDeviceToHost, c->stream));
        CSYNC(c);
        for (int b = 0; b < B; ++b) {
            const bool e1 = li[2 * b] == LLONG_MAX, e2 = li[2 * b + 1] == LLONG_MAX;
            v[2 * b] = e1 ? 0.0 : gmx[b];
            v[2 * b + 1] = e2 ? 0.0 : gmn[b];
            ix[2 * b] = e1 ? -1 : li[2 * b];
            ix[2 * b + 1] = e2 ? -1 : li[2 * b + 1];
        }
    }
    for (int k = 0; k < 2 * B; ++k) {
        out_B2[k] = v[k];
        if (idx_B2) idx_B2[k] = ix[k];
    }
    return TSW_OK;
}

tsw_status tsw_family_l2(tsw_ctx* c, double* out_BB) {
    if (!c || !out_BB) return fail(TSW_ERR_ARG, "NULL argument");
    if (!c->have_init) return fail(TSW_ERR_STATE, "no field");
    const int B = c->g.batch;
    if (B > 200) return fail(TSW_ERR_ARG, "family distances support batch <= 200");
    tsw_status st = set_dev(c);
    if (st) return st;
    FamilyArgs a;
    a.u = c->buf[c->ic];
    a.nx = c->g.nx;
    a.pitch = c->pitch;
    a.mstride = c->mstride;
    a.rows = int32_t(c->g.dim == 1 ? 1 : c->ny_local);
    a.row0 = (c->g.dim == 1) ? 0 : 1;
    a.B = B;
    a.nblk = (B + 3) / 4;
    // one thread per block of 4 × 4 member pairs (and ≥ B / 16 · FAM_TN threads for the prefetch),
    // at most FAM_MAXT per CTA: groups of blocks on blockIdx.y
    const int npairs = a.nblk * (a.nblk + 1) / 2;
    const int need_t = std::max(npairs, (B * FAM_TN + FAM_EPT - 1) / FAM_EPT);
    const int nthr = std::min(FAM_MAXT, (need_t + 31) / 32 * 32);
    const int groups = (npairs + nthr - 1) / nthr;
    a.tiles_per_row = (c->g.nx + FAM_TN - 1) / FAM_TN;
    a.ntiles = int64_t(a.rows) * a.tiles_per_row;
    const size_t smem = size_t(2) * fam_rows_elems(a.nblk) * sizeof(double);
    if (smem > 48 * 1024) {
        if (is_f64(c)) CK(cudaFuncSetAttribute(k_family_l2<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        else CK(cudaFuncSetAttribute(k_family_l2<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    // one wave: exactly the resident CTAs (all groups), each a contiguous, balanced range of tiles
    int occ = 1;
    if (is_f64(c)) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_family_l2<double>, nthr, smem));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_family_l2<float>, nthr, smem));
    const int64_t want = std::min<int64_t>(a.ntiles, std::max<int64_t>(1, int64_t(std::max(occ, 1)) * c->sm_count / groups));
    a.tiles_per_cta = (a.ntiles + want - 1) / want;
    const int ncta = int((a.ntiles + a.tiles_per_cta - 1) / a.tiles_per_cta);
    // partials [ncta][B][B] (each group writes its own pairs), then the per-pair sums [B][B]
    const size_t need = size_t(ncta + 1) * B * B;
    if (c->fam_cap < need) {
        if (c->d_fam) cudaFree(c->d_fam);
        c->d_fam = nullptr;
        c->fam_cap = 0;
        CK(cudaMalloc(&c->d_fam, need * sizeof(double)));
        c->fam_cap = need;
    }
    double* d_sum = c->d_fam + size_t(ncta) * B * B;
    CK(cudaMemsetAsync(c->d_fam, 0, size_t(ncta) * B * B * sizeof(double), c->stream));
    const dim3 grid{unsigned(ncta), unsigned(groups), 1u};
    if (is_f64(c))
        k_family_l2<double><<<grid, nthr, smem, c->stream>>>(a, c->d_fam);
    else
        k_family_l2<float><<<grid, nthr, smem, c->stream>>>(a, c->d_fam);
    CKL();
    k_family_final<<<std::max(1, (B * B + 255) / 256), 256, 0, c->stream>>>(c->d_fam, ncta, B, d_sum);
    CKL();
    c->launches += 2;
    // the sums Σ (u_i − u_j)² add over ranks on the device; weight and root on the host
    if (c->g.nranks > 1 && c->comm)
        NK(nccl().AllReduce(d_sum, d_sum, size_t(B) * B, NCCL_F64, NCCL_SUM, c->comm, c->stream));
    CK(cudaMemcpyAsync(out_BB, d_sum, sizeof(double) * B * B, cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    const double w = (c->g.dim == 1) ? c->g.dx : c->g.dx * c->g.dy;
    for (int k = 0; k < B * B; ++k) out_BB[k] = std::sqrt(w * out_BB[k]);
    return TSW_OK;
}

tsw_status tsw_field_norms(tsw_ctx* c, double* out_B4) {
    if (!c || !out_B4) return fail(TSW_ERR_ARG, "NULL argument");
    if (!c->have_init) return fail(TSW_ERR_STATE, "no field");
    tsw_status st = set_dev(c);
    if (st) return st;
    if (peer_mode(c) && (st = peer_begin(c, c->stream))) return st;   // reads ghost rows (see tsw_energy)
    NormArgs a;
    a.dim = c->g.dim;
    a.un = c->buf[c->ic];
    a.unm1 = c->buf[c->ip];
    a.nx = c->g.nx;
    a.ny = c->g.ny;
    a.r0 = c->r0;
    a.pitch = c->pitch;
    a.mstride = c->mstride;
    a.rows = int32_t(c->g.dim == 1 ? 1 : c->ny_local);
    a.nblk = grid_for(int64_t(a.rows) * c->g.nx, 256, std::min(c->nblk_red / 4, 4 * c->sm_count));
    dim3 grid(unsigned(a.nblk), unsigned(c->g.batch));
    if (is_f64(c))
        k_norms<double><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
    else
        k_norms<float><<<grid, 256, 0, c->stream>>>(a, c->d_partial);
    CKL();
    double* d4 = reinterpret_cast<double*>(c->d_argpart);  // scratch: 4·B doubles
    k_norms_final<<<c->g.batch, 32, 0, c->stream>>>(c->d_partial, a.nblk, c->g.batch, d4);
    CKL();
    c->launches += 2;
    if (peer_mode(c) && (st = peer_end(c, c->stream))) return st;
    if (c->g.nranks > 1 && c->comm) NK(nccl().AllReduce(d4, d4, size_t(4) * c->g.batch, NCCL_F64, NCCL_SUM, c->comm, c->stream));
    CK(cudaMemcpyAsync(out_B4, d4, sizeof(double) * 4 * c->g.batch, cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    const double w = (c->g.dim == 1) ? c->g.dx : c->g.dx * c->g.dy;
    for (int b = 0; b < c->g.batch; ++b) {
        double* o = out_B4 + 4 * b;
        o[0] = std::sqrt(w * o[0]);
        o[1] = (c->n >= 1) ? std::sqrt(w * o[1]) / c->dt : 0.0;  // u_t needs two levels
        o[2] = std::sqrt(w * o[2]) / c->g.dx;
        o[3] = (c->g.dim == 2) ? std::sqrt(w * o[3]) / c->g.dy : 0.0;
    }
    return TSW_OK;
}

tsw_status tsw_coeff_norms(tsw_ctx* c, double* out_B3) {
    if (!c || !out_B3) return fail(TSW_ERR_ARG, "NULL argument");
    if (!c->have_coeff) return fail(TSW_ERR_STATE, "no coefficients");
    tsw_status st = set_dev(c);
    if (st) return st;
    CoeffNormArgs a;
    a.kind = c->kind;
    a.order = c->order;
    a.hb = c->hb;
    a.xs = c->xs;
    a.ys = c->ys;
    a.dx = c->g.dx;
    a.dy = c->g.dy;
    a.eps = c->d_eps;
    a.amp = c->d_amp;
    a.prof = c->d_prof;
    a.nseg = c->prof_nseg;
    a.nsing = c->prof_nsing;
    a.h1 = c->h1;
    a.h2 = (c->g.dim == 2) ? c->h2 : nullptr;
    a.nx = c->g.nx;
    a.ny = c->g.ny;
    a.r0 = c->r0;
    a.rows = c->ny_local;
    a.pitch = c->pitch;
    a.cstride1 = c->cstride1;
    a.cstride2 = c->cstride2;
    a.mstride = c->mstride;
    a.mode = c->mode;
    unsigned long long* d = reinterpret_cast<unsigned long long*>(c->d_argpart);
    CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * 3 * c->g.batch, c->stream));
    const int64_t total = ((c->mode == MODE_LINE) ? 1 : c->ny_local) * c->g.nx;
    dim3 grid(unsigned(grid_for(total, 256, 4 * c->sm_count)), unsigned(c->g.batch));
    k_coeff_norms<<<grid, 256, 0, c->stream>>>(a, d);
    CKL();
    c->launches++;
    std::vector<unsigned long long> bits(size_t(3) * c->g.batch);
    CK(cudaMemcpyAsync(bits.data(), d, sizeof(unsigned long long) * bits.size(), cudaMemcpyDeviceToHost, c->stream));
    CSYNC(c);
    for (size_t k = 0; k < bits.size(); ++k) memcpy(&out_B3[k], &bits[k], sizeof(double));
    if (c->g.nranks > 1 && c->comm) {
        double* dd = reinterpret_cast<double*>(d);
        CK(cudaMemcpyAsync(dd, out_B3, sizeof(double) * bits.size(), cudaMemcpyHostToDevice, c->stream));
        NK(nccl().AllReduce(dd, dd, bits.size(), NCCL_F64, NCCL_MAX, c->comm, c->stream));
        CK(cudaMemcpyAsync(out_B3, dd, sizeof(double) * bits.size(), cudaMemcpyDeviceToHost, c->stream));
        CSYNC(c);
    }
    return TSW_OK;
}

tsw_status tsw_read(tsw_ctx* c, int32_t which, void* dst, int32_t to_device) {
    if (!c || !dst) return fail(TSW_ERR_ARG, "NULL argument");
    if (which != 0 && which != 1) return fail(TSW_ERR_ARG, "which must be 0 (u^n) or 1 (u^{n-1})");
    tsw_status st = set_dev(c);
    if (st) return st;
    const void* src = c->buf[which ? c->ip : c->ic];
    const cudaMemcpyKind kind = to_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const size_t w = size_t(c->g.nx) * c->esz;
    const size_t rows = size_t(c->ny_local);
    for (int b = 0; b < c->g.batch; ++b) {
        const char* s = static_cast<const char*>(src) + size_t(b) * c->mstride * c->esz +
                        (c->g.dim == 2 ? size_t(c->pitch) * c->esz : 0);
        char* d = static_cast<char*>(dst) + size_t(b) * rows * w;
        CK(cudaMemcpy2DAsync(d, w, s, size_t(c->pitch) * c->esz, w, rows, kind, c->stream));
    }
    if (!to_device) {
        CSYNC(c);
        if ((st = peer_check(c))) return st;
    }
    return TSW_OK;
}

tsw_status tsw_info(tsw_ctx* c, int64_t* n, double* t, double* dt_max) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    tsw_status st = set_dev(c);
    if (st) return st;
    CSYNC(c);
    if (n) *n = c->n;
    if (t) *t = double(c->n) * c->dt;
    if (dt_max) *dt_max = c->have_coeff ? c->dt_max : 0.0;
    return TSW_OK;
}

tsw_status tsw_sync(tsw_ctx* c) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    tsw_status st = set_dev(c);
    if (st) return st;
    CSYNC(c);
    return TSW_OK;
}

int64_t tsw_launch_count(const tsw_ctx* c) { return c ? c->launches : 0; }

tsw_status guard_fill(tsw_ctx* c);

tsw_status tsw_set_option(tsw_ctx* c, int32_t key, int64_t value) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    drop_graphs(c);  // captured launches bake in the kernel variant and its shape
    if (key == TSW_OPT_GRAPHS) {
        c->use_graphs = value != 0;
        return TSW_OK;
    }
    if (key == TSW_OPT_TBLOCK) {
        if (!(value >= 1 && value <= TSW_MAX_TB))
            return fail(TSW_ERR_ARG, "temporal blocking depth must be 1..%d", TSW_MAX_TB);
        if (value > 1 && c->g.dim != 2) return fail(TSW_ERR_ARG, "temporal blocking needs a 2D grid");
        if (value > 1 && c->g.nranks > 1 && value > c->G)
            return fail(TSW_ERR_ARG, "temporal blocking depth %d exceeds the %d ghost rows of a slab", int(value), c->G);
        tsw_status st = set_dev(c);
        if (st) return st;
        if (value > 1 && !c->buf[2]) {
            // two more levels for the out-of-place passes (zeroed: boundaries stay +0)
            const size_t bytes = size_t(c->g.batch) * c->mstride * c->esz;
            for (int k = 2; k < 4; ++k) {
                cudaError_t e = dmalloc_guarded(&c->buf[k], bytes, c->fshift, c->stream);
                if (e != cudaSuccess) {
                    for (int j = 2; j < 4; ++j) {
                        dfree_guarded(c->buf[j], c->fshift);
                        c->buf[j] = nullptr;
                    }
                    return fail(e == cudaErrorMemoryAllocation ? TSW_ERR_OOM : TSW_ERR_CUDA, "TB buffers: %s",
                                cudaGetErrorString(e));
                }
            }
        }
        c->tblock = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_SCHEME) {
        if (value != 0 && value != 1) return fail(TSW_ERR_ARG, "scheme must be 0 (leapfrog) or 1 (implicit)");
        if (value == 1) {
            if (c->g.nranks != 1) return fail(TSW_ERR_ARG, "the implicit scheme is single-rank");
            if (c->g.dim == 2 && (c->g.nx - 2 > IMP_SCAN_MAX || c->g.ny - 2 > IMP_SCAN_MAX))
                return fail(TSW_ERR_ARG, "implicit line solves: at most %d unknowns per line", IMP_SCAN_MAX);
            tsw_status st = set_dev(c);
            if (st) return st;
            const size_t fbytes = size_t(c->g.batch) * c->mstride * c->esz;
            if (!c->imp_s1) {
                cudaError_t e = dmalloc_guarded(&c->imp_s1, fbytes, c->fshift, c->stream);
                if (e != cudaSuccess) return fail(TSW_ERR_OOM, "implicit scratch: %s", cudaGetErrorString(e));
            }
            if (!c->imp_t) {
                c->imp_pt = round_up(c->g.dim == 2 ? c->g.ny : c->pitch, 32);
                const size_t tbytes = size_t(c->g.batch) * size_t(c->g.dim == 2 ? c->g.nx : 1) * c->imp_pt * c->esz;
                CK(cudaMalloc(&c->imp_t, tbytes));
                CK(cudaMemsetAsync(c->imp_t, 0, tbytes, c->stream));
            }
            if (!c->imp_tab && c->g.dim == 2) {
                c->imp_tpitch = round_up(c->g.nx, 32);
                CK(cudaMalloc(&c->imp_tab, size_t(c->g.batch) * 3 * c->imp_tpitch * c->esz));
                c->imp_fact_valid = false;
            }
        }
        c->scheme = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_ENERGY_DRIFT) {
        if (value < 0 || value > 16) return fail(TSW_ERR_ARG, "energy drift exponent must be 0..16");
        c->en_drift_k = int(value);
        c->en_ref.clear();
        return TSW_OK;
    }
    if (key == TSW_OPT_ENERGY_FUSE) {
        if (value != 0 && value != 1) return fail(TSW_ERR_ARG, "energy fuse must be 0 or 1");
        c->en_fuse = value != 0;
        c->en_level = -1;
        return TSW_OK;
    }
    if (key == TSW_OPT_HALO) {
        if (value != 0 && value != 1) return fail(TSW_ERR_ARG, "halo mode must be 0 (NCCL) or 1 (peer)");
        if (value == 1) {
            if (c->g.dim != 2) return fail(TSW_ERR_ARG, "peer halos are for 2D slabs");
            tsw_status st = set_dev(c);
            if (st) return st;
            if (!c->mbox) {
                CK(cudaMalloc(reinterpret_cast<void**>(&c->mbox), 256));
                CK(cudaMemsetAsync(c->mbox, 0, 256, c->stream));
                CSYNC(c);
            }
        }
        c->halo_mode = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_GUARD_CHECK) {
        if (value != 1) return fail(TSW_ERR_ARG, "guard check: value must be 1");
        tsw_status st = set_dev(c);
        if (st) return st;
        return guard_fill(c);
    }
    if (key == TSW_OPT_IMPLICIT_XROWS) {
        if (value != 1 && value != 2) return fail(TSW_ERR_ARG, "implicit x-solve rows per iteration must be 1 or 2");
        c->imp_x2 = (value == 2) ? 1 : 0;
        return TSW_OK;
    }
    if (key == TSW_OPT_IMPLICIT_SOLVER) {
        if (value < 0 || value > 3)
            return fail(TSW_ERR_ARG, "implicit solver must be 0 (auto), 1 (cyclic reduction), 2 (streaming scans) or 3 (cluster scans)");
        if (value == 1 && c->g.dim == 2) {
            int64_t lim = 1;  // largest 2^q − 1 whose four line arrays fit in 227 KB
            while ((2 * lim + 1) * 4 * int64_t(c->esz) <= 227 * 1024) lim = 2 * lim + 1;
            if (c->g.nx - 2 > lim || c->g.ny - 2 > lim)
                return fail(TSW_ERR_ARG, "cyclic reduction keeps a line in shared memory: at most %lld unknowns per line",
                            (long long)lim);
        }
        c->imp_solver = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_TB_DEPTH) {
        if (!(value == 0 || value == 4 || value == 8 || value == 16))
            return fail(TSW_ERR_ARG, "TB ring depth must be 0 (auto), 4, 8 or 16");
        c->tb_depth = int(value);
        for (auto& r : c->tb_occ)
            for (auto& q : r)
                for (int& o : q) o = 0;
        return TSW_OK;
    }
    if (key == TSW_OPT_TB_WARPS) {
        if (value != 0 && value != 4 && value != 8) return fail(TSW_ERR_ARG, "TB CTA width must be 0 (auto), 4 or 8 warps");
        c->tb_warps = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_ROWS_PER_ITEM) {
        if (value < 0 || value > (1 << 30)) return fail(TSW_ERR_ARG, "rows per item must be >= 0");
        c->rows_per_item_opt = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_KERNEL) {
        if (value != 0 && value != 1) return fail(TSW_ERR_ARG, "kernel must be 0 (TMA pipeline) or 1 (register)");
        c->kernel_opt = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_DEPTH) {
        if (value < 2 || value > 32) return fail(TSW_ERR_ARG, "depth must be in [2, 32]");
        c->depth_opt = int(value);
        return TSW_OK;
    }
    if (key == TSW_OPT_TIME_KERNELS) {
        c->timing = value != 0;
        c->ev_used = 0;
        c->timed_launches = 0;
        c->timed_updates = 0;
        c->timed_meta.clear();
        return TSW_OK;
    }
    return fail(TSW_ERR_ARG, "unknown option %d", key);
}

// ---- peer halo plumbing -------------------------------------------------------------------------
namespace {
struct PeerBlob {
    uint32_t magic;
    int32_t nbuf;   // bit k: buffer k exported
    int64_t ny_local, fshift, mstride, pitch, esz, batch, nx;
    cudaIpcMemHandle_t buf[4];
    cudaIpcMemHandle_t mbox;
};
constexpr uint32_t PEER_MAGIC = 0x74737770u;  // "tswp"

void set_peer(tsw_ctx* c, int side, void* const bufs[4], int64_t ny, int64_t mstride, unsigned int* mbox) {
    for (int k = 0; k < 4; ++k) c->peer_buf[side][k] = bufs[k];
    c->peer_ny[side] = ny;
    c->peer_mstride[side] = mstride;
    // the upper neighbour hears from me (its lower neighbour) in slot 1, the lower one in slot 0
    c->peer_slot[side] = mbox + (side == 0 ? 1 : 0);
}
}  // namespace

tsw_status tsw_peer_export(tsw_ctx* c, void* out, size_t cap, size_t* len) {
    if (!c || !len) return fail(TSW_ERR_ARG, "NULL argument");
    *len = sizeof(PeerBlob);
    if (!out) return TSW_OK;
    if (cap < sizeof(PeerBlob)) return fail(TSW_ERR_ARG, "buffer too small (%zu bytes needed)", sizeof(PeerBlob));
    if (!c->mbox) return fail(TSW_ERR_STATE, "enable peer halos (TSW_OPT_HALO = 1) first");
    tsw_status st = set_dev(c);
    if (st) return st;
    PeerBlob b;
    memset(&b, 0, sizeof(b));
    b.magic = PEER_MAGIC;
    b.ny_local = c->ny_local;
    b.fshift = int64_t(c->fshift);
    b.mstride = c->mstride;
    b.pitch = c->pitch;
    b.esz = c->esz;
    b.batch = c->g.batch;
    b.nx = c->g.nx;
    for (int k = 0; k < 4; ++k)
        if (c->buf[k]) {
            CK(cudaIpcGetMemHandle(&b.buf[k], static_cast<char*>(c->buf[k]) - GUARD - c->fshift));
            b.nbuf |= 1 << k;
        }
    CK(cudaIpcGetMemHandle(&b.mbox, c->mbox));
    memcpy(out, &b, sizeof(b));
    return TSW_OK;
}

tsw_status tsw_peer_import(tsw_ctx* c, int32_t side, const void* blob, size_t len) {
    if (!c || !blob) return fail(TSW_ERR_ARG, "NULL argument");
    if (side != 0 && side != 1) return fail(TSW_ERR_ARG, "side must be 0 (rank−1) or 1 (rank+1)");
    if (len < sizeof(PeerBlob)) return fail(TSW_ERR_ARG, "peer blob too short");
    if (!has_nb(c, side)) return fail(TSW_ERR_ARG, "no neighbour on that side");
    PeerBlob b;
    memcpy(&b, blob, sizeof(b));
    if (b.magic != PEER_MAGIC) return fail(TSW_ERR_ARG, "not a peer blob");
    if (b.pitch != c->pitch || b.esz != int64_t(c->esz) || b.batch != c->g.batch || b.nx != c->g.nx)
        return fail(TSW_ERR_ARG, "peer blob from a ctx of another shape");
    tsw_status st = set_dev(c);
    if (st) return st;
    void* bufs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int k = 0; k < 4; ++k)
        if (b.nbuf & (1 << k)) {
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, b.buf[k], cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(p);
            bufs[k] = static_cast<char*>(p) + GUARD + b.fshift;
        }
    void* pm = nullptr;
    CK(cudaIpcOpenMemHandle(&pm, b.mbox, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(pm);
    set_peer(c, side, bufs, b.ny_local, b.mstride, static_cast<unsigned int*>(pm));
    return TSW_OK;
}

tsw_status tsw_peer_state(tsw_ctx* c, int64_t* out3) {
    if (!c || !out3) return fail(TSW_ERR_ARG, "NULL argument");
    out3[0] = c->epoch;
    out3[1] = out3[2] = out3[3] = -1;
    if (!c->mbox) return TSW_OK;
    tsw_status st = set_dev(c);
    if (st) return st;
    cudaStream_t s;   // a private stream: the ctx stream may be waiting on a neighbour
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned int h[3] = {0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(h, c->mbox, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return fail(TSW_ERR_CUDA, "mailbox read: %s", cudaGetErrorString(e));
    out3[1] = h[0];
    out3[2] = h[1];
    out3[3] = h[2];
    return TSW_OK;
}

tsw_status tsw_peer_attach(tsw_ctx* c, int32_t side, tsw_ctx* other) {
    if (!c || !other) return fail(TSW_ERR_ARG, "NULL argument");
    if (side != 0 && side != 1) return fail(TSW_ERR_ARG, "side must be 0 (rank−1) or 1 (rank+1)");
    if (!has_nb(c, side)) return fail(TSW_ERR_ARG, "no neighbour on that side");
    if (!other->mbox) return fail(TSW_ERR_STATE, "enable peer halos (TSW_OPT_HALO = 1) on the neighbour first");
    if (other->pitch != c->pitch || other->esz != c->esz || other->g.batch != c->g.batch || other->g.nx != c->g.nx)
        return fail(TSW_ERR_ARG, "neighbour ctx of another shape");
    void* bufs[4];
    for (int k = 0; k < 4; ++k) bufs[k] = other->buf[k];
    set_peer(c, side, bufs, other->ny_local, other->mstride, other->mbox);
    return TSW_OK;
}

// ---- out-of-bounds write check ----------------------------------------------------------------
namespace {
// (raw pointer, payload bytes) of every guarded array the ctx holds
std::vector<std::pair<char*, size_t>> ctx_guarded(tsw_ctx* c) {
    std::vector<std::pair<char*, size_t>> out;
    auto add = [&](void* p, size_t shift) {
        if (!p) return;
        char* raw = static_cast<char*>(p) - GUARD - shift;
        std::lock_guard<std::mutex> lk(guard_mu());
        auto it = guard_reg().find(raw);
        if (it != guard_reg().end()) out.emplace_back(raw, it->second);
    };
    for (int k = 0; k < 4; ++k) add(c->buf[k], c->fshift);
    add(c->imp_s1, c->fshift);
    add(c->h1, c->cshift_h);
    add(c->h2, c->cshift_h);
    add(c->c1, c->cshift);
    add(c->c2, c->cshift);
    return out;
}
}  // namespace

tsw_status guard_fill(tsw_ctx* c) {
    for (auto& g : ctx_guarded(c)) {
        CK(cudaMemsetAsync(g.first, 0xFF, GUARD, c->stream));
        CK(cudaMemsetAsync(g.first + GUARD + g.second, 0xFF, GUARD, c->stream));
    }
    CSYNC(c);
    return TSW_OK;
}

tsw_status tsw_check_guards(tsw_ctx* c, int64_t* bad_bytes, int64_t* checked_bytes) {
    if (!c || !bad_bytes) return fail(TSW_ERR_ARG, "NULL argument");
    tsw_status st = set_dev(c);
    if (st) return st;
    CSYNC(c);
    std::vector<unsigned char> h(GUARD);
    int64_t bad = 0, checked = 0;
    for (auto& g : ctx_guarded(c)) {
        checked += 2 * int64_t(GUARD);
        for (int side = 0; side < 2; ++side) {
            CK(cudaMemcpyAsync(h.data(), side ? g.first + GUARD + g.second : g.first, GUARD, cudaMemcpyDeviceToHost,
                               c->stream));
            CSYNC(c);
            for (unsigned char v : h) bad += (v != 0xFF);
        }
    }
    *bad_bytes = bad;
    if (checked_bytes) *checked_bytes = checked;
    return TSW_OK;
}

tsw_status tsw_kernel_stats(tsw_ctx* c, double* total_ms, int64_t* launches, int64_t* updates) {
    if (!c) return fail(TSW_ERR_ARG, "NULL ctx");
    tsw_status st = set_dev(c);
    if (st) return st;
    CSYNC(c);
    double ms = 0.0;
    for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
        float m = 0.f;
        CK(cudaEventElapsedTime(&m, c->ev_pool[k], c->ev_pool[k + 1]));
        ms += m;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = c->timed_launches;
    if (updates) *updates = c->timed_updates;
    return TSW_OK;
}

tsw_status tsw_kernel_launches(tsw_ctx* c, int64_t cap, double* ms, int32_t* levels, int64_t* updates,
                               int64_t* count) {
    if (!c || cap < 0 || (cap > 0 && (!ms || !levels || !updates))) return fail(TSW_ERR_ARG, "bad arguments");
    tsw_status st = set_dev(c);
    if (st) return st;
    CSYNC(c);
    const int64_t n = int64_t(c->timed_meta.size());
    for (int64_t k = 0; k < std::min(n, cap); ++k) {
        float m = 0.f;
        CK(cudaEventElapsedTime(&m, c->ev_pool[2 * k], c->ev_pool[2 * k + 1]));
        ms[k] = m;
        levels[k] = c->timed_meta[k].first;
        updates[k] = c->timed_meta[k].second;
    }
    if (count) *count = n;
    return TSW_OK;
}

tsw_status tsw_alu_probe(int device, int dtype, double* ops_per_s) {
    if (!ops_per_s || (dtype != TSW_F32 && dtype != TSW_F64)) return fail(TSW_ERR_ARG, "bad arguments");
    return dtype == TSW_F64 ? alu_probe_t<double>(device, ops_per_s) : alu_probe_t<float>(device, ops_per_s);
}

tsw_status tsw_nccl_unique_id(void* out) {
    if (!out) return fail(TSW_ERR_ARG, "NULL argument");
    Nccl& N = nccl();
    if (!N.ok) return fail(TSW_ERR_NCCL, "libnccl.so.2 not found or incomplete");
    NcclId id;
    NK(N.GetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return TSW_OK;
}

tsw_status tsw_nccl_init(tsw_ctx* c, const void* uid) {
    if (!c || !uid) return fail(TSW_ERR_ARG, "NULL argument");
    Nccl& N = nccl();
    if (!N.ok) return fail(TSW_ERR_NCCL, "libnccl.so.2 not found or incomplete");
    tsw_status st = set_dev(c);
    if (st) return st;
    if (c->comm) return fail(TSW_ERR_STATE, "NCCL communicator already initialised");
    NcclId id;
    memcpy(&id, uid, sizeof(id));
    void* comm = nullptr;
    NK(N.CommInitRank(&comm, c->g.nranks, id, c->g.rank));
    c->comm = comm;
    return TSW_OK;
}

}  // extern "C"
