/*
 * include/tsw.h — C ABI of the B200-native leapfrog solver for the regularised tsunami equation
 * (arXiv 2005.11931, "Tsunami propagation for singular topographies").
 *
 * The hot path (BASELINE.json north_star): explicit second-order leapfrog time stepping of
 *     u_tt = Σ_j ∂_j( h_{j,ε}(x) ∂_j u )                    PAPER.md §2, eq. (Equation)
 * with u(0) = u0, u_t(0) = u1, homogeneous Dirichlet boundary (§3.3), on a
 * 1D or 2D uniform grid, where the singular depth is replaced by the mollified family
 * h_ε = h * φ_ε, φ_ε(x) = ε⁻¹ φ(x/ε), φ(x) = c·exp(1/(x²−1)) on |x| < 1,
 * δ ↦ φ_ε, δ² ↦ φ_ε².  Readings of the paper: DESIGN.md §3 (R1–R25).
 *
 * Conventions (all calls):
 *  - Every function returns tsw_status; no C++ exception or longjmp crosses this ABI.  On error
 *    the ctx is unchanged (arguments are validated before any device work) and
 *    tsw_last_error(ctx) returns a message (thread-local; ctx may be NULL after tsw_create).
 *  - Grid (R9): nx, ny count GLOBAL nodes including the Dirichlet boundary nodes.  Node i of an
 *    n-node axis is at ((2i + 1 − n)·d)/2 (a centred grid), face i+1/2 at ((2i + 2 − n)·d)/2.
 *  - Field layout seen by the caller: [batch][ny_local][nx] row-major, x fastest, in the ctx
 *    dtype (float or double), where ny_local is this rank's slab height (ny if nranks == 1;
 *    1 if dim == 1).  Internally rows are padded and carry one ghost row above and below.
 *  - Host buffers are only read/written during the call (copied); device buffers passed with
 *    on_device = 1 must be valid device pointers of the ctx's device and are read during the
 *    call (stream-ordered on the ctx stream).  The ctx owns all of its device memory.
 *  - Asynchrony: tsw_step is asynchronous on the ctx stream.  tsw_energy, tsw_wave2, tsw_read
 *    (to host), tsw_info and tsw_sync synchronise the ctx stream.
 *  - Threads: one ctx per host thread at a time.  Different ctxs are independent.
 *  - There is no CPU fallback: without a CUDA device tsw_create fails with TSW_ERR_CUDA.
 */
#ifndef TSW_H
#define TSW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsw_ctx tsw_ctx; /* opaque */

typedef enum {
    TSW_OK = 0,
    TSW_ERR_ARG = 1,      /* invalid argument (sizes, ε ∉ (0,1], h < c0, dt ≤ 0, …) */
    TSW_ERR_CFL = 2,      /* dt above the Gershgorin leapfrog bound (R16) */
    TSW_ERR_STATE = 3,    /* call out of order (e.g. step before set_initial, energy at n = 0) */
    TSW_ERR_CUDA = 4,     /* CUDA runtime error or no device */
    TSW_ERR_NCCL = 5,     /* NCCL unavailable or failed */
    TSW_ERR_OOM = 6,      /* device allocation failed */
    TSW_ERR_UNSTABLE = 7  /* tsw_energy: non-finite energy, or drift beyond TSW_OPT_ENERGY_DRIFT (blow-up) */
} tsw_status;

typedef enum { TSW_F32 = 0, TSW_F64 = 1 } tsw_dtype;

/* Depth kinds (§3.1 Cases; R5–R8). */
typedef enum {
    TSW_H_CONST = 0,        /* h1 = h2 = h_b */
    TSW_H_DELTA_LINE_X = 1, /* h1 = h_b + A·φ_ε(x − xs)^order, h2 = h_b  (δ-line along x = xs; 1D: δ-point) */
    TSW_H_DELTA_POINT = 2,  /* h1 = h2 = h_b + A·(φ_ε(x − xs)·φ_ε(y − ys))^order  (tensor mollifier, R3) */
    TSW_H_FACES = 3,        /* dense caller-given faces (tsw_set_coeff_faces) */
    TSW_H_PROFILE_X = 4     /* x-only profile: segments + singular terms (tsw_set_coeff_profile) */
} tsw_hkind;

/* tsw_set_initial flags */
#define TSW_ALLOW_UNSTABLE 1u /* skip the CFL check */
#define TSW_INIT_SHARED 2u    /* u0/u1 are ONE [ny_local][nx] field used by every member */

typedef struct {
    int32_t dim;          /* 1 or 2 */
    int64_t nx, ny;       /* global node counts incl. boundary; nx ≥ 3; ny ≥ 3 (2D) or 1 (1D) */
    double dx, dy;        /* grid steps > 0 (dy ignored in 1D) */
    int32_t batch;        /* B ≥ 1 members (an ε-family, §2 very weak solution net P:385–403) */
    int32_t dtype;        /* tsw_dtype: working precision T of the fields and prescaled coefficients */
    int32_t rank, nranks; /* row-slab decomposition along y (2D only); nranks = 1 ⇒ single GPU */
    int32_t device;       /* CUDA device ordinal; −1 ⇒ the calling thread's current device */
    void* stream;         /* cudaStream_t to run on, or NULL ⇒ the ctx creates its own stream */
} tsw_grid_desc;

typedef struct {
    int32_t kind;                 /* tsw_hkind (not TSW_H_FACES) */
    int32_t order;                /* 1: φ_ε (δ) ; 2: φ_ε² (δ²) */
    double h_background;          /* h_b ≥ c0 > 0 (positivity) */
    double amp;                   /* A ≥ 0 (A = 0 ⇒ background member) */
    double xs, ys;                /* singular point / line location */
    const double* eps;            /* [batch] host array, each ε ∈ (0, 1] */
    const double* amp_per_member; /* optional [batch] host array overriding amp, or NULL */
} tsw_coeff_desc;

/* Create a solver context: validates the grid, allocates the two time levels on the device.
 * Errors: TSW_ERR_ARG (bad sizes / rank), TSW_ERR_CUDA (no device), TSW_ERR_OOM. */
tsw_status tsw_create(const tsw_grid_desc* grid, tsw_ctx** out);

/* Free all device memory and the NCCL communicator owned by ctx.  NULL is a no-op. */
void tsw_destroy(tsw_ctx* ctx);

/* S1 coefficient builder (§2 h_{i,ε} = h_i * ψ_ε; §3.1): evaluates
 * h_ε in fp64 on the device at every half-grid face of this rank's slab (R2).  Validates
 * h_b > 0, A ≥ 0, ε ∈ (0, 1], order ∈ {1, 2}.  Prescaling to T happens in tsw_set_initial. */
tsw_status tsw_set_coeff(tsw_ctx* ctx, const tsw_coeff_desc* h);

/* Piecewise-constant depth in x with singular terms — the paper's own scenarios (§3.1
 * Case 1 eq. (h2case): h_0 = 100 on [0,75), 10 on [75,100]; Cases 2–3 P:773–789:
 * h_0 + δ(x−70), h_0 + δ²(x−70); §3.2.3: 100δ, 100δ²; 2D H(x,y) = h_0(x)):
 *   h_ε(x) = v_0 + Σ_k (v_k − v_{k−1})·Φ((x − b_k)/ε) + Σ_j s_b·A_j·φ_ε(x − x_j)^{o_j}
 * with Φ(t) = ∫_{−1}^{t} φ, the mollifier's primitive (convolution of a step with φ_ε).  h1 is
 * evaluated at the x faces; h2 (2D) at the node columns, including the singular terms when
 * isotropic (scalar depth H) and the segments only otherwise.  Coordinates follow the centred
 * grid of R9 (the paper's [0, 100] is x + 50 there). */
typedef struct {
    int32_t nseg;              /* 1..64 constant segments */
    const double* seg_value;   /* [nseg] depths v_k > 0 */
    const double* seg_break;   /* [nseg−1] increasing breaks b_1 < …; segment k = [b_k, b_{k+1}) */
    int32_t nsing;             /* 0..64 singular terms */
    const double* sing_loc;    /* [nsing] x_j */
    const double* sing_amp;    /* [nsing] A_j ≥ 0 */
    const int32_t* sing_order; /* [nsing] 1 (δ ↦ φ_ε) or 2 (δ² ↦ φ_ε²) */
    int32_t isotropic;         /* 2D: 1 ⇒ scalar depth (h2 = h1 profile); 0 ⇒ h2 = segments only */
} tsw_profile_desc;

/* Builds the faces of an x-only profile for every member b with ε = eps[b] (host [batch], each in
 * (0, 1]) and singular amplitudes scaled by scale[b] (host [batch] ≥ 0, NULL ⇒ 1; 0 gives the
 * background member of A₂).  A₂'s reference point xs becomes the first singular location (else
 * the first break).  Errors: TSW_ERR_ARG. */
tsw_status tsw_set_coeff_profile(tsw_ctx* ctx, const tsw_profile_desc* p, const double* eps, const double* scale);

/* Dense override of the fp64 faces (kind TSW_H_FACES), host (on_device = 0) or device pointers:
 *   h1 [batch][ny_local][nx−1]   face (i+1/2, j) of local row j
 *   h2 [batch][ny_local+1][nx]   row k = face (i, g+1/2) with g = (first global row of the slab) + k − 1;
 *                                rows outside the global grid are ignored (2D only; NULL in 1D).
 * Values must be > 0 where used. */
tsw_status tsw_set_coeff_faces(tsw_ctx* ctx, const double* h1, const double* h2, int on_device);

/* Copy the fp64 faces h_ε the stepper uses (after tsw_set_coeff or tsw_set_coeff_faces) to host
 * arrays in the tsw_set_coeff_faces layout (h1 [batch][ny_local][nx−1]; h2 [batch][ny_local+1][nx],
 * rows outside the global grid written as 0; h2 may be NULL; 1D: h1 [batch][nx−1]).  Synchronises. */
tsw_status tsw_read_faces(tsw_ctx* ctx, double* h1, double* h2);

/* Set u(0) = u0 and u_t(0) = u1, the time step dt, and reset n = 0.
 *   u0, u1: [batch][ny_local][nx] in the ctx dtype (or [ny_local][nx] with TSW_INIT_SHARED);
 *           u1 may be NULL (⇒ 0).  Boundary entries are ignored and forced to +0 (R10).
 * Prescales c = fl_T((dt²/d²)·h) (R19) and checks dt ≤ 2/√ρ_G (R16) unless TSW_ALLOW_UNSTABLE.
 * Errors: TSW_ERR_STATE (no coefficients), TSW_ERR_ARG (dt ≤ 0), TSW_ERR_CFL. */
tsw_status tsw_set_initial(tsw_ctx* ctx, const void* u0, const void* u1, double dt, int on_device,
                           uint32_t flags);

/* Advance nsteps ≥ 0 time levels (asynchronous).  From n = 0 the first level is the Taylor start
 * u¹ = (u⁰ + dt·u₁) + ½L(u⁰) (R11); every later level is leapfrog
 * u^{n+1} = (2u^n − u^{n−1}) + L(u^n) with the canonical contraction-free operator of DESIGN.md §2.
 * With nranks > 1 each level is followed by the ghost-row exchange.  Errors: TSW_ERR_STATE. */
tsw_status tsw_step(tsw_ctx* ctx, int64_t nsteps);

/* Loopback slabs on ONE device: advance ctxs[0..n−1] (ranks 0..n−1 of one decomposition, same
 * device and stream, no NCCL; 1 ≤ n ≤ 64) by nsteps.  Each level / pass runs the same per-rank
 * phases as tsw_step's NCCL path (boundary rows, exchange on the aux stream after their event,
 * interior rows, wait) with device copies in place of the NCCL messages; with peer halos
 * (TSW_OPT_HALO = 1) the ranks' operations are issued epoch by epoch.  Test and emulation path for
 * the multi-GPU decomposition.  Errors: TSW_ERR_ARG (group shape), TSW_ERR_STATE. */
tsw_status tsw_group_step(tsw_ctx** ctxs, int32_t n, int64_t nsteps);

/* S5 discrete energy E^{n−1/2} of the current levels (R17; discrete form of CL-01):
 *   E = (dx·dy/dt²)·[Σ_interior (u^n − u^{n−1})² + Σ_faces c·(Δu^n)(Δu^{n−1})]   (1D: dx/dt²)
 * accumulated in fp64 with the stepper's own rounded c; summed over ranks (NCCL) when nranks > 1
 * and tsw_nccl_init was called (a loopback-group member returns its slab's share).  When the last
 * temporally blocked pass of the preceding tsw_step produced this level (TSW_OPT_ENERGY_FUSE), the
 * value it reduced in the node form Σ(u^n − u^{n−1})² − Σ u^n·L(u^{n−1}) (the same bilinear form
 * by summation by parts, reading R30) is returned without another pass over the fields.
 *   out_B: host double[batch].  Errors: TSW_ERR_STATE if n < 1; TSW_ERR_UNSTABLE (values still
 *   written) on a non-finite energy or a drift beyond TSW_OPT_ENERGY_DRIFT; TSW_ERR_NCCL when the
 *   communicator reports an asynchronous error (it is aborted). */
tsw_status tsw_energy(tsw_ctx* ctx, double* out_B);

/* S6 second-wave amplitude (R18; §3.2.3, qualitative): for every member b
 *   A₂⁺ = max, A₂⁻ = min over nodes with x_i ≤ xs − ε_b of fl_T(u_b − u_{bg_member})
 * with the global row-major index (g·nx + i) of the first extremum; empty region ⇒ 0 and −1.
 * Reduced over ranks with NCCL when a communicator exists (else this slab's extrema).
 *   out_B2: host double[batch][2]; argidx_B2: host int64[batch][2] (may be NULL). */
tsw_status tsw_wave2(tsw_ctx* ctx, int32_t bg_member, double* out_B2, int64_t* argidx_B2);

/* ---- ε-family diagnostics -------------------------------------------- */

/* Pairwise L² distances of the members at the current level (§3.2.1, P:831–838:
 * ‖u_{ε1}(t,·) − u_{ε2}(t,·)‖_{L²}, the ε → 0 limit study of the very weak solution net):
 *   out_BB[i][j] = sqrt(dx·dy · Σ_nodes (u_i − u_j)²)   (1D: dx), symmetric, zero diagonal,
 * summed over ranks.  out_BB: host double[batch][batch]; batch ≤ 200.  Synchronises. */
tsw_status tsw_family_l2(tsw_ctx* ctx, double* out_BB);

/* The L² quantities of Theorem "lem 1" (energy estimate) at the current level:
 * out_B4[b] = { ‖u^n‖, ‖(u^n − u^{n−1})/dt‖ (0 at n = 0), ‖∂x u^n‖, ‖∂y u^n‖ } with forward
 * differences over all faces and the rectangle rule (weight dx·dy; 1D: dx).  Synchronises. */
tsw_status tsw_field_norms(tsw_ctx* ctx, double* out_B4);

/* W^{1,∞} norms of the regularised depth (Assumption eq. (assum coeff), P:344–345:
 * ‖h_ε‖_{W^{1,∞}} ≲ ε^{−N0}): out_B3[b] = { sup |h1| over the x faces, sup |∇h_ε| at the x faces
 * (analytic derivative of the regulariser for the δ-line, δ-point and profile kinds; a finite
 * difference of the faces for TSW_H_FACES), sup |h2| over the y faces (0 in 1D) }.  Synchronises. */
tsw_status tsw_coeff_norms(tsw_ctx* ctx, double* out_B3);

/* Copy a level of this rank's slab out: which = 0 ⇒ u^n, 1 ⇒ u^{n−1}; dst is [batch][ny_local][nx]
 * in the ctx dtype, host (to_device = 0, synchronous) or device (to_device = 1, stream-ordered). */
tsw_status tsw_read(tsw_ctx* ctx, int32_t which, void* dst, int32_t to_device);

/* Resume from a saved state: un = u^n, unm1 = u^{n−1} (layout as tsw_read), level n ≥ 1 and dt.
 * Coefficients must be set; they are prescaled with this dt.  Boundary entries forced to +0. */
tsw_status tsw_set_state(tsw_ctx* ctx, const void* un, const void* unm1, int64_t n, double dt,
                         int32_t on_device, uint32_t flags);

/* Current level n, time t = n·dt, and the Gershgorin bound 2/√ρ_G of the current coefficients
 * (0 if unknown).  Any pointer may be NULL.  Synchronises. */
tsw_status tsw_info(tsw_ctx* ctx, int64_t* n, double* t, double* dt_max);

/* Block until the ctx stream is idle. */
tsw_status tsw_sync(tsw_ctx* ctx);

/* Number of kernels this ctx has launched so far (the bench's gpu_launches evidence). */
int64_t tsw_launch_count(const tsw_ctx* ctx);

/* Options: TSW_OPT_ROWS_PER_ITEM — rows per warp work item of the 2D stencil (≥ 1; 0 = auto);
 *          TSW_OPT_KERNEL / TSW_OPT_DEPTH — stencil variant and its ring depth;
 *          TSW_OPT_TIME_KERNELS — 1: bracket every stencil launch (leapfrog) or every y-line
 *          solve launch k_imp_yc (implicit scan solver, the dominant kernel of a level) with CUDA
 *          events on the ctx stream (for tsw_kernel_stats), 0: off; setting it resets the
 *          statistics. */
#define TSW_OPT_ROWS_PER_ITEM 1
#define TSW_OPT_TIME_KERNELS 2
#define TSW_OPT_KERNEL 3 /* 0: CTA-wide TMA bulk-copy row pipeline (default); 1: register-prefetch kernel */
#define TSW_OPT_DEPTH 4  /* TMA ring stages per CTA, 2..32 (default 4) */
#define TSW_OPT_GRAPHS 5 /* 1 (default): single-rank steps replay a CUDA graph of two levels; 0: plain launches */
#define TSW_OPT_TBLOCK 6 /* K ∈ {1,…,10}: levels per HBM pass of the temporally blocked stencil
                            (2D, δ-line / constant / profile kinds; slabs use K-deep ghost rows;
                            allocates two more levels; results are bitwise those of K = 1).  A
                            tsw_step call's remainder of r levels (2 ≤ r < K) runs as one pass of
                            depth r.  Default 1. */
#define TSW_OPT_TB_DEPTH 7 /* input ring stages of the temporally blocked stencil: 4, 8 or 16; 0 (default):
                              8 for the one-CTA-per-SM variants (the 12-warp fp64 passes), else 4 */
#define TSW_OPT_SCHEME 8   /* 0 (default): explicit leapfrog (north_star).  1: the paper's implicit method
                              (§3.3, reading R26): factorised three-level Crank–Nicolson
                              (I − ½L_x)(I − ½L_y)(u^{n+1} + u^{n−1}) = 2u^n, start u¹ = B⁻¹u⁰ + dt·u₁ (R27),
                              line solves (2D) by the scan solvers of TSW_OPT_IMPLICIT_SOLVER, (1D)
                              Thomas; unconditionally stable (no CFL check).  Single rank, δ-line /
                              constant / profile kinds (x-only coefficients), ≤ 8192 unknowns per line. */
#define TSW_OPT_IMPLICIT_SOLVER 9 /* 2D line solves of the implicit scheme.  Scans (reading R28): x lines
                              share one matrix, whose LU is applied as two affine scans per row; y
                              lines are Toeplitz per column and solved by the closed form
                              T⁻¹ = κ⁻¹[(I − ρS)(I − ρSᵀ) + ρ²e₁e₁ᵀ]⁻¹ (exponential scans + a rank-one
                              correction), fused with the three-level update.  The y solve runs either
                              in thread-block clusters holding the columns on chip (3: 5 words per node
                              and level) or as three barrier-free streaming kernels (2: z read twice).
                              0 (default): auto — 2 for fp64 grids of ≥ 8 M nodes, else 3.
                              1: cyclic reduction per line in shared memory with tiled transposes
                              (the paper's solver), ≤ 4095 (fp64) / 8191 (fp32) unknowns per line. */
#define TSW_OPT_TB_WARPS 13 /* CTA width of the temporally blocked stencil: 8 = the wide CTA (8 warps,
                              512-column strips, two CTAs per SM; fp64 passes of depth ≥ 7: 12 warps,
                              768-column strips, one CTA per SM), 4 (256-column strips: less redundant
                              halo work on narrow grids), 0 (default): 4 where its strips compute ≥ 5 %
                              fewer columns, and for a slab's launch of its first / last K rows; else
                              the wide CTA */
#define TSW_OPT_ENERGY_FUSE 14 /* 1 (default): on a single-rank 2D temporally blocked run, the last pass of
                              every tsw_step call also reduces the discrete energy of the two levels it
                              writes (S5 fused into S3 in the node form of reading R30: per-item fp64
                              partials, summed in a fixed order by one small kernel); tsw_energy at that
                              level then only reads the result.  0: tsw_energy always runs the
                              standalone kernel */
#define TSW_OPT_ENERGY_DRIFT 15 /* blow-up detection in tsw_energy: k (default 2) — TSW_ERR_UNSTABLE
                              when the energy is non-finite or has drifted from the first energy measured
                              after tsw_set_initial / tsw_set_state by more than 10^−k relative (R17: the
                              scheme conserves it to round-off while stable; above the CFL bound it grows
                              without limit).  0: only the finiteness check.  The energies are still
                              written to out_B.  Checked on the whole grid's energy (nranks = 1, or a
                              communicator); a slab's share is not conserved */
#define TSW_OPT_IMPLICIT_XROWS 12 /* rows per iteration of the implicit x-line solve: 1 (default; LU tables
                              in registers) or 2 (the two rows' scan chains interleave, tables in shared
                              memory — measured 4 % slower at 4096², kept for comparison) */
#define TSW_OPT_HALO 11     /* ghost rows of 2D slabs.  0 (default): NCCL send/recv (tsw_nccl_init).
                              1: peer stores — the temporally blocked stencil writes its first / last K
                              owned rows straight into the neighbours' ghost rows through mapped peer
                              pointers (NVLink), one-level steps and initial ghosts are pushed by a copy
                              kernel; ordering by epochs: before halo operation e each rank's stream
                              runs a one-thread waiter until both neighbours have published e − 1 into
                              its mailbox (bounded: a ~20 s timeout sets an error word that tsw_read /
                              tsw_energy report), and afterwards publishes e.  Neighbours are mapped
                              with tsw_peer_export / tsw_peer_import (processes, CUDA IPC — one GPU per
                              rank) or tsw_peer_attach (ctxs of one process, stepped together by
                              tsw_group_step on one shared stream, epoch by epoch, so no waiter ever
                              spins), after TSW_OPT_TBLOCK and before tsw_set_initial.  tsw_set_initial
                              / tsw_set_state are one epoch; the ghost rows are pushed by the first
                              stepping call.  tsw_energy / tsw_field_norms return this slab's share
                              and are collective: every rank calls them in the same order (after a
                              step). */
#define TSW_OPT_GUARD_CHECK 10 /* 1: fill the 16 KB guard zones before and after every device array the ctx
                              holds so far (fields, scratch, faces, coefficients) with 0xFF bytes (NaN in
                              both precisions, so a stray read shows up in results too); synchronises.
                              A debugging aid: tsw_check_guards then counts guard bytes that changed. */
tsw_status tsw_set_option(tsw_ctx* ctx, int32_t key, int64_t value);

/* Peer halo plumbing (TSW_OPT_HALO = 1).  tsw_peer_export writes an opaque blob
 * (*len bytes; call with out = NULL to get the size) holding CUDA IPC handles of this ctx's field
 * buffers and mailbox; the neighbour passes it to tsw_peer_import(ctx, side, …) with side 0 for
 * rank − 1 and 1 for rank + 1 (the same blob bytes, any transport — e.g. an all-gather).  For ctxs
 * of one process, tsw_peer_attach(ctx, side, neighbour_ctx) maps directly.  Shapes must agree. */
tsw_status tsw_peer_export(tsw_ctx* ctx, void* out, size_t cap, size_t* len);
tsw_status tsw_peer_import(tsw_ctx* ctx, int32_t side, const void* blob, size_t len);
tsw_status tsw_peer_attach(tsw_ctx* ctx, int32_t side, tsw_ctx* neighbour);
/* Peer halos, host-driven lock step: issue exactly ONE halo operation (epoch) of the next
 * min(nsteps, …) levels — the ghost push, one level or one temporally blocked pass — and report
 * the levels it advanced in *consumed (0 for a ghost push).  Ranks sharing a GPU can then be
 * stepped operation by operation with a host barrier in between, so no waiter ever spins. */
tsw_status tsw_step_op(tsw_ctx* ctx, int64_t nsteps, int64_t* consumed);

/* Diagnostics: out4 = {halo epochs issued, mailbox from rank − 1, mailbox from rank + 1, wait
 * timeout word} (the mailboxes read on a private stream; −1 without peer halos). */
tsw_status tsw_peer_state(tsw_ctx* ctx, int64_t* out4);

/* Out-of-bounds write check: *bad_bytes = number of guard bytes (TSW_OPT_GUARD_CHECK) that no
 * longer hold 0xFF — any nonzero count is a kernel writing outside its array; *checked_bytes (may
 * be NULL) = guard bytes inspected.  Synchronises. */
tsw_status tsw_check_guards(tsw_ctx* ctx, int64_t* bad_bytes, int64_t* checked_bytes);

/* Live per-kernel timing of the launches TSW_OPT_TIME_KERNELS brackets (stencil S2/S3, or the
 * implicit y solve) since it was set: total device milliseconds, number of launches, and interior
 * point-updates they performed.
 * Synchronises.  Any pointer may be NULL. */
tsw_status tsw_kernel_stats(tsw_ctx* ctx, double* total_ms, int64_t* launches, int64_t* updates);

/* Per-launch view of the same timed launches: for launch k < min(count, cap), its device
 * milliseconds ms[k], the levels it advanced levels[k] (K for a temporally blocked pass, 1 for a
 * one-level step) and its interior point-updates updates[k]; *count = number of timed launches.
 * cap = 0 only queries the count.  Synchronises. */
tsw_status tsw_kernel_launches(tsw_ctx* ctx, int64_t cap, double* ms, int32_t* levels, int64_t* updates,
                               int64_t* count);

/* Measurement helper for the roofline (not a paper operation): the device's non-contracted
 * add/multiply throughput in the given dtype (TSW_F64 / TSW_F32), operations per second, from a
 * kernel of independent (x + b)·a − b chains (two adds per multiply, the stencil's mix) on every
 * SM; best of three timed launches after a warm-up.  Allocates and frees its own memory. */
tsw_status tsw_alu_probe(int device, int dtype, double* ops_per_s);

/* NCCL row-slab plumbing.  tsw_nccl_unique_id writes a 128-byte ncclUniqueId
 * (call on rank 0, broadcast it, e.g. with torch.distributed); tsw_nccl_init creates the ctx's
 * communicator over grid.nranks ranks.  libnccl.so.2 is resolved at run time. */
tsw_status tsw_nccl_unique_id(void* out_128B);
tsw_status tsw_nccl_init(tsw_ctx* ctx, const void* unique_id_128B);

/* Message of the last failing call on this thread (never NULL). */
const char* tsw_last_error(const tsw_ctx* ctx);

/* Library version string. */
const char* tsw_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TSW_H */
