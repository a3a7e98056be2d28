/*
 * oracle/tsw_oracle.c — the CPU ORACLE for the leapfrog hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2005_11931_b200/) never imports, links or executes it,
 * and it shares no code, header, table or constant generator with the CUDA
 * path: everything below is written out from PAPER.md and the readings listed
 * in DESIGN.md §3 (R-numbers).
 *
 * Plain, slow, obviously correct.  Build: gcc -O2 -ffp-contract=off (no FMA
 * contraction, no -ffast-math, no FTZ/DAZ) so every + − × below is one
 * IEEE-754 round-to-nearest operation in the stated type.  OpenMP splits
 * rows only; each node's arithmetic is independent of the thread count.
 *
 * Grid (R9): node i of an n-node axis sits at ((2i + 1 − n)·d)/2, face i+1/2
 * at ((2i + 2 − n)·d)/2 (integer × d, halved: exact mirror antisymmetry).
 * Arrays are row-major [ny][nx]; face arrays:
 *   h1/c1 [ny][nx−1]   face (i+1/2, j)  — x faces   (1D: [nx−1])
 *   h2/c2 [ny−1][nx]   face (i, j+1/2)  — y faces
 * A "window" run updates nodes 1..wnx−2 × 1..wny−2 and leaves the outer ring
 * as given: on the full grid that ring is the Dirichlet boundary (P:1129–1133,
 * R10); on a sub-window it is a fixed edge whose error travels one node per
 * step, so the window centre is exact while the window half-width exceeds the
 * step count (SURVEY §8(c) "exact lattice speed").
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py,
 * tests/test_scenarios_pins.py and tests/test_implicit_pins.py (closed forms, invariants, brute
 * force, the paper's constant c).  The wave2 diagnostic's definition (R18) has no value printed
 * in the paper; it is pinned by brute-force max/min, A = 0 ⇒ 0, Born linearity, and two closed
 * forms: the impedance-mismatch reflection coefficient R = (√h1 − √h2)/(√h1 + √h2) of the paper's
 * Case-1 jump and the thin-layer limit (Δ/2)·∂f of the δ-line.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* PAPER.md §3.1: "c ≃ 2.2523 to get ∫φ = 1".  R4: the value of
 * 1/∫_{−1}^{1} exp(1/(x²−1)) dx to double precision is 2.252283621043581010…;
 * tests pin it against a 40-digit mpmath quadrature and the paper's 2.2523. */
static const double ORACLE_MOLLIFIER_C = 2.252283621043581;

double tswo_mollifier_c(void) { return ORACLE_MOLLIFIER_C; }

void tswo_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int tswo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* PAPER.md §3.1: φ_ε(x) = ε^{-1} φ(x/ε), φ(x) = c·exp(1/(x²−1)) for
 * |x| < 1 and 0 otherwise.  The support test is on t = d/ε (reading R25 in
 * |t| < 1 in fp64; |t| == 1 gives exactly 0). */
double tswo_phi_eps(double d, double eps) {
    double t = d / eps;
    if (!(fabs(t) < 1.0)) return 0.0;
    return (ORACLE_MOLLIFIER_C / eps) * exp(1.0 / (t * t - 1.0));
}

void tswo_phi_eps_array(const double* d, int64_t n, double eps, double* out) {
    for (int64_t k = 0; k < n; ++k) out[k] = tswo_phi_eps(d[k], eps);
}

static double node_x(int64_t i, int64_t n, double d) { return ((double)(2 * i + 1 - n) * d) / 2.0; }
static double face_x(int64_t i, int64_t n, double d) { return ((double)(2 * i + 2 - n) * d) / 2.0; }

/* Regularised depth at one face (P:325–337 h_ε = h * ψ_ε; P:775–789 Cases 2/3;
 * R5/R6/R8).  kind: 0 const, 1 δ-line along x = xs (h1 only), 2 δ-point at
 * (xs, ys) with the tensor-product mollifier φ_ε(x)φ_ε(y) (R3).
 * which: 1 = x face (i+1/2, j), 2 = y face (i, j+1/2). */
static double depth_at_face(int kind, int order, double hb, double amp, double xs, double ys,
                            double eps, int64_t nx, int64_t ny, double dx, double dy,
                            int which, int64_t i, int64_t j) {
    double bump;
    if (kind == 0) return hb;
    if (kind == 1) {
        if (which == 2) return hb;               /* R6: h_2 ≡ h_b */
        bump = tswo_phi_eps(face_x(i, nx, dx) - xs, eps);
    } else if (kind == 2) {
        double x = (which == 1) ? face_x(i, nx, dx) : node_x(i, nx, dx);
        double y = (which == 1) ? node_x(j, ny, dy) : face_x(j, ny, dy);
        bump = tswo_phi_eps(x - xs, eps) * tswo_phi_eps(y - ys, eps);
    } else {
        return NAN;
    }
    if (order == 2) bump = bump * bump;          /* P:787 δ² ↦ φ_ε² */
    return hb + amp * bump;
}

/* Face arrays of the window whose node (0,0) is global node (i0, j0), size
 * wnx × wny nodes.  h1: [wny][wnx−1], h2: [wny−1][wnx] (NULL / ignored in 1D). */
int tswo_build_faces(int dim, int kind, int order, double hb, double amp, double xs, double ys,
                     double eps, int64_t nx, int64_t ny, double dx, double dy,
                     int64_t i0, int64_t j0, int64_t wnx, int64_t wny, double* h1, double* h2) {
    if (dim == 1) { ny = 1; j0 = 0; wny = 1; }
    for (int64_t jj = 0; jj < wny; ++jj)
        for (int64_t ii = 0; ii < wnx - 1; ++ii)
            h1[jj * (wnx - 1) + ii] = depth_at_face(kind, order, hb, amp, xs, ys, eps, nx, ny, dx, dy,
                                                    1, i0 + ii, j0 + jj);
    if (dim == 2 && h2)
        for (int64_t jj = 0; jj < wny - 1; ++jj)
            for (int64_t ii = 0; ii < wnx; ++ii)
                h2[jj * wnx + ii] = depth_at_face(kind, order, hb, amp, xs, ys, eps, nx, ny, dx, dy,
                                                  2, i0 + ii, j0 + jj);
    return 0;
}

/* R16: Gershgorin bound of the leapfrog CFL condition dt²ρ(K)/4 < 1, with
 * ρ(K) ≤ max over interior nodes of Σ_faces 2h_f/d_f².  Returns 2/√ρ_G. */
double tswo_gershgorin_dt_max(int dim, int64_t nx, int64_t ny, const double* h1, const double* h2,
                              double dx, double dy) {
    double rho = 0.0;
    if (dim == 1) {
        for (int64_t i = 1; i < nx - 1; ++i) {
            double r = 2.0 * ((h1[i - 1] + h1[i]) / (dx * dx));
            if (r > rho) rho = r;
        }
    } else {
        for (int64_t j = 1; j < ny - 1; ++j)
            for (int64_t i = 1; i < nx - 1; ++i) {
                double r = 2.0 * ((h1[j * (nx - 1) + i - 1] + h1[j * (nx - 1) + i]) / (dx * dx)
                                  + (h2[(j - 1) * nx + i] + h2[j * nx + i]) / (dy * dy));
                if (r > rho) rho = r;
            }
    }
    return 2.0 / sqrt(rho);
}

/* ---------------------------------------------------------------------------
 * Piecewise-constant depth with singular terms (§3.1 Case 1
 * eq. (h2case), Cases 2–3 P:773–789, §3.2.3, 2D H(x,y) = h_0(x)
 * P:1145–1149).  h = Σ segments + Σ A_k δ^{o_k}(x − x_k), regularised as
 *   h_ε(x) = (h_0 * φ_ε)(x) + Σ A_k φ_ε(x − x_k)^{o_k}
 * and for the piecewise-constant part, with values v_0 … v_{m−1} and breaks b_1 < … < b_{m−1},
 * h_0 = v_0 + Σ_k (v_k − v_{k−1}) H(x − b_k), so (H(· − b) * φ_ε)(x) = Φ((x − b)/ε) with the
 * primitive Φ(t) = ∫_{−1}^{t} φ.  Φ has no closed form: the oracle integrates
 * it by adaptive Simpson to 1e−15 (pinned against 40-digit mpmath quadrature).
 * ------------------------------------------------------------------------- */
static double phi_unit(double x) {
    if (!(fabs(x) < 1.0)) return 0.0;
    return ORACLE_MOLLIFIER_C * exp(1.0 / (x * x - 1.0));
}

static double simpson_rec(double a, double b, double eps, double whole, double fa, double fb, double fm,
                          int depth) {
    double m = 0.5 * (a + b), lm = 0.5 * (a + m), rm = 0.5 * (m + b);
    double flm = phi_unit(lm), frm = phi_unit(rm);
    double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
    double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
    if (depth <= 0 || fabs(left + right - whole) <= 15.0 * eps) return left + right + (left + right - whole) / 15.0;
    return simpson_rec(a, m, 0.5 * eps, left, fa, fm, flm, depth - 1) +
           simpson_rec(m, b, 0.5 * eps, right, fm, fb, frm, depth - 1);
}

/* Φ(t) = ∫_{−1}^{t} φ(x) dx; 0 for t ≤ −1, 1 for t ≥ 1. */
double tswo_mollifier_primitive(double t) {
    if (t <= -1.0) return 0.0;
    if (t >= 1.0) return 1.0;
    double a = -1.0, b = t;
    double fa = phi_unit(a), fb = phi_unit(b), fm = phi_unit(0.5 * (a + b));
    return simpson_rec(a, b, 1e-16, (b - a) / 6.0 * (fa + 4.0 * fm + fb), fa, fb, fm, 60);
}

/* h_ε at x: segments (nseg values, nseg−1 breaks) + (with_sing) the singular terms, each
 * amplitude multiplied by sing_scale. */
double tswo_profile_eval(double x, double eps, int nseg, const double* seg_value, const double* seg_break,
                         int with_sing, int nsing, const double* sing_loc, const double* sing_amp,
                         const int* sing_order, double sing_scale) {
    double h = seg_value[0];
    for (int k = 1; k < nseg; ++k) h += (seg_value[k] - seg_value[k - 1]) * tswo_mollifier_primitive((x - seg_break[k - 1]) / eps);
    if (with_sing)
        for (int k = 0; k < nsing; ++k) {
            double p = tswo_phi_eps(x - sing_loc[k], eps);
            if (sing_order[k] == 2) p = p * p;
            h += (sing_scale * sing_amp[k]) * p;
        }
    return h;
}

/* Faces of a window (as tswo_build_faces) for an x-only profile: h1 at x faces (i+1/2) with the
 * singular terms; h2 at y faces (i, j+1/2) evaluated at node x_i — with the singular terms when
 * isotropic (scalar depth H(x)), segments only otherwise (vector depth, R6). */
int tswo_build_faces_profile(int dim, int nseg, const double* seg_value, const double* seg_break, int nsing,
                             const double* sing_loc, const double* sing_amp, const int* sing_order,
                             double sing_scale, int isotropic, double eps, int64_t nx, int64_t ny, double dx,
                             int64_t i0, int64_t j0, int64_t wnx, int64_t wny, double* h1, double* h2) {
    (void)ny;
    (void)j0;
    if (dim == 1) wny = 1;
    for (int64_t ii = 0; ii < wnx - 1; ++ii) {
        double v = tswo_profile_eval(face_x(i0 + ii, nx, dx), eps, nseg, seg_value, seg_break, 1, nsing, sing_loc,
                                     sing_amp, sing_order, sing_scale);
        for (int64_t jj = 0; jj < wny; ++jj) h1[jj * (wnx - 1) + ii] = v;
    }
    if (dim == 2 && h2)
        for (int64_t ii = 0; ii < wnx; ++ii) {
            double v = tswo_profile_eval(node_x(i0 + ii, nx, dx), eps, nseg, seg_value, seg_break, isotropic, nsing,
                                         sing_loc, sing_amp, sing_order, sing_scale);
            for (int64_t jj = 0; jj < wny - 1; ++jj) h2[jj * wnx + ii] = v;
        }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Everything below exists once per working precision T (R19): float and
 * double, generated from one macro so both are the same text.
 * ------------------------------------------------------------------------- */
#define ORACLE_DEFINE(T, SFX)                                                                   \
/* O3: c = fl_T((dt²/d²)·h), r = (dt·dt)/(d·d) in fp64. */                                     \
void tswo_prescale_##SFX(const double* h, int64_t n, double dt, double d, T* c) {              \
    double r = (dt * dt) / (d * d);                                                            \
    for (int64_t k = 0; k < n; ++k) c[k] = (T)(r * h[k]);                                      \
}                                                                                              \
                                                                                               \
/* O5: the divergence-form operator L(u) at interior node (i, j), prescaled by dt²:           \
 *   L = (c1_{i+1/2}(u_{i+1}−u_i) − c1_{i−1/2}(u_i−u_{i−1}))                                   \
 *     + (c2_{j+1/2}(u_{j+1}−u_j) − c2_{j−1/2}(u_j−u_{j−1}))                                    \
 * (P:160 Σ_j ∂_j(h_j ∂_j u); R2 flux form with h at half-grid faces).  1D: first bracket. */  \
static T lap_##SFX(int dim, int64_t nx, const T* c1, const T* c2, const T* u, int64_t i,        \
                   int64_t j) {                                                                \
    const T* row = u + j * nx;                                                                 \
    T dxp = row[i + 1] - row[i];                                                               \
    T dxm = row[i] - row[i - 1];                                                               \
    const T* c1row = c1 + j * (nx - 1);                                                        \
    T lx = c1row[i] * dxp - c1row[i - 1] * dxm;                                                \
    if (dim == 1) return lx;                                                                   \
    T dyp = u[(j + 1) * nx + i] - row[i];                                                      \
    T dym = row[i] - u[(j - 1) * nx + i];                                                      \
    T ly = c2[j * nx + i] * dyp - c2[(j - 1) * nx + i] * dym;                                  \
    return lx + ly;                                                                            \
}                                                                                              \
                                                                                               \
void tswo_lap_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2, const T* u,     \
                    T* out) {                                                                  \
    if (dim == 1) ny = 1;                                                                      \
    memset(out, 0, sizeof(T) * (size_t)(nx * ny));                                             \
    int64_t jlo = (dim == 1) ? 0 : 1, jhi = (dim == 1) ? 1 : ny - 1;                           \
    for (int64_t j = jlo; j < jhi; ++j)                                                        \
        for (int64_t i = 1; i < nx - 1; ++i) out[j * nx + i] = lap_##SFX(dim, nx, c1, c2, u, i, j); \
}                                                                                              \
                                                                                               \
/* O4 / R11: Taylor start u¹ = (u⁰ + fl(dt·u₁)) + fl(½·L(u⁰)); ring copied from u⁰. */          \
void tswo_startup_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2, const T* u0, \
                        const T* u1, double dt, T* out) {                                      \
    if (dim == 1) ny = 1;                                                                      \
    const T dtT = (T)dt, half = (T)0.5;                                                        \
    memcpy(out, u0, sizeof(T) * (size_t)(nx * ny));                                            \
    int64_t jlo = (dim == 1) ? 0 : 1, jhi = (dim == 1) ? 1 : ny - 1;                           \
    _Pragma("omp parallel for schedule(static)")                                              \
    for (int64_t j = jlo; j < jhi; ++j)                                                        \
        for (int64_t i = 1; i < nx - 1; ++i) {                                                 \
            T v = u1 ? u1[j * nx + i] : (T)0;                                                  \
            T l = lap_##SFX(dim, nx, c1, c2, u0, i, j);                                        \
            out[j * nx + i] = (u0[j * nx + i] + dtT * v) + half * l;                           \
        }                                                                                      \
}                                                                                              \
                                                                                               \
/* O5: k leapfrog steps u^{n+1} = (2u^n − u^{n−1}) + L(u^n) (north_star's explicit           \
 * second-order leapfrog; R1).  On return un = u^{n+k}, unm1 = u^{n+k−1}. */                    \
void tswo_leapfrog_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2, T* un,      \
                         T* unm1, int64_t k) {                                                 \
    if (dim == 1) ny = 1;                                                                      \
    int64_t jlo = (dim == 1) ? 0 : 1, jhi = (dim == 1) ? 1 : ny - 1;                           \
    size_t bytes = sizeof(T) * (size_t)(nx * ny);                                              \
    T* next = (T*)malloc(bytes);                                                               \
    T* cur = (T*)malloc(bytes);                                                                \
    T* prev = (T*)malloc(bytes);                                                               \
    memcpy(cur, un, bytes);                                                                    \
    memcpy(prev, unm1, bytes);                                                                 \
    memcpy(next, unm1, bytes); /* ring of the new level = ring of the old (fixed) */           \
    for (int64_t s = 0; s < k; ++s) {                                                          \
        _Pragma("omp parallel for schedule(static)")                                          \
        for (int64_t j = jlo; j < jhi; ++j)                                                    \
            for (int64_t i = 1; i < nx - 1; ++i) {                                             \
                T l = lap_##SFX(dim, nx, c1, c2, cur, i, j);                                   \
                next[j * nx + i] = ((T)2 * cur[j * nx + i] - prev[j * nx + i]) + l;            \
            }                                                                                  \
        T* t = prev; prev = cur; cur = next; next = t;                                         \
    }                                                                                          \
    memcpy(un, cur, bytes);                                                                    \
    memcpy(unm1, prev, bytes);                                                                 \
    free(next); free(cur); free(prev);                                                         \
}                                                                                              \
                                                                                               \
/* O6 / R17: E^{n+1/2} = (dx·dy/dt²)·[Σ_interior (u^{n+1}−u^n)²                                 \
 *   + Σ_x-faces c1 (Δx u^{n+1})(Δx u^n) + Σ_y-faces c2 (Δy u^{n+1})(Δy u^n)] in fp64 with the  \
 * stepper's own rounded coefficients — the discrete analogue of CL-01.            \
 * Per-row partials (row j: its kinetic terms, its x faces, the y faces j+1/2) summed in row   \
 * order.  1D: weight dx/dt², no y terms. */                                                   \
double tswo_energy_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2,            \
                         const T* unp1, const T* un, double dx, double dy, double dt) {        \
    if (dim == 1) ny = 1;                                                                      \
    double* part = (double*)calloc((size_t)ny, sizeof(double));                                \
    _Pragma("omp parallel for schedule(static)")                                              \
    for (int64_t j = 0; j < ny; ++j) {                                                         \
        double s = 0.0;                                                                        \
        int interior_row = (dim == 1) || (j >= 1 && j <= ny - 2);                              \
        if (interior_row) {                                                                    \
            for (int64_t i = 1; i < nx - 1; ++i) {                                             \
                double a = (double)unp1[j * nx + i] - (double)un[j * nx + i];                  \
                s += a * a;                                                                    \
            }                                                                                  \
            for (int64_t i = 0; i < nx - 1; ++i) {                                             \
                double da = (double)unp1[j * nx + i + 1] - (double)unp1[j * nx + i];           \
                double db = (double)un[j * nx + i + 1] - (double)un[j * nx + i];              \
                s += ((double)c1[j * (nx - 1) + i] * da) * db;                                 \
            }                                                                                  \
        }                                                                                      \
        if (dim == 2 && j < ny - 1) {                                                          \
            for (int64_t i = 1; i < nx - 1; ++i) {                                             \
                double da = (double)unp1[(j + 1) * nx + i] - (double)unp1[j * nx + i];         \
                double db = (double)un[(j + 1) * nx + i] - (double)un[j * nx + i];             \
                s += ((double)c2[j * nx + i] * da) * db;                                       \
            }                                                                                  \
        }                                                                                      \
        part[j] = s;                                                                           \
    }                                                                                          \
    double S = 0.0;                                                                            \
    for (int64_t j = 0; j < ny; ++j) S += part[j];                                             \
    free(part);                                                                                \
    double w = (dim == 1) ? dx : dx * dy;                                                      \
    return (w / (dt * dt)) * S;                                                                \
}                                                                                              \
                                                                                               \
/* O7 / R18: second-wave amplitude — max and min of fl_T(u − u_bg) over the nodes with       \
 * x_i ≤ xs − eps (all rows), first row-major index on ties; empty region ⇒ 0 and −1. */      \
void tswo_wave2_##SFX(int dim, int64_t nx, int64_t ny, const T* u, const T* ubg, double dx,    \
                      double xs, double eps, double* out2, int64_t* idx2) {                    \
    if (dim == 1) ny = 1;                                                                      \
    double xlim = xs - eps;                                                                    \
    int have = 0;                                                                              \
    T mx = (T)0, mn = (T)0;                                                                    \
    int64_t imx = -1, imn = -1;                                                                \
    for (int64_t j = 0; j < ny; ++j)                                                           \
        for (int64_t i = 0; i < nx; ++i) {                                                     \
            if (!(node_x(i, nx, dx) <= xlim)) continue;                                        \
            T d = u[j * nx + i] - ubg[j * nx + i];                                             \
            if (!have) { mx = mn = d; imx = imn = j * nx + i; have = 1; continue; }            \
            if (d > mx) { mx = d; imx = j * nx + i; }                                          \
            if (d < mn) { mn = d; imn = j * nx + i; }                                          \
        }                                                                                      \
    out2[0] = have ? (double)mx : 0.0;                                                         \
    out2[1] = have ? (double)mn : 0.0;                                                         \
    idx2[0] = imx;                                                                             \
    idx2[1] = imn;                                                                             \
}

ORACLE_DEFINE(double, f64)
ORACLE_DEFINE(float, f32)

/* ---------------------------------------------------------------------------
 * the paper's 2D method as a second workload: "an implicit finite
 * difference scheme [Sam] and the cyclic reduction method [Gode11]" (§3.3, P:1140;
 * GPU timings Table 1).  Reading R26: the factorised three-level
 * Crank–Nicolson scheme (u^{n+1} − 2u^n + u^{n−1})/τ² = A(u^{n+1} + u^{n−1})/2 with
 * I − (τ²/2)A ≈ (I − ½L_x)(I − ½L_y), L = τ²A the prescaled operator of O5:
 *     (I − ½L_x)(I − ½L_y)(u^{n+1} + u^{n−1}) = 2u^n        (1D: (I − ½L_x)(…) = 2u^n)
 * and the implicit start (R27) u¹ = B⁻¹u⁰ + τ·u₁ (the same equation with u^{−1} = u¹ − 2τu₁).
 * The oracle solves every line with the Thomas algorithm (no cyclic reduction: a plain,
 * different solver), rows first, then columns; Dirichlet nodes stay 0.
 * Line matrix (unknowns 1..n−2 of the line):  a_i = −½c_{i−1/2},  b_i = 1 + ½(c_{i−1/2} + c_{i+1/2}),
 * c_i = −½c_{i+1/2}.
 * ------------------------------------------------------------------------- */
#define ORACLE_IMPLICIT(T, SFX)                                                                 \
/* Dirichlet ring (R10) */                                                                     \
static void zero_ring_##SFX(int dim, int64_t nx, int64_t ny, T* u) {                           \
    if (dim == 1) { u[0] = (T)0; u[nx - 1] = (T)0; return; }                                   \
    for (int64_t i = 0; i < nx; ++i) { u[i] = (T)0; u[(ny - 1) * nx + i] = (T)0; }             \
    for (int64_t j = 0; j < ny; ++j) { u[j * nx] = (T)0; u[j * nx + nx - 1] = (T)0; }          \
}                                                                                              \
                                                                                               \
/* Thomas algorithm on x[1..m] (x[0], x[m+1] are the Dirichlet zeros); face coefficient of    \
 * face k+1/2 (between unknowns k and k+1) is cf[k * cstride].  x: rhs in, solution out. */    \
static void thomas_line_##SFX(int64_t m, const T* cf, int64_t cstride, T* x, int64_t xstride,  \
                              T* cp, T* dp) {                                                  \
    const T half = (T)0.5;                                                                     \
    for (int64_t i = 1; i <= m; ++i) {                                                         \
        const T cl = cf[(i - 1) * cstride], cr = cf[i * cstride];                              \
        const T a = -(half * cl), b = (T)1 + half * (cl + cr), c = -(half * cr);                \
        const T d = x[i * xstride];                                                            \
        if (i == 1) {                                                                          \
            cp[i] = c / b;                                                                     \
            dp[i] = d / b;                                                                     \
        } else {                                                                               \
            const T den = b - a * cp[i - 1];                                                   \
            cp[i] = c / den;                                                                   \
            dp[i] = (d - a * dp[i - 1]) / den;                                                 \
        }                                                                                      \
    }                                                                                          \
    x[m * xstride] = dp[m];                                                                    \
    for (int64_t i = m - 1; i >= 1; --i) x[i * xstride] = dp[i] - cp[i] * x[(i + 1) * xstride]; \
}                                                                                              \
                                                                                               \
/* s = B⁻¹ r on the whole grid (r given on all nodes; ring ignored and s's ring set to 0). */  \
void tswo_implicit_solve_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2,      \
                               const T* r, T* s) {                                             \
    if (dim == 1) ny = 1;                                                                      \
    const int64_t N = nx > ny ? nx : ny;                                                       \
    memcpy(s, r, sizeof(T) * (size_t)(nx * ny));                                               \
    zero_ring_##SFX(dim, nx, ny, s);                                                           \
    if (dim == 1) {                                                                            \
        T* cp = (T*)malloc(sizeof(T) * (size_t)N);                                             \
        T* dp = (T*)malloc(sizeof(T) * (size_t)N);                                             \
        thomas_line_##SFX(nx - 2, c1, 1, s, 1, cp, dp);                                         \
        free(cp); free(dp);                                                                    \
        return;                                                                                \
    }                                                                                          \
    _Pragma("omp parallel")                                                                    \
    {                                                                                          \
        T* cp = (T*)malloc(sizeof(T) * (size_t)N);                                             \
        T* dp = (T*)malloc(sizeof(T) * (size_t)N);                                             \
        _Pragma("omp for schedule(static)")                                                   \
        for (int64_t j = 1; j < ny - 1; ++j)   /* x lines: (I − ½L_x) z = r */                  \
            thomas_line_##SFX(nx - 2, c1 + j * (nx - 1), 1, s + j * nx, 1, cp, dp);            \
        _Pragma("omp for schedule(static)")                                                   \
        for (int64_t i = 1; i < nx - 1; ++i)   /* y lines: (I − ½L_y) w = z */                  \
            thomas_line_##SFX(ny - 2, c2 + i, nx, s + i, nx, cp, dp);                          \
        free(cp); free(dp);                                                                    \
    }                                                                                          \
}                                                                                              \
                                                                                               \
/* k implicit levels from (u^n, u^{n−1}): u^{n+1} = B⁻¹(2u^n) − u^{n−1}. */                     \
void tswo_implicit_steps_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2,      \
                               T* un, T* unm1, int64_t k) {                                    \
    if (dim == 1) ny = 1;                                                                      \
    const size_t n = (size_t)(nx * ny);                                                        \
    T* r = (T*)malloc(sizeof(T) * n);                                                          \
    T* w = (T*)malloc(sizeof(T) * n);                                                          \
    for (int64_t s = 0; s < k; ++s) {                                                          \
        for (size_t q = 0; q < n; ++q) r[q] = (T)2 * un[q];                                    \
        tswo_implicit_solve_##SFX(dim, nx, ny, c1, c2, r, w);                                  \
        for (size_t q = 0; q < n; ++q) {                                                       \
            const T next = w[q] - unm1[q];                                                     \
            unm1[q] = un[q];                                                                   \
            un[q] = next;                                                                      \
        }                                                                                      \
        /* Dirichlet ring stays exactly 0 (w's ring is 0; the ring of u^{n−1} is 0) */         \
    }                                                                                          \
    free(r); free(w);                                                                          \
}                                                                                              \
                                                                                               \
/* R27: u¹ = B⁻¹u⁰ + fl(dt·u₁) */                                                                \
void tswo_implicit_startup_##SFX(int dim, int64_t nx, int64_t ny, const T* c1, const T* c2,    \
                                 const T* u0, const T* u1, double dt, T* out) {                \
    if (dim == 1) ny = 1;                                                                      \
    const size_t n = (size_t)(nx * ny);                                                        \
    tswo_implicit_solve_##SFX(dim, nx, ny, c1, c2, u0, out);                                   \
    if (u1) {                                                                                  \
        const T dtT = (T)dt;                                                                   \
        for (size_t q = 0; q < n; ++q) out[q] = out[q] + dtT * u1[q];                          \
        zero_ring_##SFX(dim, nx, ny, out);                                                     \
    }                                                                                          \
}

ORACLE_IMPLICIT(double, f64)
ORACLE_IMPLICIT(float, f32)
