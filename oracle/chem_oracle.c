/* chem_oracle.c — the CPU oracle.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library (see
 * oracle/__init__.py).  It shares no code, header, table or constant generator with the CUDA
 * path under paper_2510_23993_b200/.
 *
 * What it computes: each cell is an independent constant-volume ideal-gas
 * 0-D reactor integrated over [0, dt] for the ODE of oracle_rhs.inc
 * (Eq. 5, corrected Eq. 6), with
 *   - the gate of Alg. 2/3: T < T_min or solid -> cell untouched;
 *   - T from (e, Y) by Newton-Raphson at constant (e, rho), |dT| < 1e-13 T;
 *   - a dense variable-order (1..5) variable-step BDF integrator in the quasi-constant
 *     step-size backward-difference form of Shampine & Reichelt, "The MATLAB ODE suite",
 *     SIAM J. Sci. Comput. 18 (1997) (kappa = 0, i.e. plain BDF) — a C transliteration of
 *     scipy's scipy/integrate/_ivp/bdf.py (compute_R, change_D, the Newton rate test of
 *     solve_bdf_system, NEWTON_MAXITER = 4, MIN/MAX_FACTOR, the safety factor and the
 *     order selection), so the scipy-BDF pin in the tests is a transliteration check and the
 *     scipy-Radau pin is the independent one — simplified Newton with a
 *     dense Jacobian from complex-step differentiation of the loop RHS, dense LU with
 *     partial pivoting, RMS error norm, landing exactly on t_final;
 *   - reported T_out = Newton(e, Y_out) (SURVEY reading 3).
 * OpenMP parallel-for over cells, schedule(dynamic, 64).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXS 32
#define OR_MAXN (OR_MAXS + 1)

typedef struct {
    int32_t ns, nr;
    const double* W;        /* [ns] kg/mol */
    const double* Trange;   /* [ns][3] */
    const double* lo;       /* [ns][7] */
    const double* hi;       /* [ns][7] */
    const int64_t* nu_f;    /* [nr][ns] */
    const int64_t* nu_r;    /* [nr][ns] */
    const double* A;        /* [nr] */
    const double* b;
    const double* Ea;
    const int64_t* kind;    /* 0 elementary, 1 three-body, 2 Lindemann, 3 Troe */
    const int64_t* rev;
    const double* eff;      /* [nr][ns] */
    const double* A0;
    const double* b0;
    const double* Ea0;
    const double* troe;     /* [nr][4] */
    double R, p0;
} omech;

/* ---- real instantiation ---- */
#define S double
#define FN(x) r_##x
#define RE(x) (x)
#define EXP exp
#define LOG log
#include "oracle_rhs.inc"
#undef S
#undef FN
#undef RE
#undef EXP
#undef LOG
/* ---- complex instantiation (complex-step derivatives) ---- */
#define S double complex
#define FN(x) c_##x
#define RE(x) creal(x)
#define EXP cexp
#define LOG clog
#include "oracle_rhs.inc"
#undef S
#undef FN
#undef RE
#undef EXP
#undef LOG

/* ------------------------------------------------------------------ exported point functions */

void or_thermo(const omech* m, double T, double* cp, double* h, double* s) { r_thermo(m, T, cp, h, s); }

void or_rates(const omech* m, double rho, double T, const double* Y, double* wdot, double* qf, double* qr)
{
    r_rates(m, rho, T, Y, wdot, qf, qr);
}

void or_rhs(const omech* m, double rho, const double* y, double* f) { r_rhs(m, rho, y, f); }

/* J[i*n + j] = d f_i / d y_j, n = ns + 1, by complex step: Im f(y + i h e_j) / h. */
void or_jac(const omech* m, double rho, const double* y, double* J)
{
    const int n = m->ns + 1;
    double complex yc[OR_MAXN], fc[OR_MAXN];
    for (int j = 0; j < n; ++j) {
        const double hstep = 1e-40;
        for (int i = 0; i < n; ++i) yc[i] = y[i];
        yc[j] = y[j] + I * hstep;
        c_rhs(m, rho, yc, fc);
        for (int i = 0; i < n; ++i) J[i * n + j] = cimag(fc[i]) / hstep;
    }
}

/* mass-specific internal energy u(T; Y) = sum_k Y_k eps_k / W_k and c_v */
static void u_cv(const omech* m, double T, const double* Y, double* u, double* cv)
{
    double cp[OR_MAXS], h[OR_MAXS];
    r_thermo(m, T, cp, h, 0);
    double su = 0.0, sc = 0.0;
    for (int k = 0; k < m->ns; ++k) {
        su += Y[k] * (h[k] - m->R * T) / m->W[k];
        sc += Y[k] * (cp[k] - m->R) / m->W[k];
    }
    *u = su;
    *cv = sc;
}

double or_energy(const omech* m, double T, const double* Y)
{
    double u, cv;
    u_cv(m, T, Y, &u, &cv);
    return u;
}

double or_cv(const omech* m, double T, const double* Y)
{
    double u, cv;
    u_cv(m, T, Y, &u, &cv);
    return cv;
}

/* Newton-Raphson T at constant (e, rho): T <- T - (u(T) - e)/c_v(T) until
 * |dT| < 1e-13 T; returns iterations used, -1 on failure to converge in 100. */
int or_newton_T(const omech* m, double e, const double* Y, double Tguess, double* Tout)
{
    double T = Tguess;
    for (int it = 1; it <= 100; ++it) {
        double u, cv;
        u_cv(m, T, Y, &u, &cv);
        double dT = (u - e) / cv;
        T -= dT;
        if (!(fabs(dT) >= 1e-13 * fabs(T))) {   /* also exits on NaN */
            *Tout = T;
            return isfinite(T) ? it : -1;
        }
    }
    *Tout = T;
    return -1;
}

/* ------------------------------------------------------------------ dense LU, partial pivoting */

static int lu_factor(int n, double* a, int* piv)
{
    for (int k = 0; k < n; ++k) {
        int p = k;
        double amax = fabs(a[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (fabs(a[i * n + k]) > amax) { amax = fabs(a[i * n + k]); p = i; }
        piv[k] = p;
        if (amax == 0.0 || !isfinite(amax)) return -1;
        if (p != k)
            for (int j = 0; j < n; ++j) { double t = a[k * n + j]; a[k * n + j] = a[p * n + j]; a[p * n + j] = t; }
        for (int i = k + 1; i < n; ++i) {
            double l = a[i * n + k] / a[k * n + k];
            a[i * n + k] = l;
            for (int j = k + 1; j < n; ++j) a[i * n + j] -= l * a[k * n + j];
        }
    }
    return 0;
}

static void lu_solve(int n, const double* a, const int* piv, double* x)
{
    for (int k = 0; k < n; ++k)
        if (piv[k] != k) { double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) x[i] -= a[i * n + j] * x[j];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) x[i] -= a[i * n + j] * x[j];
        x[i] /= a[i * n + i];
    }
}

/* ------------------------------------------------------------------ BDF (Shampine-Reichelt form) */

#define BDF_MAXORD 5
#define NEWTON_MAXITER 4
#define MIN_FACTOR 0.2
#define MAX_FACTOR 10.0

typedef struct {
    const omech* m;
    double rho;
    int n;
    double rtol;
    const double* atol;   /* [n] */
    int64_t nfev, njev, nlu, nsteps, nrej;
} bdf_prob;

static double rms_norm(int n, const double* x, const double* scale)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i) { double v = x[i] / scale[i]; s += v * v; }
    return sqrt(s / n);
}

static void fun(bdf_prob* P, const double* y, double* f) { r_rhs(P->m, P->rho, y, f); P->nfev++; }

/* R matrix of the step-size change (Shampine-Reichelt eq. for backward differences):
 * M[i][j] = (i - 1 - factor*j)/i for i,j >= 1, M[0][j] = 1; R = cumulative product down columns. */
static void compute_R(int order, double factor, double* R /*[(order+1)^2]*/)
{
    int o1 = order + 1;
    for (int i = 0; i < o1; ++i)
        for (int j = 0; j < o1; ++j) {
            double mij = (i == 0) ? 1.0 : (j == 0 ? 0.0 : ((double)(i - 1) - factor * j) / i);
            if (i == 0 && j == 0) mij = 1.0;
            R[i * o1 + j] = (i == 0) ? mij : R[(i - 1) * o1 + j] * mij;
        }
}

static void change_D(int n, double* D /*[(BDF_MAXORD+3)][n]*/, int order, double factor)
{
    double Rm[36], U[36], RU[36], tmp[(BDF_MAXORD + 3) * OR_MAXN];
    int o1 = order + 1;
    compute_R(order, factor, Rm);
    compute_R(order, 1.0, U);
    for (int i = 0; i < o1; ++i)
        for (int j = 0; j < o1; ++j) {
            double s = 0.0;
            for (int k = 0; k < o1; ++k) s += Rm[i * o1 + k] * U[k * o1 + j];
            RU[i * o1 + j] = s;
        }
    /* D[:o1] = RU^T @ D[:o1] */
    for (int i = 0; i < o1; ++i)
        for (int c = 0; c < n; ++c) {
            double s = 0.0;
            for (int k = 0; k < o1; ++k) s += RU[k * o1 + i] * D[k * n + c];
            tmp[i * n + c] = s;
        }
    memcpy(D, tmp, sizeof(double) * o1 * n);
}

/* Integrate y over [0, tf].  Returns 0 on success, negative on failure. */
static int bdf_integrate(bdf_prob* P, double* y, double tf)
{
    const int n = P->n;
    const double EPS = 2.220446049250313e-16;
    double gamma[BDF_MAXORD + 2], alpha[BDF_MAXORD + 2], err_const[BDF_MAXORD + 2];
    gamma[0] = 0.0;
    for (int j = 1; j <= BDF_MAXORD + 1; ++j) gamma[j] = gamma[j - 1] + 1.0 / j;
    for (int j = 0; j <= BDF_MAXORD + 1; ++j) { alpha[j] = gamma[j]; err_const[j] = 1.0 / (j + 1); }
    const double newton_tol = fmax(10.0 * EPS / P->rtol, fmin(0.03, sqrt(P->rtol)));

    double f0[OR_MAXN], scale[OR_MAXN], y1[OR_MAXN], f1[OR_MAXN], tmpv[OR_MAXN];
    double D[(BDF_MAXORD + 3) * OR_MAXN];
    double J[OR_MAXN * OR_MAXN], LU[OR_MAXN * OR_MAXN];
    int piv[OR_MAXN];
    double t = 0.0;
    if (!(tf >= 0.0) || isinf(tf)) return -5;    /* negative, NaN or infinite interval: an error */
    if (tf == 0.0) return 0;

    fun(P, y, f0);
    /* initial step (Hairer-Norsett-Wanner I, II.4; scipy select_initial_step with order 1) */
    for (int i = 0; i < n; ++i) scale[i] = P->atol[i] + fabs(y[i]) * P->rtol;
    double d0 = rms_norm(n, y, scale), d1 = rms_norm(n, f0, scale), h0;
    if (d0 < 1e-5 || d1 < 1e-5) h0 = 1e-6; else h0 = 0.01 * d0 / d1;
    h0 = fmin(h0, tf);
    for (int i = 0; i < n; ++i) y1[i] = y[i] + h0 * f0[i];
    fun(P, y1, f1);
    for (int i = 0; i < n; ++i) tmpv[i] = f1[i] - f0[i];
    double d2 = rms_norm(n, tmpv, scale) / h0, h1;
    if (d1 <= 1e-15 && d2 <= 1e-15) h1 = fmax(1e-6, h0 * 1e-3);
    else h1 = pow(0.01 / fmax(d1, d2), 1.0 / 2.0);
    double h_abs = fmin(fmin(100 * h0, h1), tf);

    or_jac(P->m, P->rho, y, J);
    P->njev++;
    int lu_valid = 0, current_jac = 1;
    memset(D, 0, sizeof(D));
    for (int i = 0; i < n; ++i) { D[0 * n + i] = y[i]; D[1 * n + i] = f0[i] * h_abs; }
    int order = 1, n_equal_steps = 0;
    double y_new[OR_MAXN], d[OR_MAXN], y_pred[OR_MAXN], psi[OR_MAXN], err[OR_MAXN];

    while (t < tf) {
        double min_step = 10.0 * (nextafter(t, INFINITY) - t);
        int accepted = 0, n_iter = 0;
        double error_norm = 0.0, safety = 0.9;
        while (!accepted) {
            if (h_abs < min_step) return -2;
            double t_new = t + h_abs;
            if (t_new > tf) {
                t_new = tf;
                change_D(n, D, order, (t_new - t) / h_abs);
                n_equal_steps = 0;
                lu_valid = 0;
            }
            double h = t_new - t;
            h_abs = h;
            for (int i = 0; i < n; ++i) {
                double s = 0.0;
                for (int k = 0; k <= order; ++k) s += D[k * n + i];
                y_pred[i] = s;
                scale[i] = P->atol[i] + P->rtol * fabs(y_pred[i]);
                double ps = 0.0;
                for (int k = 1; k <= order; ++k) ps += D[k * n + i] * gamma[k];
                psi[i] = ps / alpha[order];
            }
            const double c = h / alpha[order];
            int converged = 0;
            for (;;) {
                if (!lu_valid) {
                    for (int i = 0; i < n; ++i)
                        for (int j = 0; j < n; ++j) LU[i * n + j] = (i == j ? 1.0 : 0.0) - c * J[i * n + j];
                    P->nlu++;
                    if (lu_factor(n, LU, piv) != 0) return -3;
                    lu_valid = 1;
                }
                /* simplified Newton iteration for the BDF system */
                double dy_norm_old = -1.0;
                for (int i = 0; i < n; ++i) { d[i] = 0.0; y_new[i] = y_pred[i]; }
                converged = 0;
                int k;
                for (k = 0; k < NEWTON_MAXITER; ++k) {
                    double fv[OR_MAXN], dy[OR_MAXN];
                    fun(P, y_new, fv);
                    int finite = 1;
                    for (int i = 0; i < n; ++i) finite &= isfinite(fv[i]);
                    if (!finite) break;
                    for (int i = 0; i < n; ++i) dy[i] = c * fv[i] - psi[i] - d[i];
                    lu_solve(n, LU, piv, dy);
                    double dy_norm = rms_norm(n, dy, scale);
                    double rate = (dy_norm_old < 0.0) ? -1.0 : dy_norm / dy_norm_old;
                    if (rate >= 0.0 && (rate >= 1.0 || pow(rate, NEWTON_MAXITER - k) / (1.0 - rate) * dy_norm > newton_tol))
                        break;
                    for (int i = 0; i < n; ++i) { y_new[i] += dy[i]; d[i] += dy[i]; }
                    if (dy_norm == 0.0 || (rate >= 0.0 && rate / (1.0 - rate) * dy_norm < newton_tol)) {
                        converged = 1;
                        break;
                    }
                    dy_norm_old = dy_norm;
                }
                n_iter = k + 1;
                if (converged || current_jac) break;
                or_jac(P->m, P->rho, y_pred, J);
                P->njev++;
                lu_valid = 0;
                current_jac = 1;
            }
            if (!converged) {
                double factor = 0.5;
                h_abs *= factor;
                change_D(n, D, order, factor);
                n_equal_steps = 0;
                lu_valid = 0;
                P->nrej++;
                continue;
            }
            safety = 0.9 * (2 * NEWTON_MAXITER + 1) / (double)(2 * NEWTON_MAXITER + n_iter);
            for (int i = 0; i < n; ++i) {
                scale[i] = P->atol[i] + P->rtol * fabs(y_new[i]);
                err[i] = err_const[order] * d[i];
            }
            error_norm = rms_norm(n, err, scale);
            if (error_norm > 1.0) {
                double factor = fmax(MIN_FACTOR, safety * pow(error_norm, -1.0 / (order + 1)));
                h_abs *= factor;
                change_D(n, D, order, factor);
                n_equal_steps = 0;
                P->nrej++;
            } else {
                accepted = 1;
                t = t_new;
            }
        }
        P->nsteps++;
        n_equal_steps++;
        current_jac = 0;
        for (int i = 0; i < n; ++i) y[i] = y_new[i];
        for (int i = 0; i < n; ++i) {
            D[(order + 2) * n + i] = d[i] - D[(order + 1) * n + i];
            D[(order + 1) * n + i] = d[i];
        }
        for (int k = order; k >= 0; --k)
            for (int i = 0; i < n; ++i) D[k * n + i] += D[(k + 1) * n + i];
        if (t >= tf) break;
        if (n_equal_steps < order + 1) continue;
        double em = INFINITY, ep = INFINITY;
        if (order > 1) {
            for (int i = 0; i < n; ++i) tmpv[i] = err_const[order - 1] * D[order * n + i];
            em = rms_norm(n, tmpv, scale);
        }
        if (order < BDF_MAXORD) {
            for (int i = 0; i < n; ++i) tmpv[i] = err_const[order + 1] * D[(order + 2) * n + i];
            ep = rms_norm(n, tmpv, scale);
        }
        double norms[3] = {em, error_norm, ep};
        double best = -1.0;
        int delta = 0;
        for (int q = 0; q < 3; ++q) {
            double fac = (norms[q] == 0.0) ? INFINITY : pow(norms[q], -1.0 / (order + q));
            if (isinf(norms[q])) fac = 0.0;
            if (fac > best) { best = fac; delta = q - 1; }
        }
        order += delta;
        double factor = fmin(MAX_FACTOR, safety * best);
        h_abs *= factor;
        change_D(n, D, order, factor);
        n_equal_steps = 0;
        lu_valid = 0;
        if (P->nsteps > 5000000) return -4;
    }
    return 0;
}

/* Integrate one reactor state y = (Y, T) over [0, tf] (no gate, no Newton): used for the
 * trajectory tables and ignition-delay pins.  stats[0..4] = steps, rejections, fevals, jevals, LUs. */
int or_integrate_state(const omech* m, double rho, double* y, double tf, double rtol, double atolY,
                       double atolT, int64_t* stats)
{
    double atol[OR_MAXN];
    for (int k = 0; k < m->ns; ++k) atol[k] = atolY;
    atol[m->ns] = atolT;
    bdf_prob P = {m, rho, m->ns + 1, rtol, atol, 0, 0, 0, 0, 0};
    int rc = bdf_integrate(&P, y, tf);
    if (stats) { stats[0] = P.nsteps; stats[1] = P.nrej; stats[2] = P.nfev; stats[3] = P.njev; stats[4] = P.nlu; }
    return rc;
}

/* The cell loop: SURVEY.md §8(c) steps 3-7 over n cells.  Y is cell-major [n][ns] (the oracle's
 * own layout).  status: 0 integrated, 1 gated (untouched), <0 failure code.  T_int (optional)
 * receives the integrated temperature (energy-drift check, SURVEY reading 3). */
void or_integrate_cells(const omech* m, int64_t n, const double* rho, const double* e, double* T, double* Y,
                        const uint8_t* solid, double dt, double rtol, double atolY, double atolT, double Tmin,
                        int nthreads, int64_t* nsteps, int32_t* status, double* T_int)
{
    const int ns = m->ns;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        if (T[i] < Tmin || (solid && solid[i])) {
            if (status) status[i] = 1;
            if (nsteps) nsteps[i] = 0;
            if (T_int) T_int[i] = T[i];
            continue;
        }
        double y[OR_MAXN];
        double* Yi = &Y[i * ns];
        double T0;
        int rc = 0;
        if (or_newton_T(m, e[i], Yi, T[i], &T0) < 0) rc = -10;
        for (int k = 0; k < ns; ++k) y[k] = Yi[k];
        y[ns] = T0;
        int64_t st[5] = {0, 0, 0, 0, 0};
        if (rc == 0) rc = or_integrate_state(m, rho[i], y, dt, rtol, atolY, atolT, st);
        if (rc == 0) {
            for (int k = 0; k < ns; ++k) Yi[k] = y[k];
            double Tn;
            if (or_newton_T(m, e[i], Yi, y[ns], &Tn) < 0) rc = -11;
            T[i] = Tn;
            if (T_int) T_int[i] = y[ns];
        }
        if (status) status[i] = rc;
        if (nsteps) nsteps[i] = st[0];
    }
}

/* The paper's explicit first-order adaptive scheme, written out
 * step by step for algorithmic parity with the CUDA path's CHEM_METHOD_EXPLICIT:
 *   Omega = rates(T, rho, Y); dY_k/dt = W_k Omega_k / rho                         (Eq. 5)
 *   dt = min(eps * min_{k: Y_k > 1e-12, dY_k/dt != 0} Y_k / |dY_k/dt|, t_final - t),
 *        the remaining time taken when the rule's step is within 1e-10 of it
 *   Y <- max(Y + dt dY/dt, 0)  (clip, no renormalisation)
 *   T <- Newton(e, Y) at constant (e, rho)
 * while t < t_final and k < kmax.  status: 0 done, 1 gated, 2 unfinished (kmax), <0 failure. */
void or_explicit_cells(const omech* m, int64_t n, const double* rho, const double* e, double* T, double* Y,
                       const uint8_t* solid, double dt, double eps, double Tmin, int64_t kmax, int nthreads,
                       int64_t* nsteps, int32_t* status)
{
    const int ns = m->ns;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        if (T[i] < Tmin || (solid && solid[i])) {
            if (status) status[i] = 1;
            if (nsteps) nsteps[i] = 0;
            continue;
        }
        double* Yi = &Y[i * ns];
        double Tc;
        int rc = 0;
        if (or_newton_T(m, e[i], Yi, T[i], &Tc) < 0) rc = -10;
        double t = 0.0;
        int64_t k = 0;
        while (rc == 0 && t < dt && k < kmax) {
            double w[OR_MAXS], f[OR_MAXS];
            r_rates(m, rho[i], Tc, Yi, w, 0, 0);
            double rmin = INFINITY;
            for (int s = 0; s < ns; ++s) {
                f[s] = m->W[s] * w[s] / rho[i];
                if (Yi[s] > 1e-12 && f[s] != 0.0) {
                    double r = Yi[s] / fabs(f[s]);
                    if (r < rmin) rmin = r;
                }
            }
            double h = eps * rmin;
            /* land on t_final when the rule's step reaches it to 1e-10 relative (no sliver step
             * from the rounding of t += h) */
            int last = !(h < (dt - t) * (1.0 - 1e-10));
            if (last) h = dt - t;
            for (int s = 0; s < ns; ++s) {
                double v = Yi[s] + h * f[s];
                Yi[s] = v > 0.0 ? v : 0.0;
            }
            double Tn;
            if (or_newton_T(m, e[i], Yi, Tc, &Tn) < 0) rc = -11;
            Tc = Tn;
            t = last ? dt : t + h;
            ++k;
        }
        if (rc == 0 && t < dt) rc = 2;
        T[i] = Tc;
        if (status) status[i] = rc;
        if (nsteps) nsteps[i] = k;
    }
}

int or_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
