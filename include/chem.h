/* chem.h — C ABI of libchem.so: bulk-sparse stiff chemistry integration on B200 (sm_100a).
 *
 * The operation (§2.1): every cell i is an independent constant-volume,
 * ideal-gas 0-D reactor ("each cell in the domain simulates a 0D reactor, assuming constant volume
 * and the ideal gas law") integrated over the flow step [0, dt] ("0 < t_i < dt_CFL"):
 *      dY_k/dt = W_k Omega_k / rho                                     (Eq. 5)
 *      dT/dt   = - sum_k eps_k Omega_k / (rho sum_k Y_k c_v,k)          (Eq. 6, corrected
 *                                                                         reading)
 * with Omega_k from the matrix-based rate formulation (BASELINE.json north_star; SURVEY.md §8(a)
 * A4), T recovered by Newton-Raphson at constant (e, rho), the gate of Alg. 2/3
 * (T < T_min or solid -> untouched) and the bulk-sparse schedule of
 * Alg. 3: count -> bulk bursts of <= K_max substeps while N_active > N* -> compact to a
 * cell index map -> sparse integration with K_max = 1e5.  One launch per phase
 * spans every box ("a single kernel across all cells from all grids").
 *
 * Conventions for every entry point:
 *  - Array pointers are DEVICE pointers owned by the caller unless stated otherwise.
 *  - Layout is component-major ("column-major", Alg. 1): component c of cell i
 *    is at p[c*ld + i], ld >= n.  Species order is the mechanism's.
 *  - SI units: rho kg/m^3, e J/kg (mass-specific internal energy), T K, t s, Omega mol/(m^3 s).
 *  - All device work is enqueued on `stream` (a cudaStream_t, NULL = legacy default stream), as
 *    kernels only: the library's own small transfers (box table in, counters out) go through mapped
 *    pinned memory, never through a copy engine, so a caller's large copies on other streams do not
 *    hold back its next command.
 *  - Return 0 on success or a negative CHEM_E* code; text via chem_strerror().  Per-cell
 *    problems (non-convergence, non-finite state) are NOT call errors: they are counted in
 *    chem_stats.  The library never aborts the process.
 *  - A chem_ctx is bound to one device; it is not re-entrant (one host thread at a time).
 */
#ifndef CHEM_H
#define CHEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ---------------------------------------------------------------------- */
#define CHEM_OK 0
#define CHEM_EINVAL (-1)      /* null pointer, n < 0, ld < n, dt <= 0, rtol <= 0, bad option   */
#define CHEM_EMECH (-2)       /* mechanism tables fail validation (mass/element balance > 1e-10
                                 relative, W <= 0, non-contiguous T ranges, unknown type)        */
#define CHEM_ENOSTRUCT (-3)   /* valid mechanism whose reaction structure is not compiled in    */
#define CHEM_ECUDA (-4)       /* CUDA runtime error (sticky for the ctx); see chem_strerror     */
#define CHEM_ENOWS (-5)       /* workspace too small (see chem_workspace_bytes)                 */

/* ---- mechanism tables (HOST pointers; copied by chem_init, caller may free afterwards) --- */
#define CHEM_RXN_ELEMENTARY 0
#define CHEM_RXN_THREE_BODY 1
#define CHEM_RXN_LINDEMANN 2
#define CHEM_RXN_TROE 3

typedef struct {
    int32_t ns, nr, ne;        /* species (<= 32), reaction rows, elements                     */
    const double* W;           /* [ns] molar masses, kg/mol                                    */
    const double* nasa_lo;     /* [ns][7] NASA-7 coefficients for T in [T_lo, T_mid]           */
    const double* nasa_hi;     /* [ns][7] NASA-7 coefficients for T in [T_mid, T_hi]           */
    const double* T_range;     /* [ns][3] T_lo, T_mid, T_hi                                    */
    const int32_t* elem;       /* [ns][ne] atom counts (validation)                            */
    const double* nu_f;        /* [nr][ns] reactant stoichiometric coefficients nu'            */
    const double* nu_r;        /* [nr][ns] product stoichiometric coefficients nu''            */
    const double* A;           /* [nr] pre-exponential (k_inf for falloff rows), SI-molar      */
    const double* b;           /* [nr] temperature exponent                                    */
    const double* Ea;          /* [nr] activation energy, J/mol                                */
    const int32_t* type;       /* [nr] CHEM_RXN_*                                              */
    const int32_t* reversible; /* [nr] 1: reverse rate from K_c (NASA Gibbs, p_ref)            */
    const double* eff;         /* [nr][ns] third-body efficiencies (1 = default)               */
    const double* A0;          /* [nr] falloff low-pressure limit k_0 (k_0 multiplies [M])     */
    const double* b0;          /* [nr]                                                          */
    const double* Ea0;         /* [nr] J/mol                                                    */
    const double* troe;        /* [nr][4] alpha, T***, T*, T** (T** <= 0: term absent)          */
    double R;                  /* gas constant, 8.314462618 J/(mol K)                           */
    double p_ref;              /* standard pressure of K_c, 101325 Pa                           */
} chem_mech_desc;

/* ---- options ------------------------------------------------------------------------------ */
#define CHEM_METHOD_RODAS4 0   /* 6-stage order-4 L-stable Rosenbrock, embedded order 3 (default) */
#define CHEM_METHOD_RODAS3 1   /* 4-stage order-3 L-stable Rosenbrock, embedded order 2           */
#define CHEM_METHOD_EXPLICIT 2 /* the paper's explicit 1st-order adaptive scheme: dt limited so
                                  no Y_k (> 1e-12) changes by more than eps_change of itself; Euler
                                  update clipped at 0; T from Newton every step    */

typedef struct {
    double T_min;           /* gate T_reaction_min (value unstated -> 500 K) */
    int32_t kmax_bulk;      /* attempted substeps per cell per bulk launch (K_max = 5)     */
    int64_t n_active_star;  /* bulk->sparse threshold N*_active (the paper's 1e4 is
                               H100-tuned).  < 0 (default): one resident wave of the integration
                               kernel, SMs x resident cells per SM (37 888 on a B200)             */
    int32_t kmax_sparse;    /* K_max of the sparse phase (1e5), applied as the per-cell budget
                               of attempted substeps over the whole call (bulk bursts + sparse
                               launch, or the heavy-first launch): a cell that spends it ends
                               CHEM_CELL_UNFINISHED at its last accepted state, whatever the
                               schedule (reading R10)                                   */
    double atol_T;          /* absolute tolerance on the integrated temperature, K               */
    int32_t method;         /* CHEM_METHOD_*                                                      */
    int32_t compact_bulk;   /* 1 (default): bulk bursts run over the compacted active list;
                               0: every bulk launch spans all cells of all boxes (paper's Alg. 3) */
    double eps_change;      /* CHEM_METHOD_EXPLICIT: max fractional change per step (0.01; P:96 1-5%) */
    double h0_factor;       /* first substep of a cell = h0_factor * |y|/|f(y)| (WRMS norms), capped
                               at dt (Hairer-Norsett-Wanner I.II.4 use 0.01)                      */
    int32_t lockstep;       /* bulk bursts run as 256-thread blocks whose warps take every substep
                               together (one barrier per substep), keeping an SM's warps in the same
                               code on heterogeneous fields (shared instruction cache):
                               0 off, 1 on, 2 auto (on while the previous call's bulk SIMT efficiency
                               = lane substeps / (32 x warp substeps) is below 0.9).  Results are
                               bitwise independent of this choice.                                */
    int32_t kmax_first;     /* substeps of the first bulk burst of a lockstep call (1: cells that
                               finish in one substep leave before the lockstep bursts); 0: kmax_bulk */
    int32_t schedule_lpt;   /* heavy-first schedule: the active list sorted by predicted cost and run as
                               one persistent launch with lane refill, longest cells first.  Predictions come
                               from the previous call's per-cell substeps on the same layout (kept in
                               the workspace) or, within the call, from each cell's own state after the
                               first bulk burst (remaining substeps (dt - t)/h).  0 off (Alg. 3);
                               1 previous-call hints always; 2 auto: previous-call hints when they are
                               skewed (cells above 64 substeps carried half of the work, or the largest
                               hint exceeds 1.5x the mean) and predictive (the layout's last
                               chem_stats.hint_accuracy >= 0.9), else the in-call prediction when it
                               is skewed (max > 1.5x mean); 3 in-call prediction always.
                               Bitwise-neutral.                                                     */
} chem_opts;

/* fills the defaults: T_min 500 K, kmax_bulk 5, n_active_star -1 (auto: one resident wave),
   kmax_sparse 1e5, atol_T 1e-6 K, RODAS4, compact_bulk 1, eps_change 0.01, h0_factor 0.01,
   lockstep 2 (auto), kmax_first 1, schedule_lpt 2 (auto) */
void chem_default_opts(chem_opts* o);

/* ---- per-cell outcome of the last chem_integrate* call --------------------- */
#define CHEM_CELL_UNTOUCHED 0      /* gated out (T < T_min or solid): bytes untouched            */
#define CHEM_CELL_DONE 1           /* integrated to t = dt                                       */
#define CHEM_CELL_UNFINISHED 2     /* substep budget (kmax_sparse) spent: last accepted state    */
#define CHEM_CELL_FAILED (-1)      /* Newton failure, non-finite state or step-size underflow   */

/* ---- one AMR box / grid (FAB analogue) for the fused multi-box call ----------------- */
typedef struct {
    const double* rho;      /* [ncells]        device                                           */
    const double* e;        /* [ncells]        device, mass-specific internal energy            */
    double* T;              /* [ncells]        device, in: gate + Newton guess; out: T(e, Y_out) */
    double* Y;              /* [ns][ld]        device, in/out                                   */
    const uint8_t* solid;   /* [ncells] or NULL device; nonzero = embedded solid (not integrated)*/
    int64_t ncells, ld;
    double dt;              /* t_final of this box (AMR subcycling: each level its own dt) */
} chem_box;

/* ---- statistics (host struct filled at the end of a call) ---------------------------------- */
typedef struct {
    int64_t cells;              /* cells in the call                                           */
    int64_t active0;            /* N_active after the gate (Alg. 3 §1)                          */
    int64_t bulk_iters;         /* bulk launches (Alg. 3 §2 loop trips)                         */
    int64_t sparse_cells;       /* cells handed to the sparse launch (Alg. 3 §3)                */
    int64_t steps_attempted;    /* substeps attempted (accepted + rejected), all cells          */
    int64_t steps_accepted;
    int64_t steps_frozen;       /* first steps taken as one explicit step by frozen cells (subset of attempted) */
    int64_t rhs_evals, jac_evals, lu_count;
    int64_t n_unfinished;       /* cells with t < dt whose substep budget (kmax_sparse) was spent */
    int64_t n_newton_fail;      /* temperature Newton not converged in 50 iterations            */
    int64_t n_nonfinite;        /* non-finite state / step size underflow                       */
    int64_t n_T_range;          /* finished cells whose T lies outside the NASA ranges          */
    double t_gate_ms, t_bulk_ms, t_compact_ms, t_sparse_ms;   /* CUDA-event phase times         */
    double max_energy_drift;    /* max |T_int - T(e, Y_out)| / T over finished cells            */
    int64_t active_per_iter[16];/* N_active after each of the first 16 bulk launches (App. B)   */
    int64_t warp_substeps;      /* warp-level substep issues in bulk launches (SIMT efficiency =
                                   bulk lane substeps / (32 x warp_substeps))                   */
    int64_t bulk_substeps;      /* lane substeps attempted in bulk launches                     */
    int64_t lockstep;           /* 1: this call's bulk bursts ran in lockstep                   */
    int64_t lpt;                /* heavy-first schedule of this call: 0 no, 1 on the previous call's
                                   hints, 2 on the in-call prediction after the first burst       */
    double hint_accuracy;       /* how well the cost hints (the previous call's per-cell substeps on
                                   this layout) predicted this call: sum_cells min(hint, actual) /
                                   sum_cells max(hint, actual); -1 without hints.  schedule_lpt = 2
                                   engages heavy-first only while the last value is >= 0.9        */
    int64_t kernel_launches;    /* kernels this call enqueued (integration, gate, compaction, sort,
                                   bookkeeping transfers)                                          */
} chem_stats;

typedef struct chem_ctx chem_ctx;   /* opaque, library-owned */

/* Validate the tables, match their reaction structure against the
 * compiled structures, copy the numbers for the kernels.  `opts` may be NULL (defaults).
 * device = CUDA ordinal the ctx is bound to.  On success *out is a new ctx. */
int chem_init(const chem_mech_desc* mech, const chem_opts* opts, int device, chem_ctx** out);
void chem_finalize(chem_ctx* ctx);
const char* chem_strerror(int code);
/* name of the compiled structure the ctx runs on, or "" */
const char* chem_structure_name(const chem_ctx* ctx);
int chem_set_opts(chem_ctx* ctx, const chem_opts* opts);

/* Device workspace (bytes, 256-aligned pointer) a chem_integrate* call needs for up to
 * max_cells cells in up to max_boxes boxes.  Owned by the caller (e.g. torch.zeros).  Zero-fill it
 * before its first use: it carries the per-cell cost hints of the heavy-first schedule
 * (chem_opts.schedule_lpt) from one call to the next on the same cell layout.  Results never depend
 * on its previous contents (only the processing order does). */
size_t chem_workspace_bytes(const chem_ctx* ctx, int64_t max_cells, int32_t max_boxes);

/* Molar production rates Omega.  wdot is [ns][ld].  Never synchronises. */
int chem_rates(chem_ctx* ctx, int64_t n, int64_t ld, const double* rho, const double* T,
               const double* Y, double* wdot, void* stream);

/* Integrate n cells of one box over [0, dt] (the single-box form of chem_integrate_boxes).
 * T: in = gate temperature and Newton guess, out = T(e, Y_out).  Y in/out.  solid nullable.
 * rtol, atol: tolerances of the error-controlled integrator on Y_k (atol_T from opts on T).
 * stats (HOST, nullable).  Synchronises `stream` to read the bulk-loop counters (as the paper
 * does) and once at the end. */
int chem_integrate(chem_ctx* ctx, int64_t n, int64_t ld, const double* rho, const double* e,
                   double* T, double* Y, const uint8_t* solid, double dt, double rtol, double atol,
                   void* ws, size_t ws_bytes, chem_stats* stats, void* stream);

/* The fused multi-box call: `boxes` is a HOST array of nboxes descriptors.  One launch per
 * phase spans all boxes through a cell index map.  box_cost (DEVICE, [nboxes],
 * nullable) receives the attempted substeps summed over each box's cells: the per-box
 * chemistry cost used for load balancing. */
int chem_integrate_boxes(chem_ctx* ctx, int32_t nboxes, const chem_box* boxes, double rtol,
                         double atol, void* ws, size_t ws_bytes, double* box_cost,
                         chem_stats* stats, void* stream);

/* Per-cell outcome of the last chem_integrate* call that used workspace `ws`, for global cells
 * [first, first + n), where global cells number the boxes of that call in order (box b's cell j is
 * sum_{a<b} ncells_a + j; a chem_integrate call is one box):
 *   status[i]   (DEVICE int8 [n], nullable)   CHEM_CELL_* code;
 *   substeps[i] (DEVICE int32 [n], nullable)  attempted substeps the cell took in that call (its
 *               chemistry cost; 0 for untouched cells).
 * Both owned by the caller.  Reads the workspace's per-cell state; enqueued on `stream`, no
 * synchronisation.  CHEM_EINVAL if the workspace has no recorded call on this ctx or
 * [first, first + n) lies outside that call's cells. */
int chem_cell_status(chem_ctx* ctx, const void* ws, size_t ws_bytes, int64_t first, int64_t n,
                     int8_t* status, int32_t* substeps, void* stream);

/* Caller-side helper for host-resident fields: active[b] (DEVICE int32 [nboxes], caller-owned) = the
 * cells of box b that the gate of Alg. 3 §1 would integrate (T >= T_min and not solid), read
 * from the boxes' T (and solid) only; rho, e and Y are not read, so a caller may move them to the device
 * only for boxes with active[b] > 0 before chem_integrate_boxes (gated cells are never read or written).
 * ws: a workspace of >= chem_workspace_bytes(ctx, 0, nboxes) bytes (its box table is overwritten).
 * Synchronises `stream` before returning. */
int chem_box_active(chem_ctx* ctx, int32_t nboxes, const chem_box* boxes, int32_t* active, void* ws,
                    size_t ws_bytes, void* stream);

/* Activity trace (App. B/* Activity trace (App. B: "the number of active cells after each integration step
 * for every grid").  trace: DEVICE int32 [rows][nboxes] owned by the caller; subsequent
 * chem_integrate* calls on this ctx write row 0 = active cells per box after the gate and row i =
 * active cells per box after bulk launch i (i < rows; each launch is K_max attempted substeps per
 * cell).  rows = 0 (or trace = NULL with rows = 0) turns tracing off. */
int chem_set_trace(chem_ctx* ctx, int32_t* trace, int32_t rows);

/* Test hooks and caller-side helpers ------------------------------------------------------ */
/* T = Newton(e, Y) seeded with the incoming T.  T in/out [n]. */
int chem_temperature(chem_ctx* ctx, int64_t n, int64_t ld, const double* e, const double* Y,
                     double* T, void* stream);
/* PAPER.md Alg. 1, the caller-side step before chemistry: e = rho E/rho - |u|^2/2 from the
 * conserved variables U[c*ld + i], c = 0..4 = rho, rho u_x, rho u_y, rho u_z, rho E (DEVICE). */
int chem_internal_energy(chem_ctx* ctx, int64_t n, int64_t ld, const double* U, double* e, void* stream);
/* e = u(T, Y) = sum_k Y_k eps_k(T)/W_k (the inverse of chem_temperature). */
int chem_energy(chem_ctx* ctx, int64_t n, int64_t ld, const double* T, const double* Y, double* e,
                void* stream);
/* Analytic Jacobian of the ODE right-hand side w.r.t. y = (Y_1..Y_ns, T), n_unk = ns + 1:
 * J[(i*n_unk + j)*ld + cell] = d f_i / d y_j (rows of inert species are zero). */
int chem_jacobian(chem_ctx* ctx, int64_t n, int64_t ld, const double* rho, const double* T,
                  const double* Y, double* J, void* stream);
/* ODE right-hand side f = dy/dt, f[(i)*ld + cell], i < ns + 1 (Eq. 5 and corrected Eq. 6). */
int chem_rhs(chem_ctx* ctx, int64_t n, int64_t ld, const double* rho, const double* T,
             const double* Y, double* f, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CHEM_H */
