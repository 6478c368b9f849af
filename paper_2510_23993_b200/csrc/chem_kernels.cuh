// chem_kernels.cuh — the sm_100a kernels of the bulk-sparse schedule (Alg. 3).
//
//   k_gate       A1/A2  gate + count + cell index map (ballot / block scan, one atomic per block)
//   k_integrate  A1/A6/A7/A9  bulk burst (<= K_max substeps per cell, one thread per id) and the
//                sparse launch (persistent grid; a lane whose cell finishes takes the next id from
//                an atomic cursor, so warps stay full through the long tail)
//   k_compact    A8     still-active ids -> next index map (ballot / block scan)
//   k_box_cost   A10    per-box attempted substeps (box cost for load balancing)
//   k_rates / k_rhs / k_jacobian / k_temperature / k_energy: point evaluations (C-ABI test hooks)
//
// Multi-box fusion (A10): a global cell id g indexes the concatenation of all boxes;
// box b = upper_bound(box_start, g) - 1, offset = g - box_start[b].  One launch per phase spans
// every box; no data is copied (the kernels read and write the caller's arrays in place).
#pragma once
#include "chem_device.cuh"

namespace chem {

enum CellState : uint8_t {
    ST_INACTIVE = 0,   // gated out (T < T_min or solid): never touched
    ST_FRESH = 1,      // active, not started (needs the initial Newton T)
    ST_RUNNING = 2,    // active, t < dt, state persisted in the caller's arrays + workspace
    ST_DONE = 3,       // reached t = dt
    ST_UNFINISHED = 4, // sparse K_max exhausted (P:179 safeguard)
    ST_FAILED = 5,     // Newton failure / non-finite / step-size underflow
};

enum StatIdx {
    S_ATTEMPTED = 0, S_ACCEPTED, S_RHS, S_JAC, S_LU, S_NEWTON_FAIL, S_NONFINITE, S_TRANGE, S_UNFINISHED,
    S_DONE, S_DRIFT_BITS, S_COUNT_ACTIVE, S_CURSOR, S_FROZEN, S_WARP_SUBSTEPS, S_PRED_TOTAL, S_PRED_HEAVY,
    S_PRED_MAX,
    S_PRED2_TOTAL, S_PRED2_MAX,   // in-call prediction after the first burst (sum, max of remaining substeps)
    S_SIG0, S_SIG1, S_SIG2,   // cell-layout signature of the workspace's cost hints (not cleared per call)
    S_HINT_MIN, S_HINT_MAX,   // sum over finished cells of min / max(hint, actual substeps): hint accuracy
    S_HINT_VALID,             // 1 if those sums describe valid hints (the call had the layout's history)
    S_NSTATS
};

struct DevBox {
    const double* rho;
    const double* e;
    double* T;
    double* Y;
    const uint8_t* solid;
    int64_t ncells, ld;
    double dt;
};

struct LaunchCtx {
    const DevBox* boxes;
    const int64_t* box_start;  // [nboxes + 1] prefix of ncells
    int32_t nboxes;
    int64_t total;
    double* cell_t;            // [total] local time t_i
    double* cell_h;            // [total] next substep size
    uint8_t* state;            // [total] CellState (+ bit 7: last step rejected)
    int32_t* cell_steps;       // [total] attempted substeps summed over launches
    int32_t* cell_box;         // [total] box of each active cell (written by the gate: one coalesced
                               // load in load_cell instead of a dependent-load binary search)
    int32_t* cell_hint;        // [total] the previous call's substeps of the cell (its cost hint),
                               // compared with the actual count at write-back (hint accuracy)
    unsigned long long* stats; // [S_NSTATS]
    double rtol, atol, atolT, T_min;
    double eps_change;          // explicit scheme: max fractional change per step
    double h0_factor;           // initial substep = h0_factor |y|/|f| (Hairer-Norsett-Wanner: 0.01)
    int32_t kmax_call;          // per-cell budget of attempted substeps over the whole call
                                // (chem_opts.kmax_sparse): reached in any launch -> ST_UNFINISHED
};

__device__ __forceinline__ int find_box(const LaunchCtx& L, int64_t g)
{
    int lo = 0, hi = L.nboxes - 1;
    while (lo < hi) {  // last b with box_start[b] <= g
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&L.box_start[mid]) <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Full-warp add of a per-lane value to a device counter.  Every lane of the warp must call it
// (callers __syncwarp() first); xor-shuffles with a partial mask would read inactive lanes.
__device__ __forceinline__ void warp_add(unsigned long long* p, unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(p, v);
}

// Block-wide stream compaction helper: each thread has flag `keep` and id `g`; kept ids are
// written to out[] at positions reserved with one atomicAdd per block.  Order within a block
// follows thread order.  Requires all threads of the block to call it.
template <int BS>
__device__ __forceinline__ void block_compact(bool keep, uint32_t g, uint32_t* out, unsigned long long* counter,
                                              uint32_t key = 0, uint32_t* key_out = nullptr)
{
    __shared__ int warp_cnt[BS / 32];
    __shared__ unsigned long long base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_cnt[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < BS / 32; ++w) { const int c = warp_cnt[w]; warp_cnt[w] = s; s += c; }
        base = s ? atomicAdd(counter, (unsigned long long)s) : 0ull;
    }
    __syncthreads();
    if (keep) {
        const unsigned long long at = base + warp_cnt[wid] + __popc(bal & ((1u << lane) - 1u));
        out[at] = g;
        if (key_out) key_out[at] = key;
    }
    __syncthreads();
}

// ----------------------------------------------------------------------------- A2 gate + count
// keys_out (nullable): each listed cell's attempted substeps in the previous call at the same index
// (the cost hint of the heavy-first schedule); S_PRED_TOTAL / S_PRED_HEAVY sum that hint over the
// active cells and over those above kHeavySteps.
constexpr uint32_t kHeavySteps = 64;

template <int BS>
__global__ void __launch_bounds__(BS) k_gate(LaunchCtx L, uint32_t* ids_out, uint32_t* keys_out)
{
    for (int64_t base = (int64_t)blockIdx.x * BS; base < L.total; base += (int64_t)gridDim.x * BS) {
        const int64_t g = base + threadIdx.x;
        bool act = false;
        uint32_t prev = 0;
        if (g < L.total) {
            const int b = find_box(L, g);
            const DevBox bx = L.boxes[b];
            const int64_t off = g - L.box_start[b];
            const double T = bx.T[off];
            act = (T >= L.T_min) && !(bx.solid && bx.solid[off]);   // Alg. 3 §1
            L.state[g] = act ? ST_FRESH : ST_INACTIVE;
            if (keys_out) prev = act ? (uint32_t)max(L.cell_steps[g], 0) : 0u;
            L.cell_steps[g] = 0;
            if (act) {
                L.cell_box[g] = b;
                L.cell_hint[g] = (int32_t)prev;
            }
        }
        if (keys_out) {
            warp_add(&L.stats[S_PRED_TOTAL], prev);
            warp_add(&L.stats[S_PRED_HEAVY], prev > kHeavySteps ? prev : 0u);
            unsigned mx = prev;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((threadIdx.x & 31) == 0 && mx) atomicMax(&L.stats[S_PRED_MAX], (unsigned long long)mx);
        }
        block_compact<BS>(act, (uint32_t)g, ids_out, &L.stats[S_COUNT_ACTIVE], prev, keys_out);
    }
}

// In-call cost prediction (heavy-first without cross-call hints, chem_opts.schedule_lpt 2/3): after the
// first bulk burst every still-active cell's remaining substeps are estimated from its own state as
// (dt - t) / h (h = the step the controller proposes next); keys_out[i] pairs with ids[i].
template <int BS>
__global__ void __launch_bounds__(BS) k_predict(LaunchCtx L, const uint32_t* ids, int64_t n, uint32_t* keys_out)
{
    for (int64_t base = (int64_t)blockIdx.x * BS; base < n; base += (int64_t)gridDim.x * BS) {
        const int64_t i = base + threadIdx.x;
        uint32_t key = 0;
        if (i < n) {
            const uint32_t g = ids[i];
            const double dt = L.boxes[L.cell_box[g]].dt;
            const double h = L.cell_h[g];
            const double rem = h > 0.0 ? (dt - L.cell_t[g]) / h : 16777215.0;
            key = (uint32_t)fmin(fmax(rem, 1.0), 16777215.0);
            keys_out[i] = key;
        }
        warp_add(&L.stats[S_PRED2_TOTAL], key);
        unsigned mx = key;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0 && mx) atomicMax(&L.stats[S_PRED2_MAX], (unsigned long long)mx);
    }
}

// Heavy-first ordering without a library sort: a STABLE counting sort of the cell list into 256 cost
// buckets (bucket = floor(16 log2 cost): 1/16-octave resolution up to 2^16 substeps), heaviest bucket
// first; within a bucket the list order is kept (neighbouring cells stay together: coalesced loads and
// similar cells per warp).  Three passes over tiles of kSortTile entries:
//   k_bucket_hist    per-tile bucket counts -> hist[(255 - bucket) * ntiles + tile]
//   k_scan_excl      exclusive scan of hist (heaviest bucket first, tiles in order)
//   k_bucket_scatter each tile places its entries in order (warp match + per-warp prefix)
constexpr int kCostBuckets = 256;
constexpr int kSortBS = 256;
constexpr int kSortTile = 4 * kSortBS;

// bucket = floor(16 log2 key) (1/16-octave resolution up to 2^16 substeps): 4 bits below the leading one
__device__ __forceinline__ int cost_bucket(uint32_t key)
{
    if (key <= 1u) return 0;
    const int e = 31 - __clz(key);                         // floor(log2 key)
    const int q = e >= 4 ? (int)(key >> (e - 4)) & 15 : (int)(key << (4 - e)) & 15;
    return min(kCostBuckets - 1, 16 * e + q);
}

static __global__ void __launch_bounds__(kSortBS) k_bucket_hist(const uint32_t* keys, int64_t n, unsigned* hist,
                                                         int ntiles)
{
    __shared__ unsigned h[kCostBuckets];
    for (int i = threadIdx.x; i < kCostBuckets; i += kSortBS) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortTile / kSortBS; ++r) {
        const int64_t i = base + r * kSortBS + threadIdx.x;
        if (i < n) atomicAdd(&h[cost_bucket(keys[i])], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kCostBuckets; b += kSortBS) hist[(kCostBuckets - 1 - b) * ntiles + blockIdx.x] = h[b];
}

// exclusive scan of m entries in place, one block of 1024 threads
static __global__ void __launch_bounds__(1024) k_scan_excl(unsigned* v, int64_t m)
{
    __shared__ unsigned part[1024];
    const int64_t per = (m + 1023) / 1024;
    const int64_t lo = threadIdx.x * per, hi = min(m, lo + per);
    unsigned s = 0;
    for (int64_t i = lo; i < hi; ++i) s += v[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {               // Hillis-Steele inclusive scan of the partials
        const unsigned add = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    unsigned run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
    for (int64_t i = lo; i < hi; ++i) {
        const unsigned c = v[i];
        v[i] = run;
        run += c;
    }
}

static __global__ void __launch_bounds__(kSortBS) k_bucket_scatter(const uint32_t* keys, const uint32_t* ids_in, int64_t n,
                                                            const unsigned* offs, int ntiles, uint32_t* ids_out)
{
    constexpr int NW = kSortBS / 32;
    __shared__ unsigned run[kCostBuckets];             // entries of each bucket placed by earlier rounds
    __shared__ unsigned tot[kCostBuckets];             // this round's entries per bucket
    __shared__ unsigned wcnt[NW][kCostBuckets];        // this round: per-warp counts -> exclusive prefixes
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b = threadIdx.x; b < kCostBuckets; b += kSortBS) run[b] = 0;
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortTile / kSortBS; ++r) {
        for (int b = threadIdx.x; b < NW * kCostBuckets; b += kSortBS) (&wcnt[0][0])[b] = 0;
        __syncthreads();
        const int64_t i = base + r * kSortBS + threadIdx.x;
        const bool valid = i < n;
        const int bk = valid ? cost_bucket(keys[i]) : kCostBuckets;    // invalid lanes: a bucket of their own
        const unsigned peers = __match_any_sync(0xffffffffu, bk);
        const unsigned rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) wcnt[w][bk] = __popc(peers);
        __syncthreads();
        if (threadIdx.x < kCostBuckets) {               // per bucket: exclusive prefix over the warps
            unsigned acc = 0;
            for (int ww = 0; ww < NW; ++ww) {
                const unsigned c = wcnt[ww][threadIdx.x];
                wcnt[ww][threadIdx.x] = acc;
                acc += c;
            }
            tot[threadIdx.x] = acc;
        }
        __syncthreads();
        if (valid) {
            const unsigned at = offs[(kCostBuckets - 1 - bk) * ntiles + blockIdx.x] + run[bk] + wcnt[w][bk] + rank;
            ids_out[at] = ids_in[i];
        }
        __syncthreads();
        if (threadIdx.x < kCostBuckets) run[threadIdx.x] += tot[threadIdx.x];
    }
}

// ----------------------------------------------------------------------------- A8 compaction
template <int BS>
__global__ void __launch_bounds__(BS) k_compact(LaunchCtx L, const uint32_t* ids_in, int64_t n_in, uint32_t* ids_out)
{
    for (int64_t base = (int64_t)blockIdx.x * BS; base < n_in; base += (int64_t)gridDim.x * BS) {
        const int64_t i = base + threadIdx.x;
        uint32_t g = 0;
        bool keep = false;
        if (i < n_in) {
            g = ids_in ? ids_in[i] : (uint32_t)i;
            const uint8_t s = L.state[g] & 0x7f;
            keep = (s == ST_RUNNING) || (s == ST_FRESH);
        }
        block_compact<BS>(keep, g, ids_out, &L.stats[S_COUNT_ACTIVE]);
    }
}

// ----------------------------------------------------------------------------- A10 box cost
template <int BS>
__global__ void __launch_bounds__(BS) k_box_cost(LaunchCtx L, const uint32_t* ids, int64_t n, double* box_cost)
{
    // every lane iterates the same number of times so warp collectives see a full mask
    for (int64_t base = (int64_t)blockIdx.x * BS; base < n; base += (int64_t)gridDim.x * BS) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const uint32_t g = valid ? ids[i] : 0u;
        const int b = valid ? find_box(L, g) : -1;
        const double v = valid ? (double)L.cell_steps[g] : 0.0;
        const int b0 = __shfl_sync(0xffffffffu, b, 0);
        if (__all_sync(0xffffffffu, !valid || b == b0)) {
            double s = v;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if ((threadIdx.x & 31) == 0 && b0 >= 0) atomicAdd(&box_cost[b0], s);
        } else if (valid) {
            atomicAdd(&box_cost[b], v);
        }
    }
}

// Activity trace (App. B): active cells of the index map per box.
template <int BS>
__global__ void __launch_bounds__(BS) k_box_count(LaunchCtx L, const uint32_t* ids, int64_t n, int32_t* row)
{
    for (int64_t base = (int64_t)blockIdx.x * BS; base < n; base += (int64_t)gridDim.x * BS) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const int b = valid ? find_box(L, ids[i]) : -1;
        const int b0 = __shfl_sync(0xffffffffu, b, 0);
        if (__all_sync(0xffffffffu, !valid || b == b0)) {
            const int c = __popc(__ballot_sync(0xffffffffu, valid));
            if ((threadIdx.x & 31) == 0 && b0 >= 0) atomicAdd(&row[b0], c);
        } else if (valid) {
            atomicAdd(&row[b], 1);
        }
    }
}

// ----------------------------------------------------------------------------- A6/A7/A9 integrate
// Per-thread shared memory (stride = block size, conflict-free): the n x n iteration matrix
// (I/(h gamma) - J, then its LU) and the stored stage vectors K_s (pivot rows stay in registers);
// n = NSA+1 unknowns (reacting Y_k and T, Eq. 6).  Stiffly accurate methods (RODAS4) do not store
// the last stage: y_new = Y_last + K_last and err = K_last.
template <class M, class Meth>
struct SmemLayout {
    static constexpr int n = M::NSA + 1;
    static constexpr bool none = (Meth::S == 0);   // explicit scheme: no matrix, no stages
    // stage slots: RODAS4 keeps three (ros_step's collapse), stiffly accurate methods S-1, others S
    static constexpr int nK = Meth::collapse ? 3 : (Meth::stiff_last ? Meth::S - 1 : Meth::S);
    static constexpr int off_K = none ? 0 : n * n;
    static constexpr int doubles = none ? 0 : n * n + nK * n;   // pivots are kept in registers
    static constexpr int bytes_per_thread = doubles * 8;
};

struct Counters {
    unsigned attempted = 0, accepted = 0, rhs = 0, newton_fail = 0, nonfinite = 0, trange = 0, unfinished = 0,
             done = 0, frozen = 0, warp_substeps = 0, hint_min = 0, hint_max = 0;
    double drift = 0.0;
};

template <class M>
struct Cell {
    double y[M::NSA + 1];  // integrated unknowns: reacting Y_k, T
    double Yin[M::NS];     // all species (inert ones stay constant)
    double rho, e, t, h, dt;
    int b;
    int64_t off, ld;
    uint32_t g;
    int k;                 // attempted substeps in this launch
    int kprev;             // attempted substeps in earlier launches of this call (the call budget)
    bool rej;              // last step rejected (controller memory, persisted in state bit 7)
};

// One attempted Rosenbrock substep on cell C (A6).  Returns 1 accepted, 0 rejected, -1 failure.
// The stage loop is a runtime loop (one inlined copy of the RHS in the kernel: the fully
// unrolled version overflowed the instruction cache); stage vectors live in shared memory.
template <class M, class Meth>
__device__ __forceinline__ int ros_step(const Params<M>& P, const LaunchCtx& L, Cell<M>& C, const SMat& A,
                                        double* Ks, int ss, Counters& cnt)
{
    constexpr int n = M::NSA + 1;
    constexpr int S = Meth::S;
    const double invrho = frcp(C.rho);
    double f0[n];
    rhs_jac<M, JAC_ODE>(P, C.rho, C.y, C.Yin, f0, A);
    cnt.rhs++;
    const double remaining = C.dt - C.t;
    if (!(C.h > 0.0)) {
        // initial step: 1% of the time for y to change by its own size (the d0/d1 heuristic of
        // Hairer-Norsett-Wanner I, II.4), capped at dt.
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
            const double sc = ((i < M::NSA) ? L.atol : L.atolT) + L.rtol * fabs(C.y[i]);
            d0 = fma(C.y[i] / sc, C.y[i] / sc, d0);
            d1 = fma(f0[i] / sc, f0[i] / sc, d1);
        }
        d0 = sqrt(d0 / n);
        d1 = sqrt(d1 / n);
        if (d1 * remaining < 1e-3) {
            // frozen / inert / equilibrated cell (the north_star's "cheap bulk step"): f moves y by
            // < 1e-3 tolerance units over the whole interval, so one explicit step y += dt f(y)
            // is within that bound by construction; skip the LU and the stages.
#pragma unroll
            for (int i = 0; i < n; ++i) C.y[i] = fma(remaining, f0[i], C.y[i]);
            C.t = C.dt;
            C.k++;
            cnt.attempted++;
            cnt.accepted++;
            cnt.frozen++;
            return 1;
        }
        C.h = (d0 < 1e-5) ? remaining : fmin(remaining, L.h0_factor * d0 / d1);
    }
    bool last = false;
    double h = C.h;
    if (h >= remaining) { h = remaining; last = true; }
    if (!(h > 4.0 * 2.220446049250313e-16 * C.dt) || !isfinite(h)) return -1;  // step-size underflow

    // iteration matrix A = I/(h gamma) - J, LU in place (rhs_jac left -J in A)
    const double ghinv = 1.0 / (h * Meth::gamma);
#pragma unroll
    for (int i = 0; i < n; ++i) A(i, i) = ghinv + A(i, i);
    uint64_t perm;
    const bool ok = lu_factor<n>(A, perm);

    const double hinv = 1.0 / h;
    double ylast[n];                          // stage point of the last stage (stiffly accurate)
    auto slot = [&](int j) { return Ks + (j * n) * ss; };
    if constexpr (Meth::collapse) {
        // RODAS4 in three stage slots S0..S2.  Stages 1-3 read the raw K_0..K_2; after stage 3's
        // point and correction are formed, the slots are collapsed in place into the partial sums
        // stages 4-5 need (a_5j = a_4j for j < 4, a_54 = 1; stiffly accurate):
        //   S0 = sum_j a_4j K_j,  S1 = sum_j c_4j K_j,  S2 = sum_j c_5j K_j   (j < 3)
        // and every later K_s is scatter-added into them (K_3 into all three, K_4 into S0 with
        // a_54 = 1 and into S2).  Stage 4 reads (S0, S1), stage 5 reads (S0, S2) and K_5 lands in
        // the free S1.  Same sums as the textbook form, different rounding order.
        {
            double x[n];
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = f0[i];
            lu_solve<n>(A, x);
            scatter_perm<n>(perm, x, slot(0), ss);
        }
#pragma unroll 1
        for (int s = 1; s < S; ++s) {
            double F[n];
            double ys[n];
            // stage point first; the sum_j c_sj K_j / h term is formed after the RHS from the slots
            // again, so it is not live across the rate evaluation (register pressure)
            if (s <= 3) {
#pragma unroll
                for (int i = 0; i < n; ++i) ys[i] = C.y[i];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    if (j < s) {
                        const double a = Meth::a_rt(s, j);
#pragma unroll
                        for (int i = 0; i < n; ++i) ys[i] = fma(a, slot(j)[i * ss], ys[i]);
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < n; ++i) ys[i] = C.y[i] + slot(0)[i * ss];
            }
            rhs<M>(P, C.rho, invrho, ys, C.Yin, F);
            cnt.rhs++;
            if (s <= 3) {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    if (j < s) {
                        const double c = Meth::c_rt(s, j) * hinv;
#pragma unroll
                        for (int i = 0; i < n; ++i) F[i] = fma(c, slot(j)[i * ss], F[i]);
                    }
                }
            } else {
                const double* gs = slot(s == 4 ? 1 : 2);
#pragma unroll
                for (int i = 0; i < n; ++i) F[i] = fma(hinv, gs[i * ss], F[i]);
            }
            if (s == 3) {
                // collapse (K_0, K_1, K_2) -> (sum a_4j K_j, sum c_4j K_j, sum c_5j K_j), j < 3
                const double a0 = Meth::a_rt(4, 0), a1 = Meth::a_rt(4, 1), a2 = Meth::a_rt(4, 2);
                const double c0 = Meth::c_rt(4, 0), c1 = Meth::c_rt(4, 1), c2 = Meth::c_rt(4, 2);
                const double d0 = Meth::c_rt(5, 0), d1 = Meth::c_rt(5, 1), d2 = Meth::c_rt(5, 2);
#pragma unroll
                for (int i = 0; i < n; ++i) {
                    const double k0 = slot(0)[i * ss], k1 = slot(1)[i * ss], k2 = slot(2)[i * ss];
                    slot(0)[i * ss] = fma(a2, k2, fma(a1, k1, a0 * k0));
                    slot(1)[i * ss] = fma(c2, k2, fma(c1, k1, c0 * k0));
                    slot(2)[i * ss] = fma(d2, k2, fma(d1, k1, d0 * k0));
                }
            }
            lu_solve<n>(A, F);
            if (s < 3) {
                scatter_perm<n>(perm, F, slot(s), ss);
            } else if (s == 3) {
                scatter_perm<n, true>(perm, F, slot(0), ss, Meth::a_rt(4, 3));
                scatter_perm<n, true>(perm, F, slot(1), ss, Meth::c_rt(4, 3));
                scatter_perm<n, true>(perm, F, slot(2), ss, Meth::c_rt(5, 3));
            } else if (s == 4) {
                scatter_perm<n, true>(perm, F, slot(0), ss, Meth::a_rt(5, 4));
                scatter_perm<n, true>(perm, F, slot(2), ss, Meth::c_rt(5, 4));
            } else {
                scatter_perm<n>(perm, F, slot(1), ss);   // K_5 (natural order) in the free slot
#pragma unroll
                for (int i = 0; i < n; ++i) ylast[i] = ys[i];
            }
        }
    } else {
        double Flast[Meth::reuse_last ? n : 1];   // f of the last new stage point (methods reusing it)
        {   // stage 0: K_0 = A^{-1} f(y)
            double x[n];
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = f0[i];
            if constexpr (Meth::reuse_last) {
#pragma unroll
                for (int i = 0; i < n; ++i) Flast[i] = f0[i];
            }
            lu_solve<n>(A, x);
            scatter_perm<n>(perm, x, slot(0), ss);
        }
#pragma unroll 1
        for (int s = 1; s < S; ++s) {
            double F[n];
            double ys[n];
#pragma unroll
            for (int i = 0; i < n; ++i) ys[i] = C.y[i];
            if (!Meth::reuse_last || Meth::newf_rt(s)) {
#pragma unroll
                for (int j = 0; j < S - 1; ++j) {
                    if (j < s) {
                        const double a = Meth::a_rt(s, j);
#pragma unroll
                        for (int i = 0; i < n; ++i) ys[i] = fma(a, slot(j)[i * ss], ys[i]);
                    }
                }
                rhs<M>(P, C.rho, invrho, ys, C.Yin, F);
                cnt.rhs++;
                if constexpr (Meth::reuse_last) {
#pragma unroll
                    for (int i = 0; i < n; ++i) Flast[i] = F[i];
                }
            } else {
                // the stage point equals the previous new one (a_sj = a_(s-1)j): reuse its f
#pragma unroll
                for (int i = 0; i < n; ++i) F[i] = Flast[i];
            }
#pragma unroll
            for (int j = 0; j < S - 1; ++j) {
                if (j < s) {
                    const double c = Meth::c_rt(s, j) * hinv;
#pragma unroll
                    for (int i = 0; i < n; ++i) F[i] = fma(c, slot(j)[i * ss], F[i]);
                }
            }
            lu_solve<n>(A, F);
            // the last stage of a stiffly accurate method goes to slot 0 (K_0 is no longer needed)
            const bool last_stage = Meth::stiff_last && (s == S - 1);
            scatter_perm<n>(perm, F, slot(last_stage ? 0 : s), ss);
            if (last_stage) {
#pragma unroll
                for (int i = 0; i < n; ++i) ylast[i] = ys[i];
            }
        }
    }

    double ynew[n];
    double err = 0.0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
        double v, ev;
        if constexpr (Meth::stiff_last) {
            const double xl = slot(Meth::collapse ? 1 : 0)[i * ss];   // K_last
            v = ylast[i] + xl;            // y + sum m_j K_j = Y_last + K_last
            ev = xl;                      // sum e_j K_j = K_last
        } else {
            v = C.y[i];
            ev = 0.0;
            static_for<0, S>([&](auto j_) {
                constexpr int j = decltype(j_)::value;
                const double kj = slot(j)[i * ss];
                if constexpr (Meth::m(j) != 0.0) v = fma(Meth::m(j), kj, v);
                if constexpr (Meth::e(j) != 0.0) ev = fma(Meth::e(j), kj, ev);
            });
        }
        ynew[i] = v;
        const double s = ((i < M::NSA) ? L.atol : L.atolT) + L.rtol * fmax(fabs(C.y[i]), fabs(v));
        const double q = ev * frcp(s);
        err = fma(q, q, err);
    }
    err = sqrt(err * (1.0 / n));
    cnt.attempted++;
    C.k++;
    if (!ok || !isfinite(err)) {  // singular matrix or non-finite stage: shrink hard, retry
        C.h = h * 0.1;
        C.rej = true;
        return 0;
    }
    // step-size controller (Hairer-Wanner IV.8; KPP Rosenbrock): safety 0.9, factor in [0.2, 6]
    double fac;
    if constexpr (Meth::err_exp == 0.25) fac = 0.9 / sqrt(sqrt(err));   // err^(-1/4) without libdevice pow
    else fac = 0.9 * pow(err, -Meth::err_exp);
    fac = fmin(6.0, fmax(0.2, fac));
    double hnew = h * fac;
    if (err <= 1.0) {
        cnt.accepted++;
#pragma unroll
        for (int i = 0; i < n; ++i) C.y[i] = ynew[i];
        C.t = last ? C.dt : C.t + h;
        if (C.rej) hnew = fmin(hnew, h);
        C.rej = false;
        C.h = hnew;
        return 1;
    }
    C.h = C.rej ? h * 0.1 : hnew;  // repeated rejection: factor 0.1
    C.rej = true;
    return 0;
}

// One step of the paper's explicit scheme (struct Explicit).  The
// integrated unknowns are Y; y[NSA] holds T = Newton(e, Y) after every step.  Returns 1, or -1 when
// the step cannot proceed (non-finite rate or Newton failure).
template <class M>
__device__ __forceinline__ int explicit_step(const Params<M>& P, const LaunchCtx& L, Cell<M>& C, double eps,
                                             Counters& cnt)
{
    constexpr int n = M::NSA + 1;
    double f[n];
    rhs<M>(P, C.rho, 1.0 / C.rho, C.y, C.Yin, f);
    cnt.rhs++;
    const double remaining = C.dt - C.t;
    double rmin = INFINITY;
#pragma unroll
    for (int i = 0; i < M::NSA; ++i)
        if (C.y[i] > Explicit::Y_floor && f[i] != 0.0) rmin = fmin(rmin, C.y[i] / fabs(f[i]));
    double h = eps * rmin;
    bool last = !(h < remaining * (1.0 - 1e-10));   // no sliver step from the rounding of t += h
    if (last) h = remaining;
    bool finite = true;
#pragma unroll
    for (int i = 0; i < M::NSA; ++i) {
        C.y[i] = fmax(fma(h, f[i], C.y[i]), 0.0);   // clip to 0, no renormalisation
        finite = finite && isfinite(C.y[i]);
    }
    double Yf[M::NS];
    full_Y<M>(C.y, C.Yin, Yf);
    double T = C.y[M::NSA];
    const bool ok = newton_T<M>(P, C.e, Yf, T) && finite;
    C.y[M::NSA] = T;
    C.t = last ? C.dt : C.t + h;
    C.k++;
    cnt.attempted++;
    cnt.accepted++;
    if (!ok) { cnt.newton_fail++; return -1; }
    return 1;
}

template <class M>
__device__ __forceinline__ void load_cell(const Params<M>& P, const LaunchCtx& L, uint32_t g, Cell<M>& C,
                                          uint8_t st, Counters& cnt, bool& ok)
{
    C.g = g;
    C.b = L.cell_box[g];
    const DevBox bx = L.boxes[C.b];
    C.off = g - L.box_start[C.b];
    C.ld = bx.ld;
    C.dt = bx.dt;
    C.rho = bx.rho[C.off];
    C.e = bx.e[C.off];
#pragma unroll
    for (int k = 0; k < M::NS; ++k) C.Yin[k] = bx.Y[k * C.ld + C.off];   // coalesced: consecutive ids
#pragma unroll
    for (int i = 0; i < M::NSA; ++i) C.y[i] = C.Yin[M::act(i)];
    double T = bx.T[C.off];
    C.k = 0;
    C.kprev = L.cell_steps[g];
    ok = true;
    if ((st & 0x7f) == ST_FRESH) {
        // initial temperature from (e, Y) at constant (e, rho), seeded with the input T
        if (!newton_T<M>(P, C.e, C.Yin, T)) { cnt.newton_fail++; ok = false; }
        C.t = 0.0;
        C.h = 0.0;
        C.rej = false;
    } else {
        C.t = L.cell_t[g];
        C.h = L.cell_h[g];
        C.rej = (st & 0x80) != 0;
    }
    C.y[M::NSA] = T;
}

// Write back: running cells persist (Y, T_int) in place and (t, h, flags) in the workspace;
// finished cells store Y_out and T_out = Newton(e, Y_out) (SURVEY reading 3).
template <class M>
__device__ __forceinline__ void store_cell(const Params<M>& P, const LaunchCtx& L, Cell<M>& C, uint8_t st,
                                           Counters& cnt)
{
    const DevBox bx = L.boxes[C.b];
#pragma unroll
    for (int i = 0; i < M::NSA; ++i) bx.Y[M::act(i) * C.ld + C.off] = C.y[i];
    double T = C.y[M::NSA];
    if (st == ST_DONE || st == ST_UNFINISHED) {
        double Yf[M::NS];
        full_Y<M>(C.y, C.Yin, Yf);
        const double Tint = T;
        if (!newton_T<M>(P, C.e, Yf, T)) { cnt.newton_fail++; st = ST_FAILED; }
        if (st == ST_DONE) {
            cnt.done++;
            cnt.drift = fmax(cnt.drift, fabs(Tint - T) / T);
            if (T < P.T_valid_lo || T > P.T_valid_hi) cnt.trange++;
        } else {
            cnt.unfinished++;
        }
    }
    bx.T[C.off] = T;
    L.cell_t[C.g] = C.t;
    L.cell_h[C.g] = C.h;
    L.state[C.g] = st | (C.rej ? 0x80 : 0);
    L.cell_steps[C.g] = C.kprev + C.k;
    if (st != ST_RUNNING) {   // the cell's call is over: how well did its hint predict it?
        const unsigned act = (unsigned)(C.kprev + C.k), hint = (unsigned)L.cell_hint[C.g];
        cnt.hint_min += min(act, hint);
        cnt.hint_max += max(act, hint);
    }
}

__device__ __forceinline__ void flush_counters(const LaunchCtx& L, Counters& c)
{
    warp_add(&L.stats[S_ATTEMPTED], c.attempted);
    warp_add(&L.stats[S_ACCEPTED], c.accepted);
    warp_add(&L.stats[S_RHS], c.rhs);
    warp_add(&L.stats[S_JAC], c.attempted);              // one Jacobian per attempted substep
    warp_add(&L.stats[S_LU], c.attempted - c.frozen);    // one LU per attempted Rosenbrock substep
    warp_add(&L.stats[S_FROZEN], c.frozen);
    warp_add(&L.stats[S_WARP_SUBSTEPS], c.warp_substeps);
    warp_add(&L.stats[S_NEWTON_FAIL], c.newton_fail);
    warp_add(&L.stats[S_NONFINITE], c.nonfinite);
    warp_add(&L.stats[S_TRANGE], c.trange);
    warp_add(&L.stats[S_UNFINISHED], c.unfinished);
    warp_add(&L.stats[S_DONE], c.done);
    warp_add(&L.stats[S_HINT_MIN], c.hint_min);
    warp_add(&L.stats[S_HINT_MAX], c.hint_max);
    // max drift: non-negative doubles order like their bit patterns
    unsigned long long bits = __double_as_longlong(c.drift);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, bits, o);
        bits = v > bits ? v : bits;
    }
    if ((threadIdx.x & 31) == 0 && bits) atomicMax(&L.stats[S_DRIFT_BITS], bits);
}

// Bulk (refill = 0): thread i takes ids[i] (identity when ids == nullptr, the paper's
// all-cells launch) and runs <= kmax attempted substeps.  Sparse (refill = b >= 1): persistent
// grid; each lane pulls ids from the atomic cursor S_CURSOR until the list is exhausted, the idle
// lanes of a warp that still has busy lanes waiting until b of them are idle (the host passes 1 for a
// cost-sorted list, where neighbouring entries cost alike and refilling at once is fastest — cfg3 195.8
// -> 200.7, cfg5 279.2 -> 294.3 Mcell-steps/s against b = 8, r02v — and a quarter warp for the
// gate-ordered list of Alg. 3, where joint loads of a batch win: sparse-only cfg3 61 (b = 1) vs 92, r02
// NEXT-2 sweeps).
// Both modes run the same substep code, so results are bitwise independent of K_max and N*.
// LOCK: the block's warps take each substep together (one __syncthreads_or per substep), so that on a
// heterogeneous field the SM's resident warps stay in the same code region (shared instruction cache)
// instead of drifting apart; a thread whose cell has left the burst idles at the barrier.
template <class M, class Meth, int BS, bool LOCK = false>
__global__ void __launch_bounds__(BS) k_integrate(const __grid_constant__ Params<M> P, LaunchCtx L,
                                                  const uint32_t* __restrict__ ids, int64_t n_ids, int kmax,
                                                  int refill, int final_phase)
{
    extern __shared__ double smem[];
    fm_tables_to_smem();
    using SL = SmemLayout<M, Meth>;
    constexpr int n = SL::n;
    double* mine = smem + threadIdx.x;
    SMat A{mine, BS, n};
    double* Ks = mine + SL::off_K * BS;

    Counters cnt;
    Cell<M> C;
    bool have = false;
    bool live = true;     // this thread may still take a cell
    bool first = true;
    int64_t tile = blockIdx.x;
    int64_t next_idx = 0;  // free-running bulk: the list entry this thread took last
    // one attempted substep of the lane's cell and its write-back when the cell leaves the launch
    auto substep = [&]() {
        {   // SIMT efficiency statistic: the lowest lane executing this substep counts one warp substep
            const unsigned am = __activemask();
            if ((int)(threadIdx.x & 31) == __ffs(am) - 1) cnt.warp_substeps++;
        }
        int r;
        if constexpr (Meth::S == 0) r = explicit_step<M>(P, L, C, L.eps_change, cnt);
        else r = ros_step<M, Meth>(P, L, C, A, Ks, BS, cnt);
        if (r < 0) {
            cnt.nonfinite++;
            store_cell<M>(P, L, C, ST_FAILED, cnt);
            have = false;
        } else if (C.t >= C.dt) {
            store_cell<M>(P, L, C, ST_DONE, cnt);
            have = false;
        } else if (C.kprev + C.k >= L.kmax_call) {
            // the call's per-cell budget of attempted substeps is spent, whichever launch (bulk
            // burst, sparse or heavy-first) the cell is in: the schedules stay bitwise equivalent
            store_cell<M>(P, L, C, ST_UNFINISHED, cnt);
            have = false;
        } else if (C.k >= kmax) {
            store_cell<M>(P, L, C, final_phase ? ST_UNFINISHED : ST_RUNNING, cnt);
            have = false;
        }
    };
    // take list entry idx (if it is still an active cell): load its state
    auto take = [&](int64_t idx) {
        const uint32_t g = ids ? ids[idx] : (uint32_t)idx;
        const uint8_t st = L.state[g];
        if ((st & 0x7f) != ST_FRESH && (st & 0x7f) != ST_RUNNING) return;
        bool ok;
        load_cell<M>(P, L, g, C, st, cnt, ok);
        if (!ok) { L.state[g] = ST_FAILED; return; }
        have = true;
    };
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (refill) {
            // Persistent lane refill, batched per warp: idle lanes wait until a quarter of the warp
            // is idle (or nothing runs), then take consecutive list entries with one warp-aggregated
            // atomic and load them together, so the dependent-load latency of a cell load is paid
            // once per batch instead of once per finished lane.  All 32 lanes stay in the loop until
            // the warp's (LOCK: the block's) work is exhausted (the ballots name the full warp).
            for (;;) {
                const unsigned need = __ballot_sync(FULL, !have && live);
                if (need == 0) break;
                const unsigned busy = __ballot_sync(FULL, have);
                if (busy != 0 && __popc(need) < refill) break;
                const int leader = __ffs(need) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(&L.stats[S_CURSOR], (unsigned long long)__popc(need));
                base = __shfl_sync(FULL, base, leader);
                if (!have && live) {
                    const int64_t idx = (int64_t)base + __popc(need & ((1u << lane) - 1u));
                    if (idx >= n_ids) live = false;
                    else take(idx);
                }
            }
            if constexpr (LOCK) {
                // lockstep refill (chem_opts.lockstep_sparse): the block's warps take each substep
                // together; the block leaves when none of its threads holds a cell (the cursor is
                // exhausted for every idle lane, or it would have fetched one above)
                if (!__syncthreads_or(have)) break;
            } else {
                if (!__any_sync(FULL, have)) break;
            }
            if (!have) continue;
        } else {
            while (!have && live) {
                // LOCK: persistent tiles of the block; free-running: a grid-stride walk per thread (a
                // grid smaller than the list makes the launch persistent: per-block setup paid once)
                const int64_t idx = LOCK ? (!first ? n_ids : tile * BS + threadIdx.x)
                                         : (first ? (int64_t)blockIdx.x * BS + threadIdx.x
                                                  : next_idx + (int64_t)gridDim.x * BS);
                first = false;
                next_idx = idx;
                if (idx >= n_ids) { live = false; break; }
                take(idx);
            }
            if constexpr (LOCK) {
                if (!__syncthreads_or(have)) {
                    tile += gridDim.x;                  // block-uniform: next tile of this persistent block
                    if (tile * BS >= n_ids) break;
                    first = true;
                    live = true;
                    continue;
                }
                if (!have) continue;
            } else if (!have) break;
        }
        substep();
    }
    __syncwarp();   // all lanes of the warp reach here (no early returns): reconverge for the reduction
    flush_counters(L, cnt);
}

// Caller-side helper (chem_box_active): active cells per box under the gate of Alg. 3 §1 (T >= T_min and
// not solid), without touching the workspace: lets a host-buffer caller move only the boxes a call can
// touch.  grid = (nboxes, slices); reads 8 B (+1 B solid) per cell.
template <int BS>
__global__ void __launch_bounds__(BS) k_box_active(const DevBox* __restrict__ boxes, double T_min, int32_t* active)
{
    const DevBox bx = boxes[blockIdx.x];
    int cnt = 0;
    for (int64_t i = (int64_t)blockIdx.y * BS + threadIdx.x; i < bx.ncells; i += (int64_t)gridDim.y * BS)
        cnt += (bx.T[i] >= T_min && !(bx.solid && bx.solid[i])) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&active[blockIdx.x], cnt);
}

// A11 per-cell outcome of the last call: workspace state byte -> CHEM_CELL_* code
// (0 untouched, 1 done, 2 unfinished, -1 failed; a cell still FRESH/RUNNING, which no completed call
// leaves, reads as failed), and the cell's attempted substeps of the call.  HBM-bound.
static __global__ void k_cell_status(const uint8_t* __restrict__ state, const int32_t* __restrict__ steps, int64_t n,
                                     int8_t* __restrict__ out, int32_t* __restrict__ steps_out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t s = state[i] & 0x7f;
        if (out) out[i] = s == ST_INACTIVE ? 0 : s == ST_DONE ? 1 : s == ST_UNFINISHED ? 2 : -1;
        if (steps_out) steps_out[i] = s == ST_INACTIVE ? 0 : steps[i];
    }
}

// ----------------------------------------------------------------------------- point kernels
template <class M>
__global__ void __launch_bounds__(128) k_rates(const __grid_constant__ Params<M> P, int64_t n, int64_t ld,
                                                    const double* __restrict__ rho,
                        const double* __restrict__ T, const double* __restrict__ Y, double* __restrict__ wdot)
{
    fm_tables_to_smem();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double Yc[M::NS];
#pragma unroll
        for (int k = 0; k < M::NS; ++k) Yc[k] = Y[k * ld + i];
        RateCtx<M> rc;
        rate_ctx<M>(P, rho[i], T[i], Yc, rc);
        double w[M::NS];
        rates_from_ctx<M>(P, rc, w);
#pragma unroll
        for (int k = 0; k < M::NS; ++k) wdot[k * ld + i] = w[k];
    }
}

template <class M>
__global__ void k_rhs(const __grid_constant__ Params<M> P, int64_t n, int64_t ld, const double* __restrict__ rho,
                      const double* __restrict__ T, const double* __restrict__ Y, double* __restrict__ f)
{
    fm_tables_to_smem();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double Yc[M::NS], y[M::NSA + 1], fo[M::NSA + 1];
#pragma unroll
        for (int k = 0; k < M::NS; ++k) Yc[k] = Y[k * ld + i];
#pragma unroll
        for (int a = 0; a < M::NSA; ++a) y[a] = Yc[M::act(a)];
        y[M::NSA] = T[i];
        rhs<M>(P, rho[i], 1.0 / rho[i], y, Yc, fo);
#pragma unroll
        for (int k = 0; k < M::NS; ++k) f[k * ld + i] = (M::act_of(k) >= 0) ? fo[M::act_of(k) >= 0 ? M::act_of(k) : 0] : 0.0;
        f[M::NS * ld + i] = fo[M::NSA];
    }
}

// Full (ns+1)^2 Jacobian, J[(r*(ns+1) + c)*ld + i]; staged through per-thread shared memory.
template <class M, int BS>
__global__ void __launch_bounds__(BS) k_jacobian(const __grid_constant__ Params<M> P, int64_t n, int64_t ld,
                                                 const double* __restrict__ rho, const double* __restrict__ T,
                                                 const double* __restrict__ Y, double* __restrict__ J)
{
    extern __shared__ double smem[];
    fm_tables_to_smem();
    constexpr int nn = M::NS + 1;
    SMat A{smem + threadIdx.x, BS, nn};
    const int64_t i = (int64_t)blockIdx.x * BS + threadIdx.x;
    if (i >= n) return;
    double y[nn], f[nn], Yd[M::NS];
#pragma unroll
    for (int k = 0; k < M::NS; ++k) { y[k] = Y[k * ld + i]; Yd[k] = y[k]; }
    y[M::NS] = T[i];
    rhs_jac<M, JAC_FULL>(P, rho[i], y, Yd, f, A);
#pragma unroll
    for (int r = 0; r < nn; ++r)
#pragma unroll
        for (int c = 0; c < nn; ++c) J[(int64_t)(r * nn + c) * ld + i] = A(r, c);
}

template <class M>
__global__ void k_temperature(const __grid_constant__ Params<M> P, int64_t n, int64_t ld, const double* __restrict__ e,
                              const double* __restrict__ Y, double* __restrict__ T,
                              unsigned long long* __restrict__ nfail)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double Yc[M::NS];
#pragma unroll
        for (int k = 0; k < M::NS; ++k) Yc[k] = Y[k * ld + i];
        double t = T[i];
        if (!newton_T<M>(P, e[i], Yc, t) && nfail) atomicAdd(nfail, 1ull);
        T[i] = t;
    }
}

// PAPER.md Alg. 1: internal energy from the conserved variables, column-major
// U[c*ld + i], c = rho, rho u_x, rho u_y, rho u_z, rho E:  e = rho E/rho - (u_x^2 + u_y^2 + u_z^2)/2.
// The caller-side step before chemistry (NEXT-4); HBM-bound (40 B in, 8 B out per cell).
static __global__ void k_internal_energy(int64_t n, int64_t ld, const double* __restrict__ U, double* __restrict__ e)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double rho = U[i];
        const double inv = 1.0 / rho;
        const double ux = U[ld + i] * inv, uy = U[2 * ld + i] * inv, uz = U[3 * ld + i] * inv;
        const double ke = 0.5 * (ux * ux + uy * uy + uz * uz);
        e[i] = U[4 * ld + i] * inv - ke;
    }
}

template <class M>
__global__ void k_energy(const __grid_constant__ Params<M> P, int64_t n, int64_t ld, const double* __restrict__ T,
                         const double* __restrict__ Y, double* __restrict__ e)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double Yc[M::NS];
#pragma unroll
        for (int k = 0; k < M::NS; ++k) Yc[k] = Y[k * ld + i];
        double u, cv;
        energy_cv<M>(P, T[i], Yc, u, cv);
        e[i] = u;
    }
}

}  // namespace chem
