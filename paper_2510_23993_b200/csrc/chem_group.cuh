// chem_group.cuh — lane-group-per-cell integrator (G lanes cooperate on one cell).
//
// Why: the one-thread-per-cell kernel keeps the n x n iteration matrix and the RODAS4 stage vectors
// of each cell in shared memory (1.17 KB per thread), which caps it at 6 warps per SM and leaves the
// FP64 pipe waiting on dependent DFMA chains (ncu: "wait" stalls).  Here G lanes share one cell:
// the matrix stays per cell in shared memory (1/G of it per lane), the state and stage vectors are
// distributed over the lanes' registers, the reactions of the RHS are split over the lanes
// (table-driven, so every lane runs the same instructions), and many more warps are resident.
//
// Same mathematics as chem_device.cuh (matrix-form rates A4, Eq. 5/6 RHS A5, analytic Jacobian,
// RODAS4/RODAS3 with the same controller); reductions across lanes run in a fixed order, so a cell's
// result is deterministic and independent of K_max, N*, box grouping and scheduling.
#pragma once
#include <cstring>

#include "chem_kernels.cuh"

namespace chem {

// ----------------------------------------------------------------------------- per-block tables
template <class M>
struct GTable {
    static constexpr int MAXU = 2 * M::MAXRP;   // unique species per reaction (upper bound)
    struct Rxn {
        double lnA, b, EaR, lnA0, b0, Ea0R, ta, tiT3, tiT1, tT2, tL;
        double effm1[M::MAXEFF];
        int8_t nre, npr, kind, rev, neff, tconst, t2, dnu, nu;   // nu = unique species count
        int8_t re[M::MAXRP], pr[M::MAXRP], effsp[M::MAXEFF];
        int8_t usp[MAXU], unf[MAXU], unr[MAXU];                  // unique species, nu', nu''
    };
    Rxn rx[M::NR];
    int8_t nsr[M::NS];                   // reactions with nonzero net nu for species k
    int8_t sr[M::NS][M::NR];
    int8_t snu[M::NS][M::NR];
    double cpc[2][M::NS][5], hc[2][M::NS][6], sc[2][M::NS][6], dcp[2][M::NS][4];
    double W[M::NS], invW[M::NS];
    double Tmid, R, lnp0R, T_valid_lo, T_valid_hi;
    int8_t act[M::NSA > 0 ? M::NSA : 1];   // unknown -> species
    int8_t act_of[M::NS];                  // species -> unknown (-1: inert)

    // Build from the numeric parameter block and the compile-time structure (host side).
    static void build(const Params<M>& p, GTable& t)
    {
        std::memset(&t, 0, sizeof(GTable));
        for (int r = 0; r < M::NR; ++r) {
            Rxn& x = t.rx[r];
            x.lnA = p.lnA[r]; x.b = p.b[r]; x.EaR = p.EaR[r];
            x.lnA0 = p.lnA0[r]; x.b0 = p.b0[r]; x.Ea0R = p.Ea0R[r];
            x.ta = p.troe_a[r]; x.tiT3 = p.troe_iT3[r]; x.tiT1 = p.troe_iT1[r]; x.tT2 = p.troe_T2[r];
            x.tL = p.troe_L[r];
            x.kind = (int8_t)M::kind(r); x.rev = (int8_t)M::rev(r); x.tconst = (int8_t)p.troe_const[r];
            x.t2 = (int8_t)M::troe_t2(r); x.dnu = (int8_t)M::dnu(r);
            x.nre = (int8_t)M::nreac(r); x.npr = (int8_t)M::nprod(r); x.neff = (int8_t)M::neff(r);
            for (int i = 0; i < M::MAXRP; ++i) {
                x.re[i] = (int8_t)(i < M::nreac(r) ? M::reac(r, i) : 0);
                x.pr[i] = (int8_t)(i < M::nprod(r) ? M::prod(r, i) : 0);
            }
            for (int i = 0; i < M::MAXEFF; ++i) {
                x.effsp[i] = (int8_t)(i < M::neff(r) ? M::eff_sp(r, i) : 0);
                x.effm1[i] = i < M::neff(r) ? p.effm1[M::eff_off(r) + i] : 0.0;
            }
            int nu = 0;
            for (int k = 0; k < M::NS; ++k)
                if (M::nuf(r, k) || M::nur(r, k)) {
                    x.usp[nu] = (int8_t)k; x.unf[nu] = (int8_t)M::nuf(r, k); x.unr[nu] = (int8_t)M::nur(r, k);
                    ++nu;
                }
            x.nu = (int8_t)nu;
        }
        for (int k = 0; k < M::NS; ++k) {
            int c = 0;
            for (int r = 0; r < M::NR; ++r)
                if (M::nu(r, k)) { t.sr[k][c] = (int8_t)r; t.snu[k][c] = (int8_t)M::nu(r, k); ++c; }
            t.nsr[k] = (int8_t)c;
            t.W[k] = p.W[k]; t.invW[k] = p.invW[k];
        }
        std::memcpy(t.cpc, p.cpc, sizeof(t.cpc)); std::memcpy(t.hc, p.hc, sizeof(t.hc));
        std::memcpy(t.sc, p.sc, sizeof(t.sc)); std::memcpy(t.dcp, p.dcp, sizeof(t.dcp));
        for (int i = 0; i < M::NSA; ++i) t.act[i] = (int8_t)M::act(i);
        for (int k = 0; k < M::NS; ++k) t.act_of[k] = (int8_t)M::act_of(k);
        t.Tmid = p.Tmid_common; t.R = p.R; t.lnp0R = p.lnp0R;
        t.T_valid_lo = p.T_valid_lo; t.T_valid_hi = p.T_valid_hi;
    }
};

// ----------------------------------------------------------------------------- group primitives
template <int G>
struct Grp {
    unsigned mask;
    int base, gl;
    __device__ __forceinline__ Grp()
    {
        const int lane = threadIdx.x & 31;
        gl = lane & (G - 1);
        base = lane - gl;
        mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << base);
    }
    __device__ __forceinline__ double sum(double v) const
    {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
        return v;
    }
    __device__ __forceinline__ double bcast(double v, int src) const { return __shfl_sync(mask, v, base + src); }
    __device__ __forceinline__ int bcast_i(int v, int src) const { return __shfl_sync(mask, v, base + src); }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
};

// Per-cell shared-memory region (doubles), one per lane group.
template <class M>
struct GLayout {
    static constexpr int n = M::NSA + 1;
    static constexpr int U = GTable<M>::MAXU;
    static constexpr int RW = U + 2;              // Jacobian record per reaction: dq/dc_u, dq/dT, D
    static constexpr int oA = 0;                  // n x n iteration matrix / LU
    static constexpr int oRec = oA + n * n;       // NR x RW
    static constexpr int oQ = oRec + M::NR * RW;  // q_r
    static constexpr int oY = oQ + M::NR;         // Y_k of the evaluation point (all species)
    static constexpr int oT = oY + M::NS;         // T of the evaluation point
    static constexpr int oLnc = oT + 1;
    static constexpr int oG = oLnc + M::NS;       // g_k = h/RT - s/R
    static constexpr int oC = oG + M::NS;         // c_k
    static constexpr int oH = oC + M::NS;         // h/RT
    static constexpr int oCp = oH + M::NS;        // cp/R
    static constexpr int oX = oCp + M::NS;        // n-vector scratch (permutation)
    static constexpr int oPiv = oX + n;           // n pivot bytes
    static constexpr int size = oPiv + (n + 7) / 8 + 1;   // +1: keeps cells 8-B-word odd strided
};

template <class M, int G>
struct GOwn {   // unknown i owned by lane i % G, slot i / G
    static constexpr int n = M::NSA + 1;
    static constexpr int U = (n + G - 1) / G;
    static constexpr int SPL = (M::NS + G - 1) / G;
    static constexpr int RPL = (M::NR + G - 1) / G;
};

// Thermo of one species with table coefficients (range chosen by the shared T_mid).
template <class M>
__device__ __forceinline__ void g_thermo(const GTable<M>& tb, int k, double T, double lnT, double invT,
                                         double& cpR, double& hRT, double& sR, double& dcpR)
{
    const int rg = (T < tb.Tmid) ? 0 : 1;
    const double* c = tb.cpc[rg][k];
    const double* h = tb.hc[rg][k];
    const double* s = tb.sc[rg][k];
    const double* d = tb.dcp[rg][k];
    cpR = fma(T, fma(T, fma(T, fma(T, c[4], c[3]), c[2]), c[1]), c[0]);
    hRT = fma(T, fma(T, fma(T, fma(T, h[4], h[3]), h[2]), h[1]), h[0]) + h[5] * invT;
    sR = fma(s[0], lnT, fma(T, fma(T, fma(T, fma(T, s[4], s[3]), s[2]), s[1]), s[5]));
    dcpR = fma(T, fma(T, fma(T, d[3], d[2]), d[1]), d[0]);
}

// Troe F (table-driven twin of troe_F).
template <bool DERIV, class R>
__device__ __forceinline__ double g_troe(const R& x, double T, double invT, double Pr, double& g_x, double& g_T)
{
    const double a = x.ta;
    double Fc, dFc, L;
    if (x.tconst) {
        Fc = a;
        dFc = -a * x.tiT1;
        L = x.tL;
    } else {
        const double e3 = exp(-T * x.tiT3);
        const double e1 = exp(-T * x.tiT1);
        Fc = (1.0 - a) * e3 + a * e1;
        dFc = -(1.0 - a) * x.tiT3 * e3 - a * x.tiT1 * e1;
        if (x.t2) {
            const double e2 = exp(-x.tT2 * invT);
            Fc += e2;
            dFc += x.tT2 * invT * invT * e2;
        }
        L = flog(Fc) * kLog10e;
    }
    const double C = -0.4 - 0.67 * L;
    const double N = 0.75 - 1.27 * L;
    const double xx = flog(fmax(Pr, 1e-300)) * kLog10e;
    const double u = xx + C;
    const double den = N - 0.14 * u;
    const double f1 = u / den;
    const double q = 1.0 / (1.0 + f1 * f1);
    const double lF = L * q;
    if (DERIV) {
        const double w = -L * 2.0 * f1 * q * q / (den * den);
        g_x = w * N;
        const double dlF_dL = q + w * (-0.67 * den + 1.1762 * u);
        g_T = dlF_dL * dFc / (Fc * kLn10);
    }
    return exp(lF * kLn10);
}

// One cell's evaluation context for the group: distributed unknowns y_own[U] (lane gl owns
// unknowns gl, gl+G, ...), replicated scalars.
template <class M, int G>
struct GCell {
    static constexpr int U = GOwn<M, G>::U;
    double y[U];
    double rho, e, t, h, dt;
    uint32_t g;
    int b;
    int64_t off, ld;
    int k;
    bool rej;
};

// RHS and (optionally) Jacobian of the cell at the distributed point `ys`; output f_own[U].
// With JAC, the Jacobian J = df/dy is written into the per-cell matrix A (not yet I/(h g) - J).
template <class M, int G, bool JAC>
__device__ __forceinline__ void g_rhs(const GTable<M>& tb, const Grp<G>& gr, double* cs, double rho,
                                      const double* ys, double* f_own)
{
    using LY = GLayout<M>;
    using O = GOwn<M, G>;
    constexpr int n = LY::n;
    constexpr int NSA = M::NSA;
    // 1. publish the evaluation point
#pragma unroll
    for (int u = 0; u < O::U; ++u) {
        const int i = gr.gl + u * G;
        if (i < NSA) cs[LY::oY + tb.act[i]] = ys[u];
        else if (i == NSA) cs[LY::oT] = ys[u];
    }
    gr.sync();
    const double T = cs[LY::oT];
    const double lnT = flog(T);
    const double invT = 1.0 / T;
    const double RT = tb.R * T;
    // 2. species phase: thermo, c, ln c; partial sums of cv, dcv/dT, [M]
    double cv = 0.0, dcv = 0.0, mt = 0.0;
#pragma unroll
    for (int j = 0; j < O::SPL; ++j) {
        const int k = gr.gl + j * G;
        if (k < M::NS) {
            double cpR, hRT, sR, dcpR;
            g_thermo<M>(tb, k, T, lnT, invT, cpR, hRT, sR, dcpR);
            const double Yk = cs[LY::oY + k];
            const double c = rho * fmax(Yk, 0.0) * tb.invW[k];
            cs[LY::oLnc + k] = flog(c);
            cs[LY::oC + k] = c;
            cs[LY::oG + k] = hRT - sR;
            cs[LY::oH + k] = hRT;
            cs[LY::oCp + k] = cpR;
            cv = fma(Yk * tb.invW[k], cpR - 1.0, cv);
            dcv = fma(Yk * tb.invW[k], dcpR, dcv);
            mt += c;
        }
    }
    cv = gr.sum(cv) * tb.R;
    if (JAC) dcv = gr.sum(dcv) * tb.R;
    mt = gr.sum(mt);
    gr.sync();
    // 3. reaction phase: lane gl takes reactions gl, gl+G, ...
    const double lnp0RT = tb.lnp0R - lnT;
#pragma unroll 1
    for (int j = 0; j < O::RPL; ++j) {
        const int r = gr.gl + j * G;
        if (r >= M::NR) break;
        const auto& x = tb.rx[r];
        const double lnkf = fma(x.b, lnT, x.lnA) - x.EaR * invT;
        double fac = 1.0, dfac_dM = 0.0, dfac_dT = 0.0, prk = 0.0;
        if (x.kind != 0) {
            double Mr = mt;
            for (int i = 0; i < x.neff; ++i) Mr = fma(x.effm1[i], cs[LY::oC + x.effsp[i]], Mr);
            if (x.kind == 1) {
                fac = Mr;
                dfac_dM = 1.0;
            } else {
                const double lnk0 = fma(x.b0, lnT, x.lnA0) - x.Ea0R * invT;
                prk = exp(lnk0 - lnkf);
                const double Pr = prk * Mr;
                double F = 1.0, gx = 0.0, gT = 0.0;
                if (x.kind == 3) F = g_troe<JAC>(x, T, invT, Pr, gx, gT);
                const double ip = 1.0 / (1.0 + Pr);
                fac = Pr * ip * F;
                if (JAC) {
                    const double dlnk0 = fma(x.Ea0R, invT, x.b0) * invT;
                    const double dlnkf = fma(x.EaR, invT, x.b) * invT;
                    const double dfac_dPr = F * ip * ip + F * gx * ip;
                    dfac_dM = dfac_dPr * prk;
                    dfac_dT = dfac_dPr * Pr * (dlnk0 - dlnkf) + fac * kLn10 * gT;
                }
            }
        }
        double lnqf = lnkf;
        for (int i = 0; i < x.nre; ++i) lnqf += cs[LY::oLnc + x.re[i]];
        const double qf0 = exp(lnqf);
        double qr0 = 0.0, lnKc = 0.0;
        if (x.rev) {
            lnKc = (double)x.dnu * lnp0RT;
            for (int i = 0; i < x.nre; ++i) lnKc += cs[LY::oG + x.re[i]];
            for (int i = 0; i < x.npr; ++i) lnKc -= cs[LY::oG + x.pr[i]];
            double lnqr = lnkf - lnKc;
            for (int i = 0; i < x.npr; ++i) lnqr += cs[LY::oLnc + x.pr[i]];
            qr0 = exp(lnqr);
        }
        const double d0 = qf0 - qr0;
        cs[LY::oQ + r] = d0 * fac;
        if (JAC) {
            const double dlnkf = fma(x.EaR, invT, x.b) * invT;
            double dlnKc = 0.0;
            if (x.rev) {
                double sh = 0.0;
                for (int i = 0; i < x.npr; ++i) sh += cs[LY::oH + x.pr[i]];
                for (int i = 0; i < x.nre; ++i) sh -= cs[LY::oH + x.re[i]];
                dlnKc = (sh - (double)x.dnu) * invT;
            }
            const double kf = exp(lnkf);
            const double kr = x.rev ? exp(lnkf - lnKc) : 0.0;
            double* rec = cs + LY::oRec + r * LY::RW;
            for (int m = 0; m < x.nu; ++m) {      // dq/dc_j, product form (no division by c_j)
                const int sp = x.usp[m];
                double dq = 0.0;
                if (x.unf[m]) {
                    double p = kf * (double)x.unf[m];
                    bool skipped = false;
                    for (int i = 0; i < x.nre; ++i) {
                        if (!skipped && x.re[i] == sp) { skipped = true; continue; }
                        p *= cs[LY::oC + x.re[i]];
                    }
                    dq = p;
                }
                if (x.unr[m] && x.rev) {
                    double p = kr * (double)x.unr[m];
                    bool skipped = false;
                    for (int i = 0; i < x.npr; ++i) {
                        if (!skipped && x.pr[i] == sp) { skipped = true; continue; }
                        p *= cs[LY::oC + x.pr[i]];
                    }
                    dq -= p;
                }
                rec[m] = dq * fac;
            }
            rec[LY::U] = fac * (qf0 * dlnkf - qr0 * (dlnkf - dlnKc)) + d0 * dfac_dT;   // dq/dT
            rec[LY::U + 1] = d0 * dfac_dM;                                             // D_r
        }
    }
    gr.sync();
    // 4. species rows (owner of unknown i): Omega, f, and the Jacobian rows
    const double invrho = 1.0 / rho;
    double S = 0.0, SdT = 0.0;
    double sT[JAC ? n : 1];
    if (JAC) {
#pragma unroll
        for (int j = 0; j < n; ++j) sT[j] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < O::U; ++u) {
        const int i = gr.gl + u * G;
        if (i >= NSA) {
            continue;
        }
        const int k = tb.act[i];
        double w = 0.0, wT = 0.0, base = 0.0;
        double* rowA = cs + LY::oA + i * n;
        if (JAC) {
#pragma unroll
            for (int j = 0; j < n; ++j) rowA[j] = 0.0;
        }
        const int nl = tb.nsr[k];
        for (int l = 0; l < nl; ++l) {
            const int r = tb.sr[k][l];
            const double nu = (double)tb.snu[k][l];
            w = fma(nu, cs[LY::oQ + r], w);
            if (JAC) {
                const double* rec = cs + LY::oRec + r * LY::RW;
                const auto& x = tb.rx[r];
                wT = fma(nu, rec[LY::U], wT);
                base = fma(nu, rec[LY::U + 1], base);
                for (int m = 0; m < x.nu; ++m) {
                    const int col = tb.act_of[x.usp[m]];
                    if (col >= 0) rowA[col] = fma(nu, rec[m], rowA[col]);
                }
                for (int e2 = 0; e2 < x.neff; ++e2) {
                    const int col = tb.act_of[x.effsp[e2]];
                    if (col >= 0) rowA[col] = fma(nu * x.effm1[e2], rec[LY::U + 1], rowA[col]);
                }
            }
        }
        f_own[u] = tb.W[k] * w * invrho;
        const double hk = cs[LY::oH + k];
        S = fma(hk - 1.0, w, S);
        if (JAC) {
            SdT = fma(cs[LY::oCp + k] - 1.0, w, SdT);
            const double epsW = (hk - 1.0) * RT * tb.invW[k];
#pragma unroll
            for (int j = 0; j < NSA; ++j) {
                const int kj = tb.act[j];
                const double cj = (cs[LY::oY + kj] >= 0.0) ? 1.0 : 0.0;
                const double v = tb.W[k] * tb.invW[kj] * cj * (rowA[j] + base);
                rowA[j] = v;
                sT[j] = fma(epsW, v, sT[j]);
            }
            const double jiT = tb.W[k] * wT * invrho;
            rowA[NSA] = jiT;
            sT[NSA] = fma(epsW, jiT, sT[NSA]);
        }
    }
    S = gr.sum(S);
    const double fT = -(S * RT) * invrho / cv;
#pragma unroll
    for (int u = 0; u < O::U; ++u)
        if (gr.gl + u * G == NSA) f_own[u] = fT;
    if (JAC) {
        SdT = gr.sum(SdT);
        // T row: J_Tj = -(sum_i eps_i J_ij / W_i)/cv - fT cv_j/cv ; J_TT likewise (see rhs_jac)
#pragma unroll
        for (int j = 0; j < n; ++j) sT[j] = gr.sum(sT[j]);
        const int ownerT = NSA % G;
        if (gr.gl == ownerT) {
            double* rowT = cs + LY::oA + NSA * n;
#pragma unroll
            for (int j = 0; j < NSA; ++j) {
                const int kj = tb.act[j];
                const double cvj = tb.R * (cs[LY::oCp + kj] - 1.0) * tb.invW[kj];
                rowT[j] = -sT[j] / cv - fT * cvj / cv;
            }
            rowT[NSA] = -(SdT * tb.R * invrho + sT[NSA]) / cv - fT * dcv / cv;
        }
    }
    gr.sync();
}

// ----------------------------------------------------------------------------- group LU / solve
// Rows are owned by lanes (row i -> lane i % G).  Partial pivoting: group argmax per column.
template <int n, int G>
__device__ __forceinline__ bool g_lu(const Grp<G>& gr, double* A, uint8_t* piv)
{
    bool ok = true;
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
        double best = -1.0;
        int bi = k;
#pragma unroll
        for (int u = 0; u < (n + G - 1) / G; ++u) {
            const int i = gr.gl + u * G;
            if (i >= k && i < n) {
                const double v = fabs(A[i * n + k]);
                if (v > best) { best = v; bi = i; }
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(gr.mask, best, o);
            const int oi = __shfl_xor_sync(gr.mask, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        ok = ok && (best > 0.0) && isfinite(best);
        if (gr.gl == 0) piv[k] = (uint8_t)bi;
        if (bi != k) {
            for (int j = gr.gl; j < n; j += G) {
                const double t = A[k * n + j];
                A[k * n + j] = A[bi * n + j];
                A[bi * n + j] = t;
            }
        }
        gr.sync();
        const double inv = 1.0 / A[k * n + k];
#pragma unroll
        for (int u = 0; u < (n + G - 1) / G; ++u) {
            const int i = gr.gl + u * G;
            if (i > k && i < n) {
                const double l = A[i * n + k] * inv;
                A[i * n + k] = l;
                for (int j = k + 1; j < n; ++j) A[i * n + j] = fma(-l, A[k * n + j], A[i * n + j]);
            }
        }
        gr.sync();
    }
    return ok;
}

// Solve (LU) x = b for the distributed vector b (owned slots), in place.
template <int n, int G>
__device__ __forceinline__ void g_solve(const Grp<G>& gr, const double* A, const uint8_t* piv, double* xs,
                                        double (&b)[(n + G - 1) / G])
{
    constexpr int U = (n + G - 1) / G;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = gr.gl + u * G;
        if (i < n) xs[i] = b[u];
    }
    gr.sync();
    if (gr.gl == 0) {
        for (int k = 0; k < n; ++k) {
            const int p = piv[k];
            if (p != k) { const double t = xs[k]; xs[k] = xs[p]; xs[p] = t; }
        }
    }
    gr.sync();
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = gr.gl + u * G;
        b[u] = (i < n) ? xs[i] : 0.0;
    }
    gr.sync();
    // forward (unit lower), column sweep: x_j broadcast from its owner
#pragma unroll
    for (int j = 0; j < n - 1; ++j) {
        const double xj = gr.bcast(b[j / G], j % G);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = gr.gl + u * G;
            if (i > j && i < n) b[u] = fma(-A[i * n + j], xj, b[u]);
        }
    }
    // backward
#pragma unroll
    for (int j = n - 1; j >= 0; --j) {
        double v = b[j / G];
        if (gr.gl == j % G) v = v / A[j * n + j];
        const double xj = gr.bcast(v, j % G);
        if (gr.gl == j % G) b[j / G] = xj;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = gr.gl + u * G;
            if (i < j) b[u] = fma(-A[i * n + j], xj, b[u]);
        }
    }
}

// Newton T at constant (e, rho) for the group (species Y in cs[oY]); all lanes return the same T.
template <class M, int G>
__device__ __forceinline__ bool g_newton(const GTable<M>& tb, const Grp<G>& gr, const double* cs, double e, double& T)
{
    using LY = GLayout<M>;
    using O = GOwn<M, G>;
    for (int it = 0; it < 50; ++it) {
        const double invT = 1.0 / T;
        double su = 0.0, sc = 0.0;
#pragma unroll
        for (int j = 0; j < O::SPL; ++j) {
            const int k = gr.gl + j * G;
            if (k < M::NS) {
                double cpR, hRT, sR, dcpR;
                g_thermo<M>(tb, k, T, 0.0, invT, cpR, hRT, sR, dcpR);
                const double yw = cs[LY::oY + k] * tb.invW[k];
                su = fma(yw, hRT - 1.0, su);
                sc = fma(yw, cpR - 1.0, sc);
            }
        }
        su = gr.sum(su);
        sc = gr.sum(sc);
        const double dT = (su * tb.R * T - e) / (sc * tb.R);
        T -= dT;
        if (fabs(dT) <= 1e-12 * fabs(T)) return isfinite(T);
    }
    return false;
}

// ----------------------------------------------------------------------------- group substep
template <class M, class Meth, int G>
__device__ __forceinline__ int g_step(const GTable<M>& tb, const Grp<G>& gr, const LaunchCtx& L, GCell<M, G>& C,
                                      double* cs, double (&K)[Meth::S][GOwn<M, G>::U], Counters& cnt)
{
    using LY = GLayout<M>;
    using O = GOwn<M, G>;
    constexpr int n = LY::n;
    constexpr int U = O::U;
    constexpr int S = Meth::S;
    double* A = cs + LY::oA;
    uint8_t* piv = reinterpret_cast<uint8_t*>(cs + LY::oPiv);
    double f0[U];
    g_rhs<M, G, true>(tb, gr, cs, C.rho, C.y, f0);
    cnt.rhs++;
    auto tolw = [&](int u, double yv) {
        const int i = gr.gl + u * G;
        return ((i < M::NSA) ? L.atol : L.atolT) + L.rtol * fabs(yv);
    };
    const double remaining = C.dt - C.t;
    if (!(C.h > 0.0)) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (gr.gl + u * G < n) {
                const double sc = tolw(u, C.y[u]);
                d0 = fma(C.y[u] / sc, C.y[u] / sc, d0);
                d1 = fma(f0[u] / sc, f0[u] / sc, d1);
            }
        }
        d0 = sqrt(gr.sum(d0) / n);
        d1 = sqrt(gr.sum(d1) / n);
        if (d1 * remaining < 1e-3) {   // frozen cell: one explicit step (R22)
#pragma unroll
            for (int u = 0; u < U; ++u) C.y[u] = fma(remaining, f0[u], C.y[u]);
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
    if (!(h > 4.0 * 2.220446049250313e-16 * C.dt) || !isfinite(h)) return -1;
    const double ghinv = 1.0 / (h * Meth::gamma);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = gr.gl + u * G;
        if (i < n)
            for (int j = 0; j < n; ++j) A[i * n + j] = (i == j) ? ghinv - A[i * n + j] : -A[i * n + j];
    }
    gr.sync();
    const bool ok = g_lu<n, G>(gr, A, piv);
    const double hinv = 1.0 / h;
    double* xs = cs + LY::oX;
#pragma unroll
    for (int u = 0; u < U; ++u) K[0][u] = f0[u];
    g_solve<n, G>(gr, A, piv, xs, K[0]);
#pragma unroll
    for (int s = 1; s < S; ++s) {
        double F[U];
        if (Meth::newf(s)) {
            double ys[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double v = C.y[u];
#pragma unroll
                for (int j = 0; j < s; ++j)
                    if (Meth::a(s, j) != 0.0) v = fma(Meth::a(s, j), K[j][u], v);
                ys[u] = v;
            }
            g_rhs<M, G, false>(tb, gr, cs, C.rho, ys, F);
            cnt.rhs++;
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) F[u] = f0[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double v = F[u];
#pragma unroll
            for (int j = 0; j < s; ++j)
                if (Meth::c(s, j) != 0.0) v = fma(Meth::c(s, j) * hinv, K[j][u], v);
            K[s][u] = v;
        }
        g_solve<n, G>(gr, A, piv, xs, K[s]);
    }
    double ynew[U];
    double err = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double v = C.y[u], ev = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            if (Meth::m(j) != 0.0) v = fma(Meth::m(j), K[j][u], v);
            if (Meth::e(j) != 0.0) ev = fma(Meth::e(j), K[j][u], ev);
        }
        ynew[u] = v;
        if (gr.gl + u * G < n) {
            const int i = gr.gl + u * G;
            const double sc = ((i < M::NSA) ? L.atol : L.atolT) + L.rtol * fmax(fabs(C.y[u]), fabs(v));
            err = fma(ev / sc, ev / sc, err);
        }
    }
    err = sqrt(gr.sum(err) / n);
    cnt.attempted++;
    C.k++;
    if (!ok || !isfinite(err)) {
        C.h = h * 0.1;
        C.rej = true;
        return 0;
    }
    double fac = 0.9 * pow(err, -Meth::err_exp);
    fac = fmin(6.0, fmax(0.2, fac));
    double hnew = h * fac;
    if (err <= 1.0) {
        cnt.accepted++;
#pragma unroll
        for (int u = 0; u < U; ++u) C.y[u] = ynew[u];
        C.t = last ? C.dt : C.t + h;
        if (C.rej) hnew = fmin(hnew, h);
        C.rej = false;
        C.h = hnew;
        return 1;
    }
    C.h = C.rej ? h * 0.1 : hnew;
    C.rej = true;
    return 0;
}

// ----------------------------------------------------------------------------- group load / store
template <class M, int G>
__device__ __forceinline__ bool g_load(const GTable<M>& tb, const Grp<G>& gr, const LaunchCtx& L, uint32_t g,
                                       GCell<M, G>& C, double* cs, uint8_t st, Counters& cnt)
{
    using LY = GLayout<M>;
    using O = GOwn<M, G>;
    C.g = g;
    C.b = L.cell_box[g];
    const DevBox bx = L.boxes[C.b];
    C.off = g - L.box_start[C.b];
    C.ld = bx.ld;
    C.dt = bx.dt;
    C.rho = bx.rho[C.off];
    C.e = bx.e[C.off];
    C.k = 0;
#pragma unroll
    for (int j = 0; j < O::SPL; ++j) {
        const int k = gr.gl + j * G;
        if (k < M::NS) cs[LY::oY + k] = bx.Y[k * C.ld + C.off];
    }
    gr.sync();
    double T = bx.T[C.off];
    bool ok = true;
    if ((st & 0x7f) == ST_FRESH) {
        ok = g_newton<M, G>(tb, gr, cs, C.e, T);
        if (!ok && gr.gl == 0) cnt.newton_fail++;
        C.t = 0.0;
        C.h = 0.0;
        C.rej = false;
    } else {
        C.t = L.cell_t[g];
        C.h = L.cell_h[g];
        C.rej = (st & 0x80) != 0;
    }
#pragma unroll
    for (int u = 0; u < O::U; ++u) {
        const int i = gr.gl + u * G;
        C.y[u] = (i < M::NSA) ? cs[LY::oY + tb.act[i < M::NSA ? i : 0]] : T;
    }
    gr.sync();
    return ok;
}

template <class M, int G>
__device__ __forceinline__ void g_store(const GTable<M>& tb, const Grp<G>& gr, const LaunchCtx& L, GCell<M, G>& C,
                                        double* cs, uint8_t st, Counters& cnt)
{
    using LY = GLayout<M>;
    using O = GOwn<M, G>;
    const DevBox bx = L.boxes[C.b];
    double Tint = 0.0;
#pragma unroll
    for (int u = 0; u < O::U; ++u) {
        const int i = gr.gl + u * G;
        if (i < M::NSA) {
            const int k = tb.act[i];
            bx.Y[k * C.ld + C.off] = C.y[u];
            cs[LY::oY + k] = C.y[u];
        } else if (i == M::NSA) {
            Tint = C.y[u];
        }
    }
    Tint = gr.bcast(Tint, M::NSA % G);
    gr.sync();
    double T = Tint;
    if (st == ST_DONE || st == ST_UNFINISHED) {
        if (!g_newton<M, G>(tb, gr, cs, C.e, T)) {
            if (gr.gl == 0) cnt.newton_fail++;
            st = ST_FAILED;
        }
        if (gr.gl == 0) {
            if (st == ST_DONE) {
                cnt.done++;
                cnt.drift = fmax(cnt.drift, fabs(Tint - T) / T);
                if (T < tb.T_valid_lo || T > tb.T_valid_hi) cnt.trange++;
            } else if (st == ST_UNFINISHED) {
                cnt.unfinished++;
            }
        }
    }
    if (gr.gl == 0) {
        bx.T[C.off] = T;
        L.cell_t[C.g] = C.t;
        L.cell_h[C.g] = C.h;
        L.state[C.g] = st | (C.rej ? 0x80 : 0);
        L.cell_steps[C.g] += C.k;
    }
    gr.sync();
}

// ----------------------------------------------------------------------------- group kernel
// BS threads = BS/G cells per block.  The table is copied to shared memory once per block.
template <class M, class Meth, int G, int BS>
__global__ void __launch_bounds__(BS) k_integrate_grp(const GTable<M>* __restrict__ gtab, LaunchCtx L,
                                                      const uint32_t* __restrict__ ids, int64_t n_ids, int kmax,
                                                      int refill, int final_phase)
{
    extern __shared__ double smem[];
    GTable<M>& tb = *reinterpret_cast<GTable<M>*>(smem);
    constexpr int tab_doubles = (sizeof(GTable<M>) + 7) / 8;
    {
        const double* src = reinterpret_cast<const double*>(gtab);
        for (int i = threadIdx.x; i < tab_doubles; i += BS) smem[i] = src[i];
    }
    __syncthreads();
    const Grp<G> gr;
    double* cs = smem + tab_doubles + (threadIdx.x / G) * GLayout<M>::size;
    Counters cnt;
    GCell<M, G> C;
    double K[Meth::S][GOwn<M, G>::U];
    bool have = false, first = true;
    for (;;) {
        if (!have) {
            int64_t idx = n_ids;
            if (refill) {
                if (gr.gl == 0) idx = (int64_t)atomicAdd(&L.stats[S_CURSOR], 1ull);
                idx = (int64_t)__shfl_sync(gr.mask, (long long)idx, gr.base);
            } else {
                idx = first ? ((int64_t)blockIdx.x * BS + threadIdx.x) / G : n_ids;
                first = false;
            }
            if (idx >= n_ids) break;
            const uint32_t g = ids ? ids[idx] : (uint32_t)idx;
            const uint8_t st = L.state[g];
            if ((st & 0x7f) != ST_FRESH && (st & 0x7f) != ST_RUNNING) continue;
            if (!g_load<M, G>(tb, gr, L, g, C, cs, st, cnt)) {
                if (gr.gl == 0) L.state[g] = ST_FAILED;
                continue;
            }
            have = true;
        }
        const int r = g_step<M, Meth, G>(tb, gr, L, C, cs, K, cnt);
        if (r < 0) {
            if (gr.gl == 0) cnt.nonfinite++;
            g_store<M, G>(tb, gr, L, C, cs, ST_FAILED, cnt);
            have = false;
        } else if (C.t >= C.dt) {
            g_store<M, G>(tb, gr, L, C, cs, ST_DONE, cnt);
            have = false;
        } else if (C.k >= kmax) {
            g_store<M, G>(tb, gr, L, C, cs, final_phase ? ST_UNFINISHED : ST_RUNNING, cnt);
            have = false;
        }
    }
    // per-cell counters were incremented by every lane of a group (step counts) -> count once
    if (gr.gl != 0) {
        cnt.attempted = 0; cnt.accepted = 0; cnt.rhs = 0; cnt.frozen = 0;
    }
    __syncwarp();
    flush_counters(L, cnt);
}

template <class M, int G>
constexpr size_t grp_smem_bytes(int BS)
{
    return (((sizeof(GTable<M>) + 7) / 8) + (size_t)(BS / G) * GLayout<M>::size) * 8;
}

}  // namespace chem
