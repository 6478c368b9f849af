"""Algorithmic work model of the integration kernels (SURVEY.md §8(d) "Algorithmic work per unit").

Counts what the method must compute, not what the hardware executes: no dense zeros, no
redundant work.  FP64 transcendentals are charged w_exp / w_log flops each, the
DADD + DMUL + 2*DFMA count of one libdevice exp / log on sm_100a (profiles/wt_microbench.json,
static SASS count of the kernels `exp(x)` / `log(x)` compiled for sm_100a: exp = 2 DADD + 1 DMUL +
14 DFMA -> 31, log = 8 DADD + 5 DMUL + 17 DFMA -> 47).

Per RHS evaluation (A3-A5):
  thermo 24*Ns + ln k 4*Nr + ln Kc (2*nnz(nu) + 2*Nr_rev) + ln q 2*(nnz(nu') + nnz(nu''))
  + difference Nr + third-body 2*n_eff + falloff 30*N_fo + Omega 2*nnz(nu) + source 6*Ns
  + w_log*(1 + Ns) + w_exp*(Nr + Nr_rev + N_fo) + Troe (2 w_log + 3 w_exp per row)
Per Jacobian (A6): sum_r 2 nnz_r(nu) (nnz_r(nu') + nnz_r(nu'')) + 2 Ntb nnz(nu) Ns/Nr + 15 Nr
  + 3 n^2 + w_exp*(Nr + Nr_rev)   (k_f, k_r for the product-form derivatives)
LU 2n^3/3, each stage solve 2n^2, control 10n, with n = reacting species + 1.
"""
from __future__ import annotations

import numpy as np

W_EXP = 31.0
W_LOG = 47.0


class FlopModel:
    def __init__(self, mt, stages=6):
        nu_f = np.asarray(mt.nu_f)
        nu_r = np.asarray(mt.nu_r)
        net = nu_r - nu_f
        typ = np.asarray(mt.type)
        rev = np.asarray(mt.reversible)
        ns, nr = mt.ns, mt.nr
        nnz_f = int(np.count_nonzero(nu_f))
        nnz_r = int(np.count_nonzero(nu_r))
        nnz = int(np.count_nonzero(net))
        n_rev = int(rev.sum())
        n_fo = int(np.sum(typ >= 2))
        n_troe = int(np.sum(typ == 3))
        n_tb = int(np.sum(typ >= 1))
        n_eff = int(sum(np.count_nonzero(np.asarray(mt.eff)[r] != 1.0) for r in range(nr) if typ[r] >= 1))
        active = int(np.sum(np.any(net != 0, axis=0)))
        self.n = n = active + 1
        self.rhs = (24 * ns + 4 * nr + 2 * nnz + 2 * n_rev + 2 * (nnz_f + nnz_r) + nr + 2 * n_eff + 30 * n_fo
                    + 2 * nnz + 6 * ns + W_LOG * (1 + ns) + W_EXP * (nr + n_rev + n_fo)
                    + n_troe * (2 * W_LOG + 3 * W_EXP))
        jac = 0.0
        for r in range(nr):
            jac += 2 * np.count_nonzero(net[r]) * (np.count_nonzero(nu_f[r]) + np.count_nonzero(nu_r[r]))
        jac += 2 * n_tb * nnz * ns / max(nr, 1) + 15 * nr + 3 * n * n + W_EXP * (nr + n_rev)
        self.jac = jac
        self.lu = 2.0 * n ** 3 / 3.0
        self.solve = 2.0 * n * n
        self.control = 10.0 * n
        self.stages = stages

    def flops(self, stats):
        """Algorithmic FLOPs of one chem_integrate call from its chem_stats counters."""
        frozen = stats.get("steps_frozen", 0)
        att = stats["steps_attempted"] - frozen   # frozen steps: one RHS (y += dt f), no LU/solves
        # a frozen step evaluates J in the kernel (rhs_jac runs before the frozen test) but the method
        # needs only f there, so J is not charged for it: algorithmic work, not executed work
        return (stats["rhs_evals"] * self.rhs + (stats["jac_evals"] - frozen) * self.jac
                + stats["lu_count"] * self.lu + att * (self.stages * self.solve + self.control))

    def per_step(self):
        return self.stages * self.rhs + self.jac + self.lu + self.stages * self.solve + self.control


# FP64 peak of one B200 from unit counts and clocks: 148 SMs x 64 FP64
# FMA lanes per SM per clock x 2 flops x the max SM clock.
def fp64_peak_tflops(sm_count=148, sm_mhz=1965.0, fma_per_sm=64):
    return sm_count * fma_per_sm * 2 * sm_mhz * 1e6 / 1e12
