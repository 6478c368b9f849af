"""Algorithmic work model of the integration kernels: SURVEY.md §8(d) "Algorithmic work per unit",
implemented literally, so the bench's roofline fraction can be recomputed by hand
as  (§8(d) FLOPs per substep x chem_stats counters) / (CUDA-event k_integrate time) / peak.

Per RHS evaluation (A3-A5), §8(d):
    24 Ns (thermo) + 4 Nr (ln k) + 2 nnz(nu) + 2 Nr (ln Kc) + 2 (nnz(nu') + nnz(nu'')) (ln q)
    + Nr (difference) + 2 Ns N_tb (third-body) + 30 N_fo (falloff) + 2 nnz(nu) (Omega)
    + 6 Ns (source terms) + transcendentals (1 + Ns) logs + (2 Nr + 3 N_fo) exps
Per substep: Jacobian  sum_r 2 nnz_r(nu) (nnz_r(nu') + nnz_r(nu'')) + 2 N_tb nnz(nu) Ns/Nr + 15 Nr + 3 n^2,
             LU 2 n^3 / 3, each of the s stage solves 2 n^2, control 10 n,   n = reacting species + 1;
FLOPs_call = sum over attempted substeps of (s RHS + J + LU + s solves + control).

Transcendentals are charged at the DADD + DMUL + 2 DFMA count of one libdevice exp / log, "measured
by an ncu microkernel" (§8(d)): W_EXP = 29 (1 DADD + 14 DFMA), W_LOG = 44 (8 DADD + 4 DMUL + 16 DFMA),
the executed counts per call on the B200 (tools/fp64_probe.sh -> profiles/wt_microbench.json
"dynamic"; the static SASS count, 31 / 47, includes the never-taken special-value paths).

The one departure from the literal formula, and why: a *frozen* first step (the
north_star's "cheap bulk step", DESIGN reading R22) is one explicit Euler step y += dt f(y): the
method evaluates one RHS there and no Jacobian, LU or stages, so it is charged one RHS.  At the
parity tolerance frozen steps are rare (0 on cfg2); the bench reports their count.
"""
from __future__ import annotations

import numpy as np

W_EXP = 29.0
W_LOG = 44.0


class FlopModel:
    def __init__(self, mt, stages=6):
        nu_f = np.asarray(mt.nu_f)
        nu_r = np.asarray(mt.nu_r)
        net = nu_r - nu_f
        typ = np.asarray(mt.type)
        ns, nr = mt.ns, mt.nr
        nnz_f = int(np.count_nonzero(nu_f))
        nnz_r = int(np.count_nonzero(nu_r))
        nnz = int(np.count_nonzero(net))
        n_fo = int(np.sum(typ >= 2))
        n_tb = int(np.sum(typ >= 1))
        active = int(np.sum(np.any(net != 0, axis=0)))
        self.n = n = active + 1
        self.n_log = 1 + ns
        self.n_exp = 2 * nr + 3 * n_fo
        self.rhs_plain = (24 * ns + 4 * nr + 2 * nnz + 2 * nr + 2 * (nnz_f + nnz_r) + nr + 2 * ns * n_tb
                          + 30 * n_fo + 2 * nnz + 6 * ns)
        self.rhs = self.rhs_plain + W_LOG * self.n_log + W_EXP * self.n_exp
        jac = 0.0
        for r in range(nr):
            jac += 2 * np.count_nonzero(net[r]) * (np.count_nonzero(nu_f[r]) + np.count_nonzero(nu_r[r]))
        self.jac = jac + 2 * n_tb * nnz * ns / max(nr, 1) + 15 * nr + 3 * n * n
        self.lu = 2.0 * n ** 3 / 3.0
        self.solve = 2.0 * n * n
        self.control = 10.0 * n
        self.stages = stages

    def per_step(self):
        """FLOPs of one attempted (non-frozen) substep: s RHS + J + LU + s solves + control."""
        if self.stages == 0:           # the paper's explicit scheme: one RHS per step
            return self.rhs
        return self.stages * self.rhs + self.jac + self.lu + self.stages * self.solve + self.control

    def flops(self, stats):
        """Algorithmic FLOPs of one chem_integrate call from its chem_stats counters."""
        frozen = stats.get("steps_frozen", 0)
        return (stats["steps_attempted"] - frozen) * self.per_step() + frozen * self.rhs

    def table(self):
        return {"rhs_plain": self.rhs_plain, "rhs_logs": self.n_log, "rhs_exps": self.n_exp, "w_log": W_LOG,
                "w_exp": W_EXP, "rhs": self.rhs, "jacobian": self.jac, "lu": self.lu, "solve": self.solve,
                "control": self.control, "stages": self.stages, "n": self.n, "per_substep": self.per_step()}


# FP64 peak of one B200 from unit counts and clocks: 148 SMs x 64 FP64 FMA lanes per
# SM per clock x 2 flops x the max SM clock.  The measured DFMA-loop peak is profiles/fp64_peak.json.
def fp64_peak_tflops(sm_count=148, sm_mhz=1965.0, fma_per_sm=64):
    return sm_count * fma_per_sm * 2 * sm_mhz * 1e6 / 1e12
