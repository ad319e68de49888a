"""World-free end-to-end oracle: create once, then update + solve per step.

Mirrors the reference protocol (cli.py:181-272): repartition at step 1, then
per step perturb -> update -> cg_solve with b = ones.  Used by the tests as the
checker and by bench.py's CPU-baseline legs as the timed "port" of the
reference CPU path.  Test infrastructure only.
"""

import numpy as np

from . import krylov, repart


class OraclePipeline:
    def __init__(self, problems, offsets, alpha):
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.alpha = int(alpha)
        self.n_gpu = (len(self.offsets) - 1) // self.alpha
        self.parts = [repart.build_owner(problems, self.offsets, self.alpha, k)
                      for k in range(self.n_gpu)]
        self.plans = repart.halo_plan(self.parts, self.offsets, self.alpha)
        self.values = None
        self.update(problems)

    def update(self, problems):
        """pack -> transfer -> apply_scatter for every owner (update.py:115-132)."""
        self.values = [repart.scatter_values(p, repart.owner_buffer(problems, self.alpha, p.k))
                       for p in self.parts]

    @property
    def system(self):
        return krylov.DistSystem(self.parts, self.values, self.plans)

    def rhs_ones(self):
        return [np.ones(p.hi - p.lo) for p in self.parts]

    def solve(self, method="cg", tol=1e-6, max_iter=2000, bs=None):
        bs = self.rhs_ones() if bs is None else bs
        if method == "cg":
            return krylov.cg(self.system, bs, tol, max_iter)
        if method == "pcg":
            return krylov.cg(self.system, bs, tol, max_iter, jacobi=True)
        if method == "pcg1":
            return krylov.pcg1(self.system, bs, tol, max_iter)
        if method == "pipecg":
            return krylov.pipecg(self.system, bs, tol, max_iter)
        if method == "bicgstab":
            return krylov.bicgstab(self.system, bs, tol, max_iter)
        raise ValueError(f"unknown method {method!r}")
