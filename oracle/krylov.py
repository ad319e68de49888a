"""Oracle restatement of the distributed SpMV and Krylov solvers.

CG follows the reference solver.py:80-147 operation by operation (ordered
allreduce in ascending owner rank, transport.py:450-458; true residual every
10 iterations or when the recurrence residual meets tol).  Jacobi-PCG,
BiCGStab and the single-reduction (Chronopoulos-Gear) Jacobi-PCG are not in
the reference; they follow SURVEY.md Appendix A / §8 f1 with the same
stopping rule and reduction order.  Every elementwise update is written
as separate numpy operations so each product/sum is rounded once, exactly as
the CUDA kernels do (no FMA).  Test infrastructure only.
"""

import math

import numpy as np


def allreduce(parts_values):
    """((v0 + v1) + v2) + ... in ascending owner order (transport.py:450-458)."""
    total = parts_values[0]
    for v in parts_values[1:]:
        total = total + v
    return total


class DistSystem:
    """Owner parts with their values and halo plans (world-free)."""

    def __init__(self, parts, values, plans):
        self.parts = parts          # list[OwnerPart]
        self.values = values        # list[(local_vals, nonlocal_vals)]
        self.plans = plans          # list[(send_indices, recv_slots)]

    @property
    def n_parts(self):
        return len(self.parts)

    def spmv(self, xs):
        """y_g = A_loc x_g + A_nl x_halo (solver.py:80-97), np.add.at order."""
        ys = []
        for g, p in enumerate(self.parts):
            send_unused, recv = self.plans[g]
            xh = np.zeros(len(p.halo_cols))
            for j, slots in recv.items():
                xh[slots] = xs[j][self.plans[j][0][g]]
            lv, nv = self.values[g]
            y = np.zeros(p.hi - p.lo)
            np.add.at(y, p.loc_rows, lv * xs[g][p.loc_cols])
            if len(p.nl_rows):
                np.add.at(y, p.nl_rows, nv * xh[p.nl_cols])
            ys.append(y)
        return ys

    def dot(self, a, b):
        return allreduce([float(x @ y) for x, y in zip(a, b)])

    def dinv(self):
        out = []
        for p, (lv, _) in zip(self.parts, self.values):
            d = np.zeros(p.hi - p.lo)
            m = p.loc_rows == p.loc_cols
            d[p.loc_rows[m]] = lv[m]
            out.append(1.0 / d)
        return out


class Report:
    def __init__(self, iterations, residual, converged, history, log):
        self.iterations = iterations
        self.residual = residual
        self.converged = converged
        self.history = history      # recurrence residual per iteration
        self.log = log              # every allreduce result, in call order

    def __repr__(self):
        return (f"Report(it={self.iterations}, res={self.residual:.6e}, "
                f"conv={self.converged})")


def _true_residual(S, bs, xs, bnorm, log):
    ax = S.spmv(xs)
    tr = allreduce([float(((b - y) ** 2).sum()) for b, y in zip(bs, ax)])
    log.append(tr)
    return math.sqrt(tr) / bnorm


def cg(S: DistSystem, bs, tol, max_iter, jacobi=False):
    """Distributed CG (solver.py:100-147); ``jacobi`` = SURVEY App. A PCG."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    log, hist = [], []
    xs = [np.zeros(len(b)) for b in bs]
    bb = S.dot(bs, bs)
    log.append(bb)
    if bb == 0.0:
        return xs, Report(0, 0.0, True, hist, log)
    bnorm = math.sqrt(bb)
    rs = [b.astype(np.float64).copy() for b in bs]
    if jacobi:
        dinv = S.dinv()
        zs = [d * r for d, r in zip(dinv, rs)]
        rho = S.dot(rs, zs)
        log.append(rho)
        ps = [z.copy() for z in zs]
    else:
        rho = bb
        ps = [r.copy() for r in rs]
    res, converged, it = 1.0, False, 0
    for it in range(1, max_iter + 1):
        qs = S.spmv(ps)
        pq = S.dot(ps, qs)
        log.append(pq)
        if pq <= 0.0:
            raise ValueError("cg: matrix is not positive definite")
        step = rho / pq
        for x, r, p, q in zip(xs, rs, ps, qs):
            x += step * p
            r -= step * q
        rr = S.dot(rs, rs)
        log.append(rr)
        if jacobi:
            zs = [d * r for d, r in zip(dinv, rs)]
            rho_new = S.dot(rs, zs)
            log.append(rho_new)
        else:
            zs, rho_new = rs, rr
        rec = math.sqrt(rr) / bnorm
        hist.append(rec)
        if rec <= tol or it % 10 == 0:
            res = _true_residual(S, bs, xs, bnorm, log)
            if res <= tol:
                converged = True
                break
        else:
            res = rec
        beta = rho_new / rho
        ps = [z + beta * p for z, p in zip(zs, ps)]
        rho = rho_new
    return xs, Report(it, float(res), converged, hist, log)


def bicgstab(S: DistSystem, bs, tol, max_iter):
    """Unpreconditioned BiCGStab (van der Vorst), SURVEY App. A conventions.

    r̂0 = r0 = b (x0 = 0).  Breakdown (rho == 0, r̂0·v == 0 or omega == 0)
    stops with converged=False instead of raising.
    """
    if tol <= 0:
        raise ValueError("tol must be positive")
    log, hist = [], []
    xs = [np.zeros(len(b)) for b in bs]
    bb = S.dot(bs, bs)
    log.append(bb)
    if bb == 0.0:
        return xs, Report(0, 0.0, True, hist, log)
    bnorm = math.sqrt(bb)
    rs = [b.astype(np.float64).copy() for b in bs]
    rhat = [b.astype(np.float64).copy() for b in bs]
    rho = S.dot(rhat, rs)
    log.append(rho)
    ps = vs = None
    alpha = omega = 1.0
    rho_prev = 1.0
    res, converged, it = 1.0, False, 0
    for it in range(1, max_iter + 1):
        if it == 1:
            ps = [r.copy() for r in rs]
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            ps = [r + beta * (p - omega * v) for r, p, v in zip(rs, ps, vs)]
        vs = S.spmv(ps)
        rv = S.dot(rhat, vs)
        log.append(rv)
        if rv == 0.0:
            break
        alpha = rho / rv
        ss = [r - alpha * v for r, v in zip(rs, vs)]
        ts = S.spmv(ss)
        tsd = S.dot(ts, ss)
        tt = S.dot(ts, ts)
        log += [tsd, tt]
        omega = tsd / tt if tt != 0.0 else 0.0
        xs = [x + alpha * p + omega * s for x, p, s in zip(xs, ps, ss)]
        rs = [s - omega * t for s, t in zip(ss, ts)]
        rr = S.dot(rs, rs)
        rho_prev, rho = rho, S.dot(rhat, rs)
        log += [rr, rho]
        rec = math.sqrt(rr) / bnorm
        hist.append(rec)
        if rec <= tol or it % 10 == 0:
            res = _true_residual(S, bs, xs, bnorm, log)
            if res <= tol:
                converged = True
                break
        else:
            res = rec
        if omega == 0.0 or rho == 0.0:
            break
    return xs, Report(it, float(res), converged, hist, log)


def pcg1(S: DistSystem, bs, tol, max_iter):
    """Single-reduction Jacobi-PCG (Chronopoulos-Gear).

    CG's iterates with the two reductions of an iteration fused into one:
    u = M r (M = diag^-1), w = A u, s = A p kept as recurrences,
      beta = gamma / gamma_prev, eta = delta - beta * (gamma / alpha_prev),
      alpha = gamma / eta;  p = u + beta p,  s = w + beta s,
      x += alpha p,  r -= alpha s,  u = M r,  w = A u,
      (gamma, delta, rho) = (r.u, w.u, r.r)    -- one fused allreduce.
    Same stopping rule as cg_solve (solver.py:136-142): recurrence residual
    sqrt(rho)/|b|, true residual when it meets tol or every 10 iterations.
    eta <= 0 raises like the reference's p.q <= 0 (solver.py:129-130).
    """
    if tol <= 0:
        raise ValueError("tol must be positive")
    log, hist = [], []
    xs = [np.zeros(len(b)) for b in bs]
    bb = S.dot(bs, bs)
    log.append(bb)
    if bb == 0.0:
        return xs, Report(0, 0.0, True, hist, log)
    bnorm = math.sqrt(bb)
    dinv = S.dinv()
    rs = [b.astype(np.float64).copy() for b in bs]
    us = [d * r for d, r in zip(dinv, rs)]
    ws = S.spmv(us)
    gamma, delta = S.dot(rs, us), S.dot(ws, us)
    log += [gamma, delta]
    gamma_prev = alpha_prev = 1.0
    ps = ss = None
    res, converged, it = 1.0, False, 0
    for it in range(1, max_iter + 1):
        first = it == 1
        beta = 0.0 if first else gamma / gamma_prev
        eta = delta if first else delta - beta * (gamma / alpha_prev)
        if eta <= 0.0:
            raise ValueError("cg: matrix is not positive definite")
        alpha = gamma / eta
        if first:
            ps = [u.copy() for u in us]
            ss = [w.copy() for w in ws]
        else:
            ps = [u + beta * p for u, p in zip(us, ps)]
            ss = [w + beta * s_ for w, s_ in zip(ws, ss)]
        for x, p in zip(xs, ps):
            x += alpha * p
        rs = [r - alpha * s_ for r, s_ in zip(rs, ss)]
        us = [d * r for d, r in zip(dinv, rs)]
        ws = S.spmv(us)
        gamma_prev, alpha_prev = gamma, alpha
        gamma, delta, rr = S.dot(rs, us), S.dot(ws, us), S.dot(rs, rs)
        log += [gamma, delta, rr]
        rec = math.sqrt(rr) / bnorm
        hist.append(rec)
        if rec <= tol or it % 10 == 0:
            res = _true_residual(S, bs, xs, bnorm, log)
            if res <= tol:
                converged = True
                break
        else:
            res = rec
    return xs, Report(it, float(res), converged, hist, log)


def pipecg(S: DistSystem, bs, tol, max_iter):
    """Pipelined Jacobi-PCG (Ghysels-Vanroose).

    The iteration's SpMV n = A m (m = M w) does not depend on the scalars of
    the reduction issued just before it, so that reduction can complete while
    the SpMV runs (the B200 kernel reads it one phase late):
      beta = gamma / gamma_prev, eta = delta - beta * (gamma / alpha_prev),
      alpha = gamma / eta;  n = A (M w);
      z = n + beta z,  s = w + beta s,  p = M r + beta p,
      x += alpha p,  r -= alpha s,  w -= alpha z,
      (gamma, delta, rho) = (r.Mr, w.Mr, r.r)   -- one fused allreduce.
    With M = diag^-1 the preconditioned recurrences u = M r, m = M w and
    q = M s of the published algorithm are formed directly from r, w and s
    (the same vectors in exact arithmetic; no drift of u against r).  CG's
    iterates up to rounding; same stopping rule as cg_solve
    (solver.py:136-142) and the same breakdown error as the reference's
    p.q <= 0 (solver.py:129-130).
    """
    if tol <= 0:
        raise ValueError("tol must be positive")
    log, hist = [], []
    xs = [np.zeros(len(b)) for b in bs]
    bb = S.dot(bs, bs)
    log.append(bb)
    if bb == 0.0:
        return xs, Report(0, 0.0, True, hist, log)
    bnorm = math.sqrt(bb)
    dinv = S.dinv()
    rs = [b.astype(np.float64).copy() for b in bs]
    us = [d * r for d, r in zip(dinv, rs)]
    ws = S.spmv(us)
    gamma, delta = S.dot(rs, us), S.dot(ws, us)
    log += [gamma, delta]
    gamma_prev = alpha_prev = 1.0
    zs = ss = ps = None
    res, converged, it = 1.0, False, 0
    for it in range(1, max_iter + 1):
        first = it == 1
        beta = 0.0 if first else gamma / gamma_prev
        eta = delta if first else delta - beta * (gamma / alpha_prev)
        if eta <= 0.0:
            raise ValueError("cg: matrix is not positive definite")
        alpha = gamma / eta
        ns = S.spmv([d * w for d, w in zip(dinv, ws)])
        if first:
            zs = ns
            ss = [w.copy() for w in ws]
            ps = [d * r for d, r in zip(dinv, rs)]
        else:
            zs = [n + beta * z for n, z in zip(ns, zs)]
            ss = [w + beta * s_ for w, s_ in zip(ws, ss)]
            ps = [d * r + beta * p for d, r, p in zip(dinv, rs, ps)]
        for x, p in zip(xs, ps):
            x += alpha * p
        rs = [r - alpha * s_ for r, s_ in zip(rs, ss)]
        ws = [w - alpha * z for w, z in zip(ws, zs)]
        us = [d * r for d, r in zip(dinv, rs)]
        gamma_prev, alpha_prev = gamma, alpha
        gamma, delta, rr = S.dot(rs, us), S.dot(ws, us), S.dot(rs, rs)
        log += [gamma, delta, rr]
        rec = math.sqrt(rr) / bnorm
        hist.append(rec)
        if rec <= tol or it % 10 == 0:
            res = _true_residual(S, bs, xs, bnorm, log)
            if res <= tol:
                converged = True
                break
        else:
            res = rec
    return xs, Report(it, float(res), converged, hist, log)
