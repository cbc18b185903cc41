"""CPU emulation of the row-slab multi-GPU solve; TEST
INFRASTRUCTURE ONLY.

Every rank of a torch.distributed group (gloo on CPU) owns the row bands that
paper_2010_10232_b200.slabs.plan() assigns it and runs the DC_MG-preconditioned
GMRES of the reference (src/precond.cpp:196-265, src/linalg.cpp:10-92) on them,
communicating exactly where the device implementation will:

* halo exchange (neighbour send/recv of ``band`` rows) before every level apply
  and before every transfer whose input rows cross a slab boundary;
* allgather of the restricted right-hand side at the gather level (the rest of
  the V-cycle and the coarsest direct solve run redundantly) and of the
  deflation coarse vector (redundant E solve);
* three deterministic allreduces per iteration: pass 1 of the one-reduction
  Arnoldi (s = V^H w and the new Gram row, 2j+1 complex), pass 2 (||u_{j+1}||)
  and the true-residual monitor.  "Deterministic" = allgather of the per-rank
  partials, summed in rank order on every rank.

Operators are the Kronecker sums of the banded 1D factors (the device layout);
the result is compared with the oracle's single-domain solve in
tests/test_slabs.py.  Counts of every communication are returned so the plan's
per-iteration model can be checked.
"""
from __future__ import annotations

import collections
import os

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_2010_10232_b200 import slabs


class Comm:
    def __init__(self, rank: int, ws: int):
        self.rank, self.ws = rank, ws
        self.counts = collections.Counter()
        if ws > 1:
            import torch
            import torch.distributed as dist
            self.torch, self.dist = torch, dist

    def _t(self, a):
        a = np.ascontiguousarray(a)
        if np.iscomplexobj(a):
            a = a.view(np.float64)
        return self.torch.from_numpy(a.astype(np.float64, copy=True))

    def allreduce(self, a):
        """Sum over ranks in rank order (deterministic)."""
        a = np.asarray(a)
        if self.ws == 1:
            return a.copy()
        self.counts["allreduce"] += 1
        t = self._t(a.reshape(-1))
        parts = [self.torch.empty_like(t) for _ in range(self.ws)]
        self.dist.all_gather(parts, t)
        tot = parts[0].numpy().copy()
        for p in parts[1:]:
            tot = tot + p.numpy()
        if np.iscomplexobj(a):
            tot = tot.view(np.complex128)
        return tot.reshape(a.shape)

    def allgather_rows(self, local, bounds, n_cols):
        """Concatenate the row bands (rank order) into the whole level vector."""
        if self.ws == 1:
            return local.copy()
        self.counts["allgather"] += 1
        rows = [bounds[r + 1] - bounds[r] for r in range(self.ws)]
        mx = max(rows)
        buf = np.zeros((mx, n_cols), np.complex128)
        buf[: local.shape[0]] = local
        t = self._t(buf)
        parts = [self.torch.empty_like(t) for _ in range(self.ws)]
        self.dist.all_gather(parts, t)
        out = [p.numpy().view(np.complex128).reshape(mx, n_cols)[: rows[r]] for r, p in enumerate(parts)]
        return np.concatenate(out, axis=0)

    def exchange(self, local, top, bottom):
        """Return local extended by ``top`` rows of the upper neighbour and
        ``bottom`` rows of the lower one (zeros at the domain edges)."""
        n_cols = local.shape[1]
        ext = np.zeros((top + local.shape[0] + bottom, n_cols), np.complex128)
        ext[top: top + local.shape[0]] = local
        if self.ws == 1 or (top == 0 and bottom == 0):
            return ext
        self.counts["halo_exchange"] += 1
        self.counts["halo_bytes"] += 16 * n_cols * ((top if self.rank > 0 else 0) +
                                                    (bottom if self.rank < self.ws - 1 else 0))
        dist, r = self.dist, self.rank
        ops, recv = [], {}
        if r > 0:
            if bottom:
                ops.append(dist.P2POp(dist.isend, self._t(local[:bottom]), r - 1))
            if top:
                recv["top"] = self.torch.empty(2 * top * n_cols, dtype=self.torch.float64)
                ops.append(dist.P2POp(dist.irecv, recv["top"], r - 1))
        if r < self.ws - 1:
            if top:
                ops.append(dist.P2POp(dist.isend, self._t(local[local.shape[0] - top:]), r + 1))
            if bottom:
                recv["bot"] = self.torch.empty(2 * bottom * n_cols, dtype=self.torch.float64)
                ops.append(dist.P2POp(dist.irecv, recv["bot"], r + 1))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if "top" in recv:
            ext[:top] = recv["top"].numpy().view(np.complex128).reshape(top, n_cols)
        if "bot" in recv:
            ext[top + local.shape[0]:] = recv["bot"].numpy().view(np.complex128).reshape(bottom, n_cols)
        return ext


def band_of(*mats):
    b = 0
    for m in mats:
        r, c = np.nonzero(np.abs(m) > 0)
        if r.size:
            b = max(b, int(np.max(np.abs(r - c))))
    return b


def linear_z(fine):  # src/precond.cpp:57-76 (0-based: coarse q <- fine 2q, 2q+1, 2q+2)
    nc = fine // 2
    z = np.zeros((fine, nc))
    for q in range(nc):
        z[2 * q, q] += 0.5
        z[2 * q + 1, q] += 1.0
        if 2 * q + 2 < fine:
            z[2 * q + 2, q] += 0.5
    return z


def bezier_z(fine, drop):  # src/precond.cpp:34-55 (coarse q <- fine 2q-1 .. 2q+3)
    nc = fine // 2
    z = np.zeros((fine, nc))
    for q in range(nc):
        for off, w in ((-1, 0.125), (0, 0.5), (1, (6.0 - drop) / 8.0), (2, 0.5), (3, 0.125)):
            i = 2 * q + off
            if 0 <= i < fine:
                z[i, q] += w
    return z


class KronLevel:
    """sum_t coef_t outer_t (x) inner_t on an n x n grid (x fastest)."""

    def __init__(self, terms):
        self.terms = terms
        self.n = terms[0][1].shape[0]
        self.band = band_of(*[a for _, a, _ in terms], *[b for _, _, b in terms])
        self.diag = sum(c * np.outer(np.diag(a), np.diag(b)) for c, a, b in terms)

    def galerkin(self, z):
        return KronLevel([(c, z.T @ a @ z, z.T @ b @ z) for c, a, b in self.terms])

    def apply_rows(self, ext, r0, r1, top):
        """Rows [r0, r1) of L x from ext = x rows [r0-top, r0-top+len(ext))."""
        e0 = r0 - top
        lo, hi = max(0, e0), min(self.n, e0 + ext.shape[0])
        xs = ext[lo - e0: hi - e0]
        return sum(c * (a[r0:r1, lo:hi] @ xs @ b.T) for c, a, b in self.terms)

    def sparse(self):
        return sum(c * sp.kron(sp.csr_matrix(a), sp.csr_matrix(b), format="csc") for c, a, b in self.terms)


def restrict_rows(z, ext, top, f0, q0, q1):
    """rc rows [q0, q1) = (z^T R z)[q0:q1] from fine rows ext = R[f0-top ...]."""
    e0 = f0 - top
    lo, hi = max(0, e0), min(z.shape[0], e0 + ext.shape[0])
    return z[lo:hi, q0:q1].T @ ext[lo - e0: hi - e0] @ z


def prolong_rows(z, ext, top, q0, f0, f1):
    """rows [f0, f1) of z E z^T from coarse rows ext = E[q0-top ...]."""
    e0 = q0 - top
    lo, hi = max(0, e0), min(z.shape[1], e0 + ext.shape[0])
    return z[f0:f1, lo:hi] @ ext[lo - e0: hi - e0] @ z.T


class SlabSolver:
    def __init__(self, comm, S1, M1, k, spec, per_dim, agglomerate_at=200, min_rows=8):
        self.comm = comm
        c_a = complex(k * k)
        c_m = complex(k * k) * complex(1.0, -spec.beta2)
        self.A = KronLevel([(1.0, M1, S1), (1.0, S1, M1), (-c_a, M1, M1)])
        self.spec = spec
        # MG hierarchy (Galerkin with linear z, src/precond.cpp:115-124)
        sizes = slabs.level_sizes(per_dim)
        self.levels = [KronLevel([(1.0, M1, S1), (1.0, S1, M1), (-c_m, M1, M1)])]
        self.zl = []
        for n in sizes[:-1]:
            z = linear_z(n)
            self.zl.append(z)
            self.levels.append(self.levels[-1].galerkin(z))
        self.coarsest = spla.splu(self.levels[-1].sparse())
        # deflation (src/precond.cpp:93-108): E = Z^T A Z, Z = zb (x) zb
        self.zb = bezier_z(per_dim, spec.drop)
        # E itself is formed as the reference forms it (sparse Z^T A Z): its LU
        # amplifies rounding differences of its entries by cond(E)
        self.E = self.A.galerkin(self.zb)  # band only
        Z = sp.kron(sp.csr_matrix(self.zb), sp.csr_matrix(self.zb), format="csr").astype(np.complex128)
        E = (Z.T @ self.A.sparse() @ Z).tocsc()
        E.eliminate_zeros()
        self.E_lu = spla.splu(E)
        self.plan = slabs.plan(per_dim, [L.band for L in self.levels], comm.ws, self.E.band,
                               agglomerate_at=agglomerate_at, min_rows=min_rows)
        self.n = per_dim
        self.rows = self.plan.fine.rows(comm.rank)

    # ---- level primitives on row bands
    def lev_apply(self, l, x):
        pl = self.plan.levels[l]
        L = self.levels[l]
        if not pl.distributed:
            return L.apply_rows(x, 0, pl.n, 0)
        r0, r1 = pl.rows(self.comm.rank)
        b = L.band
        return L.apply_rows(self.comm.exchange(x, b, b), r0, r1, b)

    def lev_diag(self, l):
        pl = self.plan.levels[l]
        r0, r1 = pl.rows(self.comm.rank)
        return self.levels[l].diag[r0:r1]

    def smooth(self, l, b, x, steps, x_zero):  # src/precond.cpp:136-142
        om = self.spec.omega
        d = self.lev_diag(l)
        for s in range(steps):
            if x_zero and s == 0:
                x = om * (b / d)  # x + om D^-1 (b - M 0), exact
            else:
                x = x + om * ((b - self.lev_apply(l, x)) / d)
        return x

    def restrict(self, l, r):
        pl, pc = self.plan.levels[l], self.plan.levels[l + 1]
        if not pl.distributed:
            return restrict_rows(self.zl[l], r, 0, 0, 0, pc.n)
        f0, _ = pl.rows(self.comm.rank)
        q0, q1 = pc.bounds[self.comm.rank], pc.bounds[self.comm.rank + 1]
        top, bot = slabs.TRANSFER_HALO[("restrict", "linear")]
        rc = restrict_rows(self.zl[l], self.comm.exchange(r, top, bot), top, f0, q0, q1)
        if not pc.distributed:
            rc = self.comm.allgather_rows(rc, pc.bounds, pc.n)
        return rc

    def prolong(self, l, ec):
        pl, pc = self.plan.levels[l], self.plan.levels[l + 1]
        if not pl.distributed:
            return prolong_rows(self.zl[l], ec, 0, 0, 0, pl.n)
        f0, f1 = pl.rows(self.comm.rank)
        if pc.distributed:
            q0, _ = pc.rows(self.comm.rank)
            top, bot = slabs.TRANSFER_HALO[("prolong", "linear")]
            return prolong_rows(self.zl[l], self.comm.exchange(ec, top, bot), top, q0, f0, f1)
        return prolong_rows(self.zl[l], ec, 0, 0, f0, f1)  # gathered: every coarse row is local

    def cycle(self, l, b, x, x_zero):  # src/precond.cpp:144-153
        if l == len(self.levels) - 1:
            return self.coarsest.solve(b.reshape(-1)).reshape(b.shape)
        nu = self.spec.smooth_steps
        x = self.smooth(l, b, x, nu, x_zero)
        r = b - self.lev_apply(l, x)
        rc = self.restrict(l, r)
        ec = self.cycle(l + 1, rc, np.zeros_like(rc), True)
        x = x + self.prolong(l, ec)
        return self.smooth(l, b, x, nu, False)

    def mg_solve(self, b):  # src/precond.cpp:159-163
        x = np.zeros_like(b)
        for c in range(self.spec.cycles):
            x = self.cycle(0, b, x, c == 0)
        return x

    def apply_Q(self, v):  # Z E^-1 Z^T v (src/precond.cpp:93-108)
        pf, pc = self.plan.fine, self.plan.coarse
        f0, f1 = self.rows
        top, bot = slabs.TRANSFER_HALO[("restrict", "bezier")]
        ext = self.comm.exchange(v, top, bot) if self.comm.ws > 1 else v
        if self.comm.ws > 1:
            q0, q1 = pc.bounds[self.comm.rank], pc.bounds[self.comm.rank + 1]
            rc = restrict_rows(self.zb, ext, top, f0, q0, q1)
            rc = self.comm.allgather_rows(rc, pc.bounds, pc.n)
        else:
            rc = restrict_rows(self.zb, v, 0, 0, 0, pc.n)
        ec = self.E_lu.solve(rc.reshape(-1)).reshape(rc.shape)
        return prolong_rows(self.zb, ec, 0, 0, f0, f1)

    def fine_apply(self, v):
        if self.comm.ws == 1:
            return self.A.apply_rows(v, 0, self.n, 0)
        b = self.A.band
        f0, f1 = self.rows
        return self.A.apply_rows(self.comm.exchange(v, b, b), f0, f1, b)

    def project(self, w):
        return w - self.apply_Q(self.fine_apply(w))

    def op(self, v):  # src/precond.cpp:236-245
        return self.project(self.mg_solve(self.fine_apply(v)))

    def norm(self, v):
        return float(np.sqrt(self.comm.allreduce(np.array([np.vdot(v, v).real]))[0]))

    # ---- one-reduction Arnoldi GMRES (algebraically src/linalg.cpp:10-92)
    def gmres(self, f_local, maxit=100, tol=1e-7):
        comm = self.comm
        fnorm = self.norm(f_local)
        scale = fnorm if fnorm > 0.0 else 1.0

        def monitor(x):
            return self.norm(f_local - self.fine_apply(x)) / scale

        rhs = self.project(self.mg_solve(f_local))
        x0 = self.apply_Q(f_local)
        hist = []
        r0 = monitor(x0)
        if r0 <= tol:
            return x0, 0, True, [r0], dict(comm.counts), dict(comm.counts)
        r = rhs - self.op(x0)
        beta = self.norm(r)
        U, sig = [r], [1.0 / beta]
        H = np.zeros((maxit + 1, maxit), np.complex128)
        Lg = np.zeros((maxit + 1, maxit + 1), np.complex128)
        g = np.zeros(maxit + 1, np.complex128)
        g[0] = beta
        cs = np.zeros(maxit, np.complex128)
        sn = np.zeros(maxit, np.complex128)
        x = x0
        conv = False
        setup_counts = dict(comm.counts)
        it = 0
        for j in range(maxit):
            w = self.op(U[j]) * sig[j]
            # pass 1: s_i = v_i^H w (i <= j), Gram row v_j^H v_l (l < j): ONE allreduce
            loc = np.empty(2 * j + 1, np.complex128)
            for i in range(j + 1):
                loc[i] = sig[i] * np.vdot(U[i], w)
            for l in range(j):
                loc[j + 1 + l] = sig[j] * sig[l] * np.vdot(U[j], U[l])
            tot = comm.allreduce(loc)
            s, Lg[j, :j] = tot[: j + 1], tot[j + 1:]
            h = np.empty(j + 1, np.complex128)
            for i in range(j + 1):  # (I + L) h = s
                h[i] = s[i] - np.dot(Lg[i, :i], h[:i])
            u = w.copy()
            for i in range(j + 1):
                u -= (h[i] * sig[i]) * U[i]
            hnew = self.norm(u)  # pass 2: ONE allreduce
            H[: j + 1, j] = h
            H[j + 1, j] = hnew
            for i in range(j):  # redundant Givens on every rank (:49-66)
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + np.conj(cs[i]) * H[i + 1, j]
                H[i, j] = t
            den = np.sqrt(abs(H[j, j]) ** 2 + abs(H[j + 1, j]) ** 2)
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = np.conj(H[j, j]) / den, np.conj(H[j + 1, j]) / den
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            m = j + 1
            y = np.zeros(m, np.complex128)
            for i in range(m - 1, -1, -1):
                y[i] = (g[i] - np.dot(H[i, i + 1: m], y[i + 1: m])) / H[i, i]
            x = x0.copy()
            for i in range(m):
                x += (y[i] * sig[i]) * U[i]
            rr = monitor(x)  # ONE allreduce
            hist.append(rr)
            it = j + 1
            if rr <= tol:
                conv = True
                break
            if hnew < 1e-300:
                break
            U.append(u)
            sig.append(1.0 / hnew)
        return x, it, conv, hist, setup_counts, dict(comm.counts)


def run_rank(rank, ws, port, out_dir, cfg):
    """Entry point of one emulated rank (torch.multiprocessing.spawn target)."""
    import sys
    sys.path.insert(0, cfg["root"])
    from oracle import helmdef_oracle as O  # test infrastructure: builds the inputs
    if ws > 1:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        pb = O.point_source_2d(cfg["elements"], cfg["p"], cfg["k"])
        sys_ = O.assemble(pb)
        spec = O.to_spec(cfg["tag"], cfg["p"], cfg["k"], beta2=cfg.get("beta2", "1"),
                         cycles=cfg.get("cycles", 1), smoothing=cfg.get("smoothing", 1),
                         omega=cfg.get("omega", 0.6))
        comm = Comm(rank, ws)
        S1 = np.asarray(sys_.S1.toarray() if sp.issparse(sys_.S1) else sys_.S1)
        M1 = np.asarray(sys_.M1.toarray() if sp.issparse(sys_.M1) else sys_.M1)
        sol = SlabSolver(comm, S1, M1, sys_.k, spec, sys_.per_dim, agglomerate_at=cfg.get("agglomerate_at", 200),
                         min_rows=cfg.get("min_rows", 8))
        n = sys_.per_dim
        f0, f1 = sol.rows
        F = sys_.rhs.reshape(n, n)
        res = {}
        # component checks on a seeded vector: fine apply, MG solve, Q, op
        rng = np.random.default_rng(7)
        V = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        res["apply"] = sol.fine_apply(V[f0:f1])
        res["mg"] = sol.mg_solve(V[f0:f1])
        res["Q"] = sol.apply_Q(V[f0:f1])
        res["op"] = sol.op(V[f0:f1])
        comm.counts.clear()
        x, it, conv, hist, c_setup, c_all = sol.gmres(F[f0:f1].copy(), cfg.get("maxit", 100), cfg.get("tol", 1e-7))
        res["x"] = x
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), rows=np.array([f0, f1]), iterations=it, converged=conv,
                 hist=np.array(hist), gather_level=sol.plan.gather_level,
                 setup_counts=np.array([c_setup.get(k_, 0) for k_ in ("allreduce", "allgather", "halo_exchange")]),
                 all_counts=np.array([c_all.get(k_, 0) for k_ in ("allreduce", "allgather", "halo_exchange")]),
                 halo_bytes=c_all.get("halo_bytes", 0), **res)
    finally:
        if ws > 1:
            dist.destroy_process_group()
