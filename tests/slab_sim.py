"""TEST INFRASTRUCTURE: numpy restatement of the i-slab decomposed interleaved
PCG that libacg_cuda.so runs across GPUs (one slab per rank), used by
test_decomposition_gloo.py to check the host-side decomposition logic on CPU
with real torch.distributed (gloo) collectives:

  * the slab plan comes from the library itself (acg_partition_plan);
  * halo exchange of one ghost i-plane per neighbour before every stencil;
  * per-column partials -> slab-local pairwise tree -> all_gather of the slab
    sums -> perfect tree over slabs (when the plan is tree-aligned);
  * the scalar recurrences of solver.hpp:288-364 replicated on every rank.

Arithmetic follows the reference's association order (numpy float64
elementwise ops are plain IEEE operations), so the result must equal the
full-domain oracle bit for bit.
"""
import numpy as np
import torch
import torch.distributed as dist


def psum(v):
    """parallel.hpp:11-20"""
    n = len(v)
    if n <= 8:
        s = 0.0
        for x in v:
            s += x
        return s
    h = n // 2
    return psum(v[:h]) + psum(v[h:])


def perfect(vals):
    v = list(vals)
    w = 1
    while w < len(v):
        for s in range(0, len(v) - w, 2 * w):
            v[s] = v[s] + v[s + w]
        w *= 2
    return v[0]


class Slab:
    def __init__(self, o, i0, i1, rank, world, exact):
        self.o, self.i0, self.i1, self.rank, self.world, self.exact = o, i0, i1, rank, world, exact
        m, n_z = o.prob.m, o.prob.n_z
        self.m, self.n_z, self.ml = m, n_z, i1 - i0
        self.ap, self.bp, self.cp, self.d = o.ap, o.bp, o.cp, o.d
        gi = np.arange(i0, i1)
        self.area = o.area[i0:i1]
        self.adiag = o.diag[i0:i1]
        east = np.zeros((m, m))
        north = np.zeros((m, m))
        if m > 1:
            east[:m - 1] = o.east
            north[:, :m - 1] = o.north
        self.ae = np.where((gi + 1 < m)[:, None], east[i0:i1], 0.0)
        self.aw = np.where((gi > 0)[:, None], east[np.maximum(gi - 1, 0)], 0.0)
        self.an = np.where(np.arange(m)[None, :] + 1 < m, north[i0:i1], 0.0)
        self.as_ = np.where(np.arange(m)[None, :] > 0, np.roll(north[i0:i1], 1, axis=1), 0.0)
        self.has_e = (gi + 1 < m)[:, None]
        self.has_w = (gi > 0)[:, None]

    # ------------------------------------------------------------ halos
    def halo(self, x):
        """x: (ml+2, m, n_z) with ghost planes 0 and ml+1."""
        reqs = []
        if self.rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[1])), self.rank - 1))
        if self.rank + 1 < self.world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[self.ml])), self.rank + 1))
        if self.rank > 0:
            t = torch.empty(x[0].shape, dtype=torch.float64)
            dist.recv(t, self.rank - 1)
            x[0] = t.numpy()
        if self.rank + 1 < self.world:
            t = torch.empty(x[0].shape, dtype=torch.float64)
            dist.recv(t, self.rank + 1)
            x[self.ml + 1] = t.numpy()
        for r in reqs:
            r.wait()

    def stencil(self, x, k):
        """7-point value at level k for the slab's columns (operator.hpp:127-132)."""
        c = x[1:-1, :, k]
        up = x[1:-1, :, k + 1] if k + 1 < self.n_z else c
        dn = x[1:-1, :, k - 1] if k > 0 else c
        e = np.where(self.has_e, x[2:, :, k], c)
        w = np.where(self.has_w, x[:-2, :, k], c)
        nb = np.concatenate([c[:, 1:], c[:, -1:]], axis=1)
        sb = np.concatenate([c[:, :1], c[:, :-1]], axis=1)
        A = self.area
        t = ((self.ap[k] - self.bp[k] - self.cp[k]) * A - self.adiag) * c
        t = t + A * self.bp[k] * up
        t = t + A * self.cp[k] * dn
        t = t + self.ae * e
        t = t + self.aw * w
        t = t + self.an * nb
        t = t + self.as_ * sb
        return t

    # ------------------------------------------------------------ reductions
    def reduce(self, parts):
        """parts: list of (ml, m) per-column partial arrays -> global sums."""
        local = [psum(list(p.reshape(-1))) for p in parts]
        gathered = [None] * self.world
        dist.all_gather_object(gathered, local)
        out = []
        for a in range(len(parts)):
            vals = [g[a] for g in gathered]
            out.append(perfect(vals) if self.exact else psum(vals))
        return out

    # ------------------------------------------------------------ kernels
    def apply(self, x):
        self.halo(x)
        y = np.zeros_like(x)
        for k in range(self.n_z):
            y[1:-1, :, k] = self.stencil(x, k) * self.d[k]
        return y

    def dot_parts(self, x, y):
        s = np.zeros((self.ml, self.m))
        for k in range(self.n_z):
            s = s + x[1:-1, :, k] * y[1:-1, :, k]
        return s

    def precondition(self, y):
        x = np.zeros_like(y)
        A = self.area
        at = self.adiag / A
        phi = np.zeros((self.ml, self.m, self.n_z))
        dg = (self.ap[0] - self.bp[0] - self.cp[0]) - at
        phi[:, :, 0] = self.bp[0] / dg
        x[1:-1, :, 0] = y[1:-1, :, 0] / (A * self.d[0]) / dg
        for k in range(1, self.n_z):
            dg = ((self.ap[k] - self.bp[k] - self.cp[k]) - at) - phi[:, :, k - 1] * self.cp[k]
            phi[:, :, k] = self.bp[k] / dg
            x[1:-1, :, k] = (y[1:-1, :, k] / (A * self.d[k]) - self.cp[k] * x[1:-1, :, k - 1]) / dg
        for k in range(self.n_z - 2, -1, -1):
            x[1:-1, :, k] = x[1:-1, :, k] - phi[:, :, k] * x[1:-1, :, k + 1]
        return x

    def fused_prec(self, r, z, q, alpha):
        A = self.area
        at = self.adiag / A
        phi = np.zeros((self.ml, self.m, self.n_z))
        r2 = np.zeros((self.ml, self.m))
        dg = (self.ap[0] - self.bp[0] - self.cp[0]) - at
        phi[:, :, 0] = self.bp[0] / dg
        rs = r[1:-1, :, 0] - alpha * q[1:-1, :, 0]
        r2 = r2 + rs * rs
        z[1:-1, :, 0] = rs / (dg * A * self.d[0])
        r[1:-1, :, 0] = rs
        for k in range(1, self.n_z):
            dg = ((self.ap[k] - self.bp[k] - self.cp[k]) - at) - phi[:, :, k - 1] * self.cp[k]
            phi[:, :, k] = self.bp[k] / dg
            rs = r[1:-1, :, k] - alpha * q[1:-1, :, k]
            r2 = r2 + rs * rs
            z[1:-1, :, k] = (rs / (A * self.d[k]) - self.cp[k] * z[1:-1, :, k - 1]) / dg
            r[1:-1, :, k] = rs
        n = self.n_z - 1
        kap = z[1:-1, :, n] * r[1:-1, :, n]
        for k in range(self.n_z - 2, -1, -1):
            zs = z[1:-1, :, k] - phi[:, :, k] * z[1:-1, :, k + 1]
            kap = kap + zs * r[1:-1, :, k]
            z[1:-1, :, k] = zs
        return r2, kap

    def fused_spmv(self, u, p, q, z, alpha, beta):
        self.halo(z)
        sig = np.zeros((self.ml, self.m))
        for k in range(self.n_z):
            ps, qs, zs = p[1:-1, :, k], q[1:-1, :, k], z[1:-1, :, k]
            u[1:-1, :, k] = u[1:-1, :, k] + alpha * ps
            ps = beta * ps + zs
            qs = beta * qs
            p[1:-1, :, k] = ps
            dq = self.stencil(z, k)
            qs = qs + self.d[k] * dq
            sig = sig + ps * qs
            q[1:-1, :, k] = qs
        return sig

    # ------------------------------------------------------------ driver
    def solve(self, f_full, epsilon, tau, maxiter):
        """pcg_interleaved (solver.hpp:275-370) over the slab; returns (u slab, history)."""
        shape = (self.ml + 2, self.m, self.n_z)
        u, r, z, p, q = (np.zeros(shape) for _ in range(5))
        r[1:-1] = f_full[self.i0:self.i1]
        q = self.apply(u)
        r[1:-1] = -1.0 * q[1:-1] + r[1:-1]
        (s,) = self.reduce([self.dot_parts(r, r)])
        rn = np.sqrt(s)
        r0 = rn
        hist = [rn]
        if r0 <= tau:
            return u[1:-1], hist, 0
        z = self.precondition(r)
        (kold,) = self.reduce([self.dot_parts(r, z)])
        p = z.copy()
        q = self.apply(p)
        (sg,) = self.reduce([self.dot_parts(p, q)])
        al = kold / sg
        it = 0
        for it in range(1, maxiter + 1):
            r2p, kp = self.fused_prec(r, z, q, al)
            s2, ka = self.reduce([r2p, kp])
            rn = np.sqrt(s2)
            hist.append(rn)
            if rn / r0 < epsilon or rn < tau:
                u[1:-1] = al * p[1:-1] + u[1:-1]
                break
            be = ka / kold
            kold = ka
            sgp = self.fused_spmv(u, p, q, z, al, be)
            (sg,) = self.reduce([sgp])
            al = kold / sg
        return u[1:-1], hist, it
