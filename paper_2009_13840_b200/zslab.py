"""z-slab sharding of the 3D face-block solve across ranks.

The reference is serial; BASELINE.json config 5 shards "faces by z-slab
across the GPUs, with face-halo exchange and FGMRES dot-product allreduce".
This module is that path:

* partition — elements by z-layer slab (64/P layers each), every face owned
  by the slab of its first-seen (`left`) element. First-seen numbering walks
  the elements layer by layer, so every rank owns one contiguous face range.
* local operators — a rank keeps the block rows of its owned faces; its block
  columns are the faces of the elements touching them: ghost faces of the
  slab below, its own, ghost faces of the slab above — numbered so that local
  column order equals global column order, hence every owned row folds its
  entries in the reference's order (csr.hpp:68-74) and a sharded SpMV equals
  the single-GPU one bit for bit. Block-Jacobi (face blocks) and the p-level
  inheritance are per face, i.e. local.
* exchange — before every operator application the ghost face values are
  received from the two neighbour slabs (point-to-point; NCCL on the GPU,
  gloo on the CPU); Krylov dot products are local partial sums combined by an
  allreduce.
* coarse level — replicated: the owned coarse defects are
  all-gathered and every rank runs the reference's coarse ILU-GMRES on the
  full coarse operator, so the coarse solve is partition-independent.

The orchestration (FGMRES(30) over V-cycles of block-Jacobi-preconditioned
GMRES(s) smoothing, plevels.hpp:170-197, gmres.hpp:38-173) is written once
over a small `ops` interface with two backends: `GpuOps` (the sm_100a
kernels through the C ABI on device tensors) and `CpuOps` (numpy / the
oracle; test infrastructure for the multi-process CPU tests). Differences
from the single-GPU solver: dot products are sums of per-rank partials
(rounding-level differences, so iteration counts agree and histories match
to ~1e-9 rather than bitwise).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------

@dataclass
class RankView:
    rank: int
    nranks: int
    f0: int                  # owned faces [f0, f1)
    f1: int
    faces: np.ndarray        # local block columns (global face ids, ascending)
    nbelow: int              # ghost faces below (local ids [0, nbelow))
    elements: np.ndarray     # elements touching an owned face
    brow_ptr: np.ndarray     # local block pattern: owned rows, local columns
    bcols: np.ndarray
    send_down: np.ndarray    # owned faces the rank below holds as ghosts (local owned idx)
    send_up: np.ndarray      # owned faces the rank above holds as ghosts
    recv_down: int           # ghost faces received from the rank below
    recv_up: int

    @property
    def nown(self) -> int:
        return self.f1 - self.f0

    @property
    def ncols(self) -> int:
        return len(self.faces)


class SlabPartition:
    """z-slab partition of a Mesh3 over `nranks` ranks."""

    def __init__(self, mesh, nranks: int):
        n = mesh.n
        if nranks < 1 or nranks > n:
            raise ValueError("z-slab partition: 1 <= ranks <= layers")
        self.mesh = mesh
        self.nranks = nranks
        f = mesh.faces()
        self.ef = mesh.element_faces()
        layer = np.arange(mesh.n_elements) // (n * n)
        self.erank = layer * nranks // n
        self.frank = self.erank[f[:, 4]]
        if np.any(np.diff(self.frank) < 0):
            raise RuntimeError("z-slab partition: owned faces are not contiguous")
        self.starts = np.searchsorted(self.frank, np.arange(nranks + 1))
        self.starts[-1] = mesh.n_faces
        self.brp, self.bcols = mesh.block_pattern()

    def view(self, r: int) -> RankView:
        f0, f1 = int(self.starts[r]), int(self.starts[r + 1])
        touch = np.any((self.ef >= f0) & (self.ef < f1), axis=1)
        elements = np.nonzero(touch)[0]
        faces = np.unique(self.ef[elements])
        nbelow = int(np.searchsorted(faces, f0))
        rows = np.arange(f0, f1)
        brp = np.zeros(len(rows) + 1, np.int64)
        brp[1:] = np.cumsum(self.brp[rows + 1] - self.brp[rows])
        gcols = np.concatenate([self.bcols[self.brp[g]:self.brp[g + 1]] for g in rows])
        bcols = np.searchsorted(faces, gcols).astype(np.int32)
        assert np.array_equal(faces[bcols], gcols)

        def ghosts_of(q):
            if q < 0 or q >= self.nranks:
                return np.zeros(0, np.int64)
            g0, g1 = int(self.starts[q]), int(self.starts[q + 1])
            e = np.nonzero(np.any((self.ef >= g0) & (self.ef < g1), axis=1))[0]
            return np.unique(self.ef[e])

        below, above = ghosts_of(r - 1), ghosts_of(r + 1)
        send_down = below[(below >= f0) & (below < f1)] - f0
        send_up = above[(above >= f0) & (above < f1)] - f0
        return RankView(r, self.nranks, f0, f1, faces, nbelow, elements, brp, bcols,
                        send_down.astype(np.int64), send_up.astype(np.int64), nbelow,
                        len(faces) - nbelow - (f1 - f0))


# ---------------------------------------------------------------------------
# distributed Krylov over an ops backend
# ---------------------------------------------------------------------------

class Dist:
    """Collectives for the solver: ghost exchange and sums of partials."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group

    def allreduce(self, v: float) -> float:
        if self.dist is None or self.dist.get_world_size() == 1:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    device = "cpu"


class ZSlabSolver:
    """FGMRES(restart) preconditioned by one p-multigrid V-cycle per
    iteration (plevels.hpp:170-239) on a z-slab sharded face-block system."""

    def __init__(self, ops, dist: Dist, levels: int, smoother_iters: int = 2,
                 coarse_rtol: float = 1e-3, coarse_maxit: int = 400):
        self.ops = ops
        self.d = dist
        self.nlev = levels
        self.s = smoother_iters
        self.coarse_rtol = coarse_rtol
        self.coarse_maxit = coarse_maxit
        self.coarse_its = 0
        self.vcycles = 0

    # distributed vector algebra (owned parts)
    def dot(self, a, b) -> float:
        return self.d.allreduce(self.ops.dot(a, b))

    def norm(self, a) -> float:
        return math.sqrt(self.dot(a, a))

    def _arnoldi(self, j, w, V, H, cs, sn, g):
        for i in range(j + 1):
            H[i, j] = self.dot(w, V[i])
            w = w - H[i, j] * V[i]
        H[j + 1, j] = self.norm(w)
        sub = H[j + 1, j]
        V.append(w / H[j + 1, j] if H[j + 1, j] > 0.0 else w * 0.0)
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        den = math.hypot(H[j, j], H[j + 1, j])
        cs[j] = 1.0 if den == 0.0 else H[j, j] / den
        sn[j] = 0.0 if den == 0.0 else H[j + 1, j] / den
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        return abs(g[j + 1]), sub

    @staticmethod
    def _solve_y(H, g, m):
        y = np.zeros(m)
        for i in range(m - 1, -1, -1):
            s = g[i]
            for q in range(i + 1, m):
                s = s - H[i, q] * y[q]
            y[i] = s / H[i, i]
        return y

    def gmres_left(self, l, rhs, x0, its):
        """gmres(A_l, BJ_l, rhs, x0, its, rtol 0, Left) (gmres.hpp:103-139)."""
        op = self.ops

        def a(x):
            return op.bj(l, op.spmv(l, x))
        prhs = op.bj(l, rhs)
        r0 = prhs - (a(x0) if x0 is not None else op.zeros_like(prhs))
        beta = self.norm(r0)
        if beta == 0.0:
            return x0 if x0 is not None else op.zeros_like(prhs)
        V, Z = [r0 / beta], []
        H = np.zeros((its + 1, its))
        cs, sn, g = np.zeros(its), np.zeros(its), np.zeros(its + 1)
        g[0] = beta
        m = 0
        for j in range(its):
            Z.append(V[j])
            est, sub = self._arnoldi(j, a(Z[j]), V, H, cs, sn, g)
            m = j + 1
            if sub == 0.0:
                break
        y = self._solve_y(H, g, m)
        x = x0.clone() if hasattr(x0, "clone") else (x0.copy() if x0 is not None
                                                      else op.zeros_like(prhs))
        for i in range(m):
            x = x + y[i] * Z[i]
        return x

    def vcycle(self, l, d):
        op = self.ops
        if l + 1 == self.nlev:
            x, its = op.coarse_solve(d, self.coarse_rtol, self.coarse_maxit)
            self.coarse_its += its
            return x
        w = self.gmres_left(l, d, None, self.s)
        dc = op.resid_restrict(l, d, w)
        c = self.vcycle(l + 1, dc)
        w = op.prolong_add(l, w, c)
        return self.gmres_left(l, d, w, self.s)

    def solve(self, rhs, rtol=1e-8, maxit=1000, restart=30):
        """FGMRES(restart) with the fgmres_hist control flow of the oracle
        (gmres.hpp:145-173 plus restarts); returns (x, hist, its, converged)."""
        op = self.ops
        bnorm = self.norm(rhs)
        hist = []
        x0 = op.zeros_like(rhs)
        cycle = restart if restart > 0 else maxit
        total = 0
        r0, beta = rhs, bnorm
        self.coarse_its = self.vcycles = 0
        while True:
            mm = min(cycle, maxit - total)
            V, Z = [r0 / beta], []
            H = np.zeros((mm + 1, mm))
            cs, sn, g = np.zeros(mm), np.zeros(mm), np.zeros(mm + 1)
            g[0] = beta
            restart_now = False
            x = None
            for j in range(mm):
                Z.append(self.vcycle(0, V[j]))
                self.vcycles += 1
                est, sub = self._arnoldi(j, op.spmv(0, Z[j]), V, H, cs, sn, g)
                total += 1
                hist.append(est / bnorm)
                m = j + 1
                last = total == maxit
                if est <= rtol * bnorm or sub == 0.0 or last:
                    y = self._solve_y(H, g, m)
                    x = x0
                    for i in range(m):
                        x = x + y[i] * Z[i]
                    rel = self.norm(rhs - op.spmv(0, x)) / bnorm
                    if rel <= rtol:
                        return x, np.array(hist), total, True
                    if last:
                        return x, np.array(hist), total, False
                    if j + 1 == mm:
                        restart_now = True
                        x0 = x
                elif j + 1 == mm:
                    restart_now = True
                    y = self._solve_y(H, g, m)
                    x = x0
                    for i in range(m):
                        x = x + y[i] * Z[i]
                    x0 = x
            if not restart_now:
                return x, np.array(hist), total, False
            r0 = rhs - op.spmv(0, x0)
            beta = self.norm(r0)


# ---------------------------------------------------------------------------
# CPU backend (numpy + the oracle): multi-process tests of the sharded path
# ---------------------------------------------------------------------------

class CpuOps:
    """Sharded level operators on the CPU: the rank's block rows expanded to
    CSR with local columns (row folds in the reference's order through the
    oracle's po_csr_multiply), block-Jacobi by explicit face-block inverses,
    the replicated coarse solve with the reference's own gmres + Ilu0."""

    def __init__(self, view: RankView, levels, group=None):
        """levels: list of dicts per level l with keys bs (block size), vals
        (local block values, column-major blocks, owned rows), in_block
        (coarse-within-fine block map to level l+1), and for the coarsest the
        full coarse CSR in 'coarse_csr' (replicated)."""
        import oracle_ref as O
        import torch.distributed as dist

        self.O = O
        self.v = view
        self.levels = levels
        self.group = group
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        import ctypes as C

        self._csr, self._bj = [], []
        for L in levels[:-1]:
            bs = L["bs"]
            # columns bs * local column + c: the [below | own | above] layout
            rp, cols = O.bsr_to_csr_pattern(view.brow_ptr, view.bcols, bs)
            vals = _bsr_vals_to_csr(L["vals"], view.brow_ptr, bs)
            self._csr.append(O.Csr(rp, cols, vals))
            # the oracle's block-Jacobi (po_bj_factor, same LU + inverse as the
            # device) on the owned rows, columns shifted to the owned range
            shifted = O.Csr(rp, (cols.astype(np.int64) - view.nbelow * bs).astype(np.int32), vals)
            lay = O.PoLayout(1, 2, 0, view.nown, 0, 0, bs, 0, 0, 3)
            inv = np.zeros(O.port_lib().po_bj_size(C.byref(lay)))
            bad = C.c_int64(-1)
            if O.port_lib().po_bj_factor(C.byref(O.po_csr(shifted)), C.byref(lay), inv, C.byref(bad)):
                raise RuntimeError(f"block-Jacobi: singular block {bad.value}")
            self._bj.append((lay, inv))
        cc = levels[-1]["coarse_csr"]
        self._coarse = O.RefCsr(cc)
        self._coarse_ilu = O.RefIlu(self._coarse)

    # vector helpers
    @staticmethod
    def zeros_like(a):
        return np.zeros_like(a)

    @staticmethod
    def dot(a, b) -> float:
        return float(np.dot(a, b))

    def _exchange(self, l, x_own):
        v, bs = self.v, self.levels[l]["bs"]
        below = np.zeros(v.recv_down * bs)
        above = np.zeros(v.recv_up * bs)
        if self.dist is not None and v.nranks > 1:
            import torch

            reqs = []
            xo = x_own.reshape(-1, bs)
            if v.rank > 0:
                reqs.append(self.dist.isend(torch.from_numpy(np.ascontiguousarray(
                    xo[v.send_down].ravel())), v.rank - 1, group=self.group))
                tb = torch.zeros(v.recv_down * bs, dtype=torch.float64)
                reqs.append(self.dist.irecv(tb, v.rank - 1, group=self.group))
            if v.rank + 1 < v.nranks:
                reqs.append(self.dist.isend(torch.from_numpy(np.ascontiguousarray(
                    xo[v.send_up].ravel())), v.rank + 1, group=self.group))
                ta = torch.zeros(v.recv_up * bs, dtype=torch.float64)
                reqs.append(self.dist.irecv(ta, v.rank + 1, group=self.group))
            for q in reqs:
                q.wait()
            if v.rank > 0:
                below = tb.numpy()
            if v.rank + 1 < v.nranks:
                above = ta.numpy()
        return np.concatenate([below, x_own, above])

    def spmv(self, l, x_own):
        import ctypes as C

        ext = self._exchange(l, np.ascontiguousarray(x_own, np.float64))
        a = self._csr[l]
        y = np.zeros(a.n)
        self.O.port_lib().po_csr_multiply(C.byref(self.O.po_csr(a)), ext, y)
        return y

    def bj(self, l, x_own):
        import ctypes as C

        lay, inv = self._bj[l]
        y = np.zeros(len(x_own))
        self.O.port_lib().po_bj_apply(C.byref(lay), inv, np.ascontiguousarray(x_own, np.float64), y)
        return y

    def resid_restrict(self, l, d, w):
        r = d - self.spmv(l, w)
        m = self.levels[l]["in_block"]
        return r.reshape(-1, self.levels[l]["bs"])[:, m].ravel()

    def prolong_add(self, l, w, c):
        m = self.levels[l]["in_block"]
        out = w.reshape(-1, self.levels[l]["bs"]).copy()
        out[:, m] = out[:, m] + c.reshape(len(out), -1)
        return out.ravel()

    def coarse_solve(self, d_own, rtol, maxit):
        full = _allgather(self.dist, self.group, d_own, self.v.nranks)
        r = self.O.ref_gmres(self._coarse, self._coarse_ilu, full, np.zeros(len(full)), maxit,
                             rtol, left=False)
        bs = self.levels[-1]["bs"]
        return r["x"][self.v.f0 * bs:self.v.f1 * bs].copy(), r["its"]


def _allgather(dist, group, own, nranks):
    if dist is None or nranks == 1:
        return np.ascontiguousarray(own)
    import torch

    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(nranks)]
    dist.all_gather(sizes, torch.tensor([len(own)], dtype=torch.int64), group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    t = torch.zeros(mx, dtype=torch.float64)  # equal-size buffers (gloo / NCCL all_gather)
    t[:len(own)] = torch.from_numpy(np.ascontiguousarray(own))
    parts = [torch.zeros(mx, dtype=torch.float64) for _ in range(nranks)]
    dist.all_gather(parts, t, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)]).numpy()


def _bsr_vals_to_csr(vals, brow_ptr, bs):
    """Column-major block values -> CSR values of the dense expansion (row
    f bs + r: blocks ascending, columns within a block ascending)."""
    nb = len(brow_ptr) - 1
    out = []
    v = np.asarray(vals)
    for f in range(nb):
        q0, q1 = int(brow_ptr[f]), int(brow_ptr[f + 1])
        blk = v[q0 * bs * bs:q1 * bs * bs].reshape(q1 - q0, bs, bs)  # [q, c, r]
        out.append(np.transpose(blk, (2, 0, 1)).ravel())  # [r, q, c]
    return np.concatenate(out)



# ---------------------------------------------------------------------------
# GPU backend: the sm_100a kernels through the C ABI on device tensors
# ---------------------------------------------------------------------------

class GpuOps:
    """Sharded level operators on the GPU: rank-local face-block operators
    (pscu_bsr_create_local / pscu_assembly_*_local: owned block rows, ghost
    block columns), inherited per level with pscu_inherit, block-Jacobi by
    pscu_bj_*, SpMV by the bitwise face-block kernel; the replicated coarse
    ILU-GMRES by pscu_gmres on the gathered coarse operator. Vectors are
    float64 CUDA tensors; ghost exchange and gathers go through
    torch.distributed (NCCL)."""

    def __init__(self, view: RankView, fine, k: int, partition: SlabPartition, ctx, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _native as N
        from . import solver as S

        self.C, self.N, self.S, self.torch = C, N, S, torch
        self.v, self.ctx, self.group = view, ctx, group
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.dev = torch.device("cuda", torch.cuda.current_device())
        lib = ctx.lib
        self.mats, self.bjs, self.bs, self.in_block = [fine], [], [], []
        lay = S.make_layout3(k, view.nown, 0)
        layouts = [lay]
        for kc in range(k - 1, -1, -1):
            lc = S.make_layout3(kc, view.nown, 0)
            self.mats.append(S.inherit_matrix(self.mats[-1], layouts[-1], lc))
            c2f = S.coarse_to_fine_map(layouts[-1], lc)
            fbc = 3 * lc.face_vel + lc.face_press
            self.in_block.append(torch.as_tensor(c2f[:fbc], device=self.dev))
            layouts.append(lc)
        for l, L in enumerate(layouts):
            self.bs.append(3 * L.face_vel + L.face_press)
            if l + 1 < len(layouts):
                self.bjs.append(S.BlockJacobi(self.mats[l], L))
        # replicated coarse operator: gather the owned coarse block rows
        bsc = self.bs[-1]
        _, _, own_vals = self.mats[-1].download_blocks()
        full = _allgather(self.dist, group, own_vals, view.nranks) if self.dist is None else \
            self._gather_dev(torch.as_tensor(own_vals, device=self.dev)).cpu().numpy()
        self.coarse = S.bsr_matrix(partition.brp, partition.bcols, full, bsc, ctx=ctx)
        self.coarse_ilu = S.Ilu0(self.coarse)
        self.lib = lib

    # vector helpers
    def zeros_like(self, a):
        return self.torch.zeros_like(a)

    @staticmethod
    def dot(a, b) -> float:
        return float((a * b).sum().item())

    def _sync(self):
        self.torch.cuda.current_stream().synchronize()

    def _gather_dev(self, own):
        torch = self.torch
        if self.dist is None or self.v.nranks == 1:
            return own
        n = torch.tensor([own.numel()], device=self.dev)
        sizes = [torch.zeros_like(n) for _ in range(self.v.nranks)]
        self.dist.all_gather(sizes, n, group=self.group)
        mx = int(max(int(s.item()) for s in sizes))
        buf = torch.zeros(mx, dtype=own.dtype, device=self.dev)
        buf[:own.numel()] = own
        parts = [torch.zeros_like(buf) for _ in range(self.v.nranks)]
        self.dist.all_gather(parts, buf, group=self.group)
        return torch.cat([p[:int(s.item())] for p, s in zip(parts, sizes)])

    def _exchange(self, l, x_own):
        torch, v, bs = self.torch, self.v, self.bs[l]
        below = torch.zeros(v.recv_down * bs, dtype=x_own.dtype, device=self.dev)
        above = torch.zeros(v.recv_up * bs, dtype=x_own.dtype, device=self.dev)
        if self.dist is not None and v.nranks > 1:
            xo = x_own.view(-1, bs)
            ops = []
            if v.rank > 0:
                ops.append(self.dist.P2POp(self.dist.isend, xo[torch.as_tensor(
                    v.send_down, device=self.dev)].reshape(-1).contiguous(), v.rank - 1,
                    group=self.group))
                ops.append(self.dist.P2POp(self.dist.irecv, below, v.rank - 1, group=self.group))
            if v.rank + 1 < v.nranks:
                ops.append(self.dist.P2POp(self.dist.isend, xo[torch.as_tensor(
                    v.send_up, device=self.dev)].reshape(-1).contiguous(), v.rank + 1,
                    group=self.group))
                ops.append(self.dist.P2POp(self.dist.irecv, above, v.rank + 1, group=self.group))
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        return torch.cat([below, x_own, above])

    def spmv(self, l, x_own):
        ext = self._exchange(l, x_own.contiguous())
        y = self.torch.empty(self.mats[l].n, dtype=ext.dtype, device=self.dev)
        self._sync()
        self.N.check(self.lib.pscu_spmv(self.ctx.h, self.mats[l].h, self.N.ptr(ext),
                                        self.N.ptr(y), self.N.PSCU_DEVICE))
        return y

    def bj(self, l, x_own):
        x = x_own.contiguous()
        y = self.torch.empty_like(x)
        self._sync()
        self.N.check(self.lib.pscu_bj_apply(self.ctx.h, self.bjs[l].h, self.N.ptr(x), self.N.ptr(y),
                                            self.N.PSCU_DEVICE))
        return y

    def resid_restrict(self, l, d, w):
        r = d - self.spmv(l, w)
        return r.view(-1, self.bs[l])[:, self.in_block[l]].reshape(-1)

    def prolong_add(self, l, w, c):
        out = w.view(-1, self.bs[l]).clone()
        out[:, self.in_block[l]] = out[:, self.in_block[l]] + c.view(out.shape[0], -1)
        return out.reshape(-1)

    def coarse_solve(self, d_own, rtol, maxit):
        C, N = self.C, self.N
        full = self._gather_dev(d_own.contiguous())
        x = self.torch.zeros_like(full)
        its, rel, conv = C.c_int(), C.c_double(), C.c_int()
        self._sync()
        N.check(self.lib.pscu_gmres(self.ctx.h, self.coarse.h, self.coarse_ilu.h, N.ptr(full), None,
                                    maxit, rtol, 0, N.ptr(x), C.byref(its), C.byref(rel),
                                    C.byref(conv), N.PSCU_DEVICE))
        bs = self.bs[-1]
        return x[self.v.f0 * bs:self.v.f1 * bs].clone(), its.value


def assemble_local(mesh, view: RankView, k: int, data: str = "random", seed: int = 0,
                   batch: int = 4096, ctx=None):
    """The rank's shard of assemble_hho (3D HHO-hp vp-cond): local blocks of
    the elements touching an owned face, condensed on the device and scattered
    into the owned block rows (ghost block columns kept); returns the shard
    operator and its owned reduced load."""
    import ctypes as C

    from . import _native as N
    from . import host
    from . import solver as S

    ctx = ctx or S.default_context()
    L = host.HpLocal3(k)
    h = C.c_void_p()
    N.check(ctx.lib.pscu_assembly_begin_local(ctx.h, view.nown, view.ncols, L.face_block,
                                              view.nbelow, view.brow_ptr.ctypes.data,
                                              view.bcols.ctypes.data, C.byref(h)))
    A = S.CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
    A._owned = True
    ef = mesh.element_faces()
    keep_pos = np.ascontiguousarray(L.keep_pos, np.int32)
    n = L.n_local
    els = view.elements
    for b0 in range(0, len(els), batch):
        sel = els[b0:b0 + batch]
        mats = np.empty(len(sel) * n * n)
        rhs = np.empty(len(sel) * n)
        # build the selected elements, one producer call per run of ids
        off = 0
        runs = np.split(sel, np.nonzero(np.diff(sel) != 1)[0] + 1)
        for run in runs:
            e0, e1 = int(run[0]), int(run[-1]) + 1
            m_ = mats[off * n * n:(off + e1 - e0) * n * n]
            r_ = rhs[off * n:(off + e1 - e0) * n]
            L.local_blocks(mesh, e0, e1, data=data, seed=seed, out=(m_, r_))
            off += e1 - e0
        cols = np.searchsorted(view.faces, ef[sel]).astype(np.int32)
        rows = np.where((ef[sel] >= view.f0) & (ef[sel] < view.f1), ef[sel] - view.f0, -1)
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        N.check(ctx.lib.pscu_assembly_add_local(ctx.h, A.h, int(sel[0]), len(sel), n,
                                                mats.ctypes.data, rhs.ctypes.data, L.n_elim,
                                                L.elim.ctypes.data, rows.ctypes.data,
                                                cols.ctypes.data, 6, keep_pos.ctypes.data,
                                                N.PSCU_HOST))
    b = np.zeros(A.n)
    N.check(ctx.lib.pscu_assembly_rhs(ctx.h, A.h, b.ctypes.data, N.PSCU_HOST))
    return A, b
