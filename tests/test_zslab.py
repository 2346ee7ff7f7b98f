"""z-slab sharded solve (paper_2009_13840_b200/zslab.py) on
the CPU with gloo at world size 2 against world size 1 and the oracle's
unsharded solve: the partition (contiguous owned faces, ghost and send
lists), the sharded operator (owned rows equal to the global rows bit for
bit through the ghost exchange), and the whole FGMRES(30) / V-cycle solve
(iteration counts equal; history and solution to 1e-9 relative, the dot
products being sums of per-rank partials)."""
import os
import socket

import numpy as np
import pytest

import oracle_ref as O

pytestmark = pytest.mark.skipif(not O.port_available(), reason="oracle restatement not built")

N = 4  # 4 z-layers: 2 per rank


def _system():
    from paper_2009_13840_b200 import build, host
    build.build_host()
    m = host.Mesh3(N, jitter=0.1, seed=4)
    L = host.HpLocal3(2)
    mats, rhs = L.local_blocks(m, 0, m.n_elements, data="random", seed=5)
    brp, bcols = m.block_pattern()
    rp, cols = O.bsr_to_csr_pattern(brp, bcols, L.face_block)
    lay = O.po_layout(1, 2, 2, m.n_faces, m.n_elements, dim=3)
    a, b = O.port_condense_assemble(mats, rhs, L.n_local, L.elim, L.kept_global(m.element_faces()),
                                    lay, rp, cols)
    return m, a, b, lay, brp, bcols


def _levels(view, hier, brp, bcols):
    """Per-level rank-local block values (owned rows) from the oracle's
    inherited level operators, and the replicated coarse CSR."""
    from paper_2009_13840_b200.solver import csr_to_bsr_values
    out = []
    for l, bs in enumerate((24, 12, 4)):
        csr = hier.level_csr(l)
        if l == 2:
            out.append(dict(bs=bs, coarse_csr=csr))
            continue
        bv = csr_to_bsr_values(csr.row_ptr, csr.cols, csr.vals, brp, bcols, bs)
        q0, q1 = int(brp[view.f0]), int(brp[view.f1])
        nbc = (12, 4)[l]
        # coarse dofs of a face block: the leading modes of each component
        fvf, fvc = {24: 6, 12: 3}[bs], {12: 3, 4: 1}[nbc]
        in_block = np.concatenate([np.arange(c * fvf, c * fvf + fvc) for c in range(4)])
        out.append(dict(bs=bs, vals=bv[q0 * bs * bs:q1 * bs * bs], in_block=in_block))
    return out


def _solve(rank, nranks, port, result):
    import torch.distributed as dist

    from paper_2009_13840_b200 import zslab
    if nranks > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=nranks)
    m, a, b, lay, brp, bcols = _system()
    hier = O.PortHierarchy(a, lay, [2, 1, 0], smoother_iters=2, smoother=1)
    part = zslab.SlabPartition(m, nranks)
    v = part.view(rank)
    ops = zslab.CpuOps(v, _levels(v, hier, brp, bcols))
    solver = zslab.ZSlabSolver(ops, zslab.Dist(), 3, smoother_iters=2)
    bo = b[v.f0 * 24:v.f1 * 24]
    # sharded operator rows == global rows (bitwise)
    xg = np.random.default_rng(1).standard_normal(a.n)
    y = ops.spmv(0, xg[v.f0 * 24:v.f1 * 24])
    x, hist, its, conv = solver.solve(bo, rtol=1e-8, maxit=200, restart=30)
    out = dict(rank=rank, y=y, x=x, hist=hist, its=its, conv=conv, coarse_its=solver.coarse_its,
               f0=v.f0, f1=v.f1)
    if nranks > 1:
        gathered = [None] * nranks
        dist.all_gather_object(gathered, out)
        dist.destroy_process_group()
        if rank == 0:
            result.put(gathered)
    else:
        result.put([out])


def _run(nranks):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_solve, args=(r, nranks, port, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    return res


def test_partition_views():
    from paper_2009_13840_b200 import build, host, zslab
    build.build_host()
    m = host.Mesh3(6, jitter=0.1, seed=4)
    for P in (1, 2, 3):
        part = zslab.SlabPartition(m, P)
        views = [part.view(r) for r in range(P)]
        assert views[0].f0 == 0 and views[-1].f1 == m.n_faces
        for r in range(P - 1):
            assert views[r].f1 == views[r + 1].f0
            # what r sends up is exactly what r+1 holds as ghosts below
            assert views[r].send_up.size == views[r + 1].recv_down
            up = views[r].f0 + views[r].send_up
            assert np.array_equal(up, views[r + 1].faces[:views[r + 1].nbelow])
            down = views[r + 1].f0 + views[r + 1].send_down
            lo = views[r].nbelow + views[r].nown
            assert np.array_equal(down, views[r].faces[lo:])


def test_sharded_solve_matches_unsharded():
    one = _run(1)[0]
    two = _run(2)
    m, a, b, lay, brp, bcols = _system()
    ref = O.PortHierarchy(a, lay, [2, 1, 0], smoother_iters=2, smoother=1).solve(
        b, rtol=1e-8, maxit=200, restart=30)
    # operator rows bitwise
    y2 = np.concatenate([r["y"] for r in two])
    assert y2.tobytes() == one["y"].tobytes()
    import ctypes as C
    xg = np.random.default_rng(1).standard_normal(a.n)
    yg = np.zeros(a.n)
    O.port_lib().po_csr_multiply(C.byref(O.po_csr(a)), xg, yg)
    assert one["y"].tobytes() == yg.tobytes()
    # the solve: ITs equal (sharded, unsharded, oracle), solution / history 1e-9
    assert one["conv"] and all(r["conv"] for r in two) and ref["converged"]
    assert one["its"] == two[0]["its"] == ref["its"]
    x2 = np.concatenate([r["x"] for r in two])
    scale = np.max(np.abs(ref["x"]))
    assert np.max(np.abs(x2 - ref["x"])) <= 1e-9 * scale
    assert np.max(np.abs(one["x"] - ref["x"])) <= 1e-9 * scale
    assert np.all(np.abs(two[0]["hist"] - ref["hist"]) <= 1e-9 * np.abs(ref["hist"]))
