"""GPU side of the z-slab sharding (paper_2009_13840_b200/zslab.py, SURVEY.md
§8(e)) on one device: the shard-local device assembly of every rank of a
2- and 3-way partition equals the owned rows of the global device assembly
bit for bit; the sharded face-block SpMV of every shard, fed the ghost
values, equals the global SpMV bit for bit; and the sharded FGMRES/V-cycle
driver on the device (GpuOps, one rank) matches the unsharded device solver
(iteration counts equal, solution within 1e-9; the multi-process exchange
itself is covered on the CPU by tests/test_zslab.py)."""
import numpy as np
import pytest

import oracle_ref as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.port_available(),
                                                  reason="oracle restatement not built")]


@pytest.fixture(scope="module")
def M():
    from paper_2009_13840_b200 import build, host, solver, zslab
    build.build_host()
    mesh = host.Mesh3(6, jitter=0.1, seed=4)
    A, b, lay, info = host.assemble_stokes3(mesh, 2, data="random", seed=5)
    return host, solver, zslab, mesh, A, b, lay


@pytest.mark.parametrize("P", [2, 3])
def test_shard_assembly_and_spmv_bitwise(M, P):
    host, S, z, mesh, A, b, lay = M
    brp, bcols, vals = A.download_blocks()
    part = z.SlabPartition(mesh, P)
    x = np.random.default_rng(2).standard_normal(A.n)
    y = A.multiply(x)
    for r in range(P):
        v = part.view(r)
        Al, bl = z.assemble_local(mesh, v, 2, data="random", seed=5)
        _, _, lv = Al.download_blocks()
        q0, q1 = int(brp[v.f0]), int(brp[v.f1])
        assert lv.tobytes() == vals[q0 * 576:q1 * 576].tobytes()
        assert bl.tobytes() == b[v.f0 * 24:v.f1 * 24].tobytes()
        ext = x.reshape(-1, 24)[v.faces].ravel()
        assert Al.multiply(ext).tobytes() == y[v.f0 * 24:v.f1 * 24].tobytes()


def test_sharded_driver_matches_device_solver(M):
    import torch

    host, S, z, mesh, A, b, lay = M
    part = z.SlabPartition(mesh, 1)
    v = part.view(0)
    Al, bl = z.assemble_local(mesh, v, 2, data="random", seed=5)
    ops = z.GpuOps(v, Al, 2, part, S.default_context())
    solver = z.ZSlabSolver(ops, z.Dist(), 3, smoother_iters=2)
    x, hist, its, conv = solver.solve(torch.as_tensor(bl, device="cuda"), rtol=1e-8, maxit=200,
                                      restart=30)
    cfg = S.LevelConfig(degrees=[2, 1, 0], smoother="bjacobi", smoother_iters=2,
                        coarse="gmres-ilu", outer_rtol=1e-8, restart=30)
    xr, hr, rep = S.LevelHierarchy(A, lay, cfg).solve(b)
    assert conv and rep.converged and its == rep.outer_its
    x = x.cpu().numpy()
    assert np.max(np.abs(x - xr)) <= 1e-9 * np.max(np.abs(xr))
    assert np.all(np.abs(hist - hr) <= 1e-9 * np.abs(hr))
