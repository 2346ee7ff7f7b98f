"""Device 3D local element blocks: pscu_local_blocks3
(repo:paper_2009_13840_b200/csrc/local3.cu) against the host producer's
psh3_local_blocks (the 3D HHO-hp build_local), bit for bit — every matrix
entry and load of every element, for jittered meshes, k = 0..2, zero and
random-modal data — and the streamed assembly from device-built blocks
equal to the host-built one."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_2009_13840_b200 import build, host
    build.build_host()
    return host


@pytest.mark.parametrize("n,jit,k,data", [(2, 0.0, 2, "random"), (3, 0.15, 2, "random"),
                                          (3, 0.15, 1, "zero"), (2, 0.2, 0, "random"),
                                          (4, 0.1, 2, "zero")])
def test_local_blocks_bitwise(H, n, jit, k, data):
    mesh = H.Mesh3(n, jitter=jit, seed=4)
    L = H.HpLocal3(k)
    e0, e1 = 0, mesh.n_elements
    want_m, want_r = L.local_blocks(mesh, e0, e1, data=data, seed=5)
    got_m, got_r = H.local_blocks3_device(mesh, k, e0, e1, data=data, seed=5)
    assert got_r.tobytes() == want_r.tobytes()
    bad = np.nonzero(got_m != want_m)[0]
    assert got_m.tobytes() == want_m.tobytes(), (len(bad), bad[:10] % (L.n_local ** 2))


def test_local_blocks_batch_offset(H):
    mesh = H.Mesh3(3, jitter=0.1, seed=2)
    L = H.HpLocal3(2)
    want_m, want_r = L.local_blocks(mesh, 5, 17, data="random", seed=9)
    got_m, got_r = H.local_blocks3_device(mesh, 2, 5, 17, data="random", seed=9)
    assert got_m.tobytes() == want_m.tobytes() and got_r.tobytes() == want_r.tobytes()


def test_local_blocks_device_rejects_closed_form_data(H):
    mesh = H.Mesh3(2)
    with pytest.raises(ValueError, match="data kinds"):
        H.local_blocks3_device(mesh, 2, 0, 2, data="manufactured")


@pytest.mark.parametrize("recovery", [False, True])
def test_streamed_assembly_device_producer_bitwise(H, recovery):
    """assemble_stokes3 with the blocks built on the device equals the
    host-producer assembly: face-block values, rhs and recovery data."""
    mesh = H.Mesh3(4, jitter=0.1, seed=3)
    Ad, bd, _, infod = H.assemble_stokes3(mesh, 2, data="random", seed=7, batch=13,
                                          producer="device", recovery=recovery)
    Ah, bh, _, infoh = H.assemble_stokes3(mesh, 2, data="random", seed=7, batch=13,
                                          producer="host", recovery=recovery)
    assert infod["producer"] == "device"
    assert Ad.download_blocks()[2].tobytes() == Ah.download_blocks()[2].tobytes()
    assert bd.tobytes() == bh.tobytes()
    if recovery:
        assert infod["elim_coupling"].tobytes() == infoh["elim_coupling"].tobytes()
        assert infod["elim_rhs"].tobytes() == infoh["elim_rhs"].tobytes()
