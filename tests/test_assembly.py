"""SEM assembly -- direct-stiffness summation Q Q^T and its halo exchange
(paper_1503_07659_b200/assembly.py, csrc/dssum.cu).

Not a reference entry point (the reference operator is element-local), so
parity is pinned to a plain-Python restatement of the definition (every
global node's copies summed left to right in ascending element order, the
sum written back to every copy), which the C oracle (lfo_dssum_f64) must
match bitwise, and to the properties of Q Q^T.  CPU: the oracle and the
multi-rank protocol (gloo, 2-4 ranks, oracle-backed local kernels) -- bitwise
the single-domain result.  GPU: the device kernel vs the oracle, the
protocol with the device kernels on 2 ranks, and the assembled operator."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import REPO
from paper_1503_07659_b200.assembly import BoxMesh, dssum_sharded

MESHES = [(2, 3, 2, 4), (3, 1, 2, 5), (1, 1, 3, 2), (2, 2, 2, 8),
          (1, 2, 1, 3)]


def restated_dssum(w, mesh):
    """Definition of Q Q^T, in Python: global node of (e, i, j, k) is
    (ex p + i, ey p + j, ez p + k); copies summed in ascending e."""
    n, p = mesh.n, mesh.p
    groups = {}
    for e in range(mesh.nelt):
        ex, r = e % mesh.ex, e // mesh.ex
        ey, ez = r % mesh.ey, r // mesh.ey
        for k in range(n):
            for j in range(n):
                for i in range(n):
                    g = (ex * p + i, ey * p + j, ez * p + k)
                    groups.setdefault(g, []).append(
                        (e, i + n * j + n * n * k + n ** 3 * e))
    out = w.copy()
    for copies in groups.values():
        copies.sort()
        s = w[copies[0][1]]
        for _e, q in copies[1:]:
            s = s + w[q]
        for _e, q in copies:
            out[q] = s
    return out


def _field(mesh, seed):
    return np.random.default_rng(seed).random(mesh.nelt * mesh.n ** 3) * 2 - 1


@pytest.mark.parametrize("mesh", MESHES)
def test_oracle_is_the_definition(mesh):
    mesh = BoxMesh(*mesh)
    w = _field(mesh, 1)
    want = restated_dssum(w, mesh)
    got = oracle.dssum(w.copy(), mesh.n, mesh.ex, mesh.ey, mesh.ez)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("mesh", MESHES)
def test_qqt_properties(mesh):
    """Q Q^T 1 = multiplicity; symmetric; Q^T Q = diag(multiplicity of the
    global nodes) makes (Q Q^T)^2 = Q Q^T scaled: applied to an assembled
    (continuous) field it multiplies each node by its multiplicity."""
    mesh = BoxMesh(*mesh)
    ones = np.ones(mesh.nelt * mesh.n ** 3)
    mult = mesh.multiplicity().numpy()
    assert np.array_equal(oracle.dssum(ones, mesh.n, mesh.ex, mesh.ey,
                                       mesh.ez), mult)
    a, b = _field(mesh, 2), _field(mesh, 3)
    qa = oracle.dssum(a.copy(), mesh.n, mesh.ex, mesh.ey, mesh.ez)
    qb = oracle.dssum(b.copy(), mesh.n, mesh.ex, mesh.ey, mesh.ez)
    assert abs(qa @ b - a @ qb) <= 1e-12 * (np.abs(qa) @ np.abs(b))
    qqa = oracle.dssum(qa.copy(), mesh.n, mesh.ex, mesh.ey, mesh.ez)
    assert np.allclose(qqa, qa * mult, rtol=1e-13, atol=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_op(w, slab):
    def op(zlo, zhi, mode, plane_in=None, plane_out=None):
        oracle.dssum(w, slab.n, slab.ex, slab.ey, slab.ez, zlo, zhi, mode,
                     None if plane_in is None else plane_in.numpy(),
                     None if plane_out is None else plane_out.numpy())
    return op


def _rank_oracle(rank, world, port, mesh_t, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mesh = BoxMesh(*mesh_t)
    w = _field(mesh, 7)
    z0, z1 = mesh.layers(rank, world)
    per = mesh.ex * mesh.ey * mesh.n ** 3
    mine = w[z0 * per:z1 * per].copy()
    slab = mesh.slab(rank, world)
    wt = torch.from_numpy(mine)
    dssum_sharded(wt, mesh, rank, world, local_op=_oracle_op(mine, slab),
                  plane_device=torch.device("cpu"))
    q.put((rank, z0, mine.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mesh", [(2, (2, 3, 2, 4)), (3, (2, 2, 5, 3)),
                                        (4, (1, 2, 4, 5)), (2, (3, 1, 3, 8))])
def test_sharded_protocol_is_bitwise_single_domain(world, mesh):
    """gloo, one process per rank: interior layers locally, the interface
    planes through partial -> continue -> write-back; the gathered result is
    bitwise the single-domain oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_oracle, args=(r, world, port, mesh, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    m = BoxMesh(*mesh)
    want = oracle.dssum(_field(m, 7), m.n, m.ex, m.ey, m.ez)
    got = b"".join(r[2] for r in res)
    assert got == want.tobytes()


# {{{ device

@pytest.mark.gpu
@pytest.mark.parametrize("mesh", MESHES + [(4, 4, 4, 16), (16, 16, 8, 8)])
def test_device_dssum_matches_the_oracle(cuda, mesh):
    from paper_1503_07659_b200.assembly import dssum
    mesh = BoxMesh(*mesh)
    w = _field(mesh, 11)
    d = torch.from_numpy(w).to(cuda)
    dssum(d, mesh)
    want = oracle.dssum(w.copy(), mesh.n, mesh.ex, mesh.ey, mesh.ez)
    assert d.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("n", list(range(2, 17)))
def test_device_dssum_every_order(cuda, n):
    """The default kernel is instantiated per order (p a compile-time
    constant): every n = 2..16 on a ragged box, whole mesh and a Z range,
    bitwise against the oracle."""
    from paper_1503_07659_b200.assembly import _launch, dssum
    mesh = BoxMesh(3, 2, 4, n)
    w = _field(mesh, n)
    d = torch.from_numpy(w).to(cuda)
    dssum(d, mesh)
    want = oracle.dssum(w.copy(), n, mesh.ex, mesh.ey, mesh.ez)
    assert d.cpu().numpy().tobytes() == want.tobytes()
    # a Z sub-range (as a rank's interior layers): the oracle over the same
    # range
    zlo, zhi = 1, mesh.top - 1
    d = torch.from_numpy(w).to(cuda)
    _launch(d, mesh, zlo, zhi, 0)
    want = oracle.dssum(w.copy(), n, mesh.ex, mesh.ey, mesh.ez, zlo=zlo,
                        zhi=zhi)
    assert d.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.gpu
def test_device_dssum_modes_chain(cuda):
    """Modes 1 -> 2 -> 3 on two slabs of one mesh (in one process) give the
    single-domain kernel's bits."""
    from paper_1503_07659_b200.assembly import _launch, dssum
    mesh = BoxMesh(3, 2, 4, 6)
    w = torch.from_numpy(_field(mesh, 12)).to(cuda)
    whole = w.clone()
    dssum(whole, mesh)
    per = mesh.ex * mesh.ey * mesh.n ** 3
    lo, hi = w[:2 * per], w[2 * per:]
    s_lo, s_hi = mesh.slab(0, 2), mesh.slab(1, 2)
    _launch(lo, s_lo, 0, s_lo.top - 1, 0)
    _launch(hi, s_hi, 1, s_hi.top, 0)
    part = torch.empty(mesh.plane, dtype=torch.float64, device=cuda)
    tot = torch.empty_like(part)
    _launch(lo, s_lo, s_lo.top, s_lo.top, 1, None, part)
    _launch(hi, s_hi, 0, 0, 2, part, tot)
    _launch(lo, s_lo, s_lo.top, s_lo.top, 3, tot, None)
    assert torch.equal(w, whole)


def _rank_device(rank, world, port, mesh_t, q):
    import sys
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mesh = BoxMesh(*mesh_t)
    w = _field(mesh, 13)
    z0, z1 = mesh.layers(rank, world)
    per = mesh.ex * mesh.ey * mesh.n ** 3
    d = torch.from_numpy(w[z0 * per:z1 * per].copy()).cuda()
    dssum_sharded(d, mesh, rank, world)
    torch.cuda.synchronize()
    q.put((rank, d.cpu().numpy().tobytes()))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_sharded_dssum(cuda, world):
    """dssum_sharded with the device kernels, one process per rank (all on
    cuda:0 over gloo -- NCCL refuses two ranks on one GPU): bitwise the
    single-domain oracle."""
    mesh = (4, 3, 6, 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_device, args=(r, world, port, mesh, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    m = BoxMesh(*mesh)
    want = oracle.dssum(_field(m, 13), m.n, m.ex, m.ey, m.ez)
    assert b"".join(r[1] for r in res) == want.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 50])
def test_assembled_operator(cuda, variant):
    """apply_operator = Q Q^T semlap(u): the oracle's semlap followed by the
    oracle's dssum -- bitwise (variant 0); DFMA mode within 1e-12 of the
    magnitude of the summed terms."""
    import paper_1503_07659_b200 as lfb
    from paper_1503_07659_b200 import fixtures as fx
    from paper_1503_07659_b200.assembly import apply_operator
    mesh = BoxMesh(4, 4, 4, 8)
    _r, knl = fx.translate(fx.semlap_source(8, block=1))
    env = lfb.make_device_env(knl, {"nelt": mesh.nelt}, seed=3, device=cuda)
    u, d, g = (env.arrays[a].data.cpu().numpy() for a in ("u", "d", "g"))
    out = apply_operator(knl, env, mesh, variant=variant)
    got = out.arrays["w"].data.cpu().numpy()
    ref = oracle.semlap(np.zeros_like(u), u, d, g, 8, mesh.nelt)
    oracle.dssum(ref, 8, mesh.ex, mesh.ey, mesh.ez)
    if variant == 0:
        assert got.tobytes() == ref.tobytes()
    else:
        mag = oracle.semlap(np.zeros_like(u), np.abs(u), np.abs(d),
                            np.abs(g), 8, mesh.nelt)
        oracle.dssum(mag, 8, mesh.ex, mesh.ey, mesh.ez)
        assert (np.abs(got - ref) <= 1e-12 * mag).all()

# }}}
