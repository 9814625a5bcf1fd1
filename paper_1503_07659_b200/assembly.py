"""SEM assembly: direct-stiffness summation (gather-scatter, Q Q^T) and its
halo exchange across GPUs -- SURVEY.md §8(f) row 4.

The reference's SEM operator is element-local: each
element's w depends only on its own u and g, and interp.py:385-399 runs the
elements as independent outer loops.  A solver built on it (the paper's
motivating application) follows every operator application with the
assembly step w <- Q Q^T w: the values of a node shared by neighbouring
elements are summed and the sum is written back to every copy.  This module
adds that step on the device, for structured boxes of hexahedral elements
(the element numbering the bench and the tests use), so ``apply_operator``
is the full matrix-free SEM operator.

* :class:`BoxMesh` -- Ex x Ey x Ez elements, n points per direction;
  element e = ex + Ex (ey + Ey ez), local node (i, j, k) at
  w[i + n j + n^2 k + n^3 e] (the semlap layout).
* :func:`dssum` -- one device: ``lfb_dssum_f64`` (csrc/dssum.cu), one
  thread per global node, copies summed in ascending element order, so the
  result is deterministic and bitwise the oracle's.
* :func:`dssum_sharded` -- one process per GPU, each owning a slab of
  element layers in z (contiguous element ranges, like dist.shard_range).
  Interface planes get exactly the single-GPU sum: the lower rank forms the
  partial over its copies (mode 1), sends it up, the upper rank continues
  the same left-to-right chain with its copies (mode 2) and sends the total
  back, which the lower rank writes (mode 3).  Two point-to-point exchanges
  of one node plane each between neighbours (NCCL over NVLink on the box,
  gloo on CPU in the tests) -- the only data-path communication, and
  bitwise the single-GPU result.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import abi
from ._loopforge import InterpError


@dataclass(frozen=True)
class BoxMesh:
    """Ex x Ey x Ez hexahedral elements, n points per direction."""

    ex: int
    ey: int
    ez: int
    n: int

    def __post_init__(self):
        if self.n < 2 or min(self.ex, self.ey, self.ez) < 1:
            raise InterpError(f"bad mesh {self}: need n >= 2 and >= 1 "
                              "element per direction")

    @property
    def nelt(self):
        return self.ex * self.ey * self.ez

    @property
    def p(self):
        return self.n - 1

    @property
    def plane(self):
        """Global nodes of one z-plane: (Ex p + 1)(Ey p + 1)."""
        return (self.ex * self.p + 1) * (self.ey * self.p + 1)

    @property
    def top(self):
        return self.ez * self.p

    def multiplicity(self):
        """Local copies per node, element-local layout (float64, CPU): the
        result of Q Q^T applied to ones."""
        n, p = self.n, self.p

        def axis(E):
            # copies along one direction for (element, local index)
            el = torch.arange(E)[:, None]
            m = torch.ones(E, n, dtype=torch.float64)
            m[:, 0] += (el[:, 0] > 0).double()
            m[:, p] += (el[:, 0] < E - 1).double()
            return m

        mx, my, mz = axis(self.ex), axis(self.ey), axis(self.ez)
        # flat order, slowest first: ez, ey, ex, k, j, i
        out = (mz[:, None, None, :, None, None]
               * my[None, :, None, None, :, None]
               * mx[None, None, :, None, None, :])
        return out.reshape(-1)

    def layers(self, rank, world):
        """[z0, z1) element layers of rank *rank* of *world* (contiguous, as
        even as possible)."""
        if world > self.ez:
            raise InterpError(f"{world} ranks for {self.ez} element layers")
        return self.ez * rank // world, self.ez * (rank + 1) // world

    def slab(self, rank, world):
        z0, z1 = self.layers(rank, world)
        return BoxMesh(self.ex, self.ey, z1 - z0, self.n)


def _launch(w, mesh, zlo, zhi, mode, plane_in=None, plane_out=None,
            stream=None):
    if w.dtype != torch.float64 or not w.is_cuda or not w.is_contiguous() \
            or w.numel() < mesh.nelt * mesh.n ** 3:
        raise InterpError("dssum: w must be a contiguous CUDA float64 tensor "
                          f"of >= {mesh.nelt * mesh.n ** 3} elements")
    if stream is None:
        stream = torch.cuda.current_stream(w.device).cuda_stream
    lib = abi.load()
    ptr = abi.C.c_void_p
    abi.check(lib.lfb_dssum_f64(
        ptr(w.data_ptr()), mesh.n, mesh.ex, mesh.ey, mesh.ez, zlo, zhi, mode,
        None if plane_in is None else ptr(plane_in.data_ptr()),
        None if plane_out is None else ptr(plane_out.data_ptr()), stream),
        "dssum_f64")


def dssum(w, mesh, stream=None):
    """Q Q^T on element-local *w* (flat, semlap layout), in place, on one
    device (stream ordered, asynchronous)."""
    _launch(w, mesh, 0, mesh.top, 0, stream=stream)
    return w


def device_local_op(w, mesh):
    """The per-rank kernel calls of :func:`dssum_sharded` on the device."""
    def op(zlo, zhi, mode, plane_in=None, plane_out=None):
        _launch(w, mesh, zlo, zhi, mode, plane_in, plane_out)
    return op


def dssum_sharded(w, mesh, rank, world, group=None, local_op=None,
                  plane_device=None):
    """Q Q^T over a mesh whose element layers are split across *world*
    ranks (this rank holds the element-local *w* of ``mesh.slab(rank,
    world)``, in place).  Bitwise the single-domain :func:`dssum` of the
    whole mesh.  *local_op(zlo, zhi, mode, plane_in, plane_out)* runs the
    local kernel (default: the device kernel on *w*); the interface planes
    live on *plane_device* (default: w's device; NCCL sends them directly,
    gloo through host copies)."""
    import torch.distributed as dist
    slab = mesh.slab(rank, world)
    if local_op is None:
        local_op = device_local_op(w, slab)
    lower, upper = rank > 0, rank < world - 1
    top = slab.top
    zlo, zhi = (1 if lower else 0), (top - 1 if upper else top)
    if zlo <= zhi:
        local_op(zlo, zhi, 0)
    if world == 1:
        return w
    if plane_device is None:
        plane_device = w.device
    # NCCL moves device planes directly; gloo needs host copies
    host_comm = dist.get_backend(group) != "nccl" and \
        plane_device.type == "cuda"

    def plane():
        return torch.empty(slab.plane, dtype=torch.float64,
                           device=plane_device)

    def exchange(send, recv):
        """One point-to-point step: send (tensor, peer) / recv (tensor,
        peer), either may be None."""
        ops, fix = [], None
        if send is not None:
            t = send[0].cpu() if host_comm else send[0]
            ops.append(dist.P2POp(dist.isend, t, send[1], group))
        if recv is not None:
            t = torch.empty(recv[0].shape, dtype=recv[0].dtype) \
                if host_comm else recv[0]
            ops.append(dist.P2POp(dist.irecv, t, recv[1], group))
            fix = (t, recv[0])
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if fix is not None and host_comm:
            fix[1].copy_(fix[0])

    # 1: the partial sums of the top interface plane go up
    part = plane() if upper else None
    if upper:
        local_op(top, top, 1, None, part)
    incoming = plane() if lower else None
    exchange((part, rank + 1) if upper else None,
             (incoming, rank - 1) if lower else None)
    # 2: the upper side of each interface continues the chain and sends the
    # totals back down
    total = plane() if lower else None
    if lower:
        local_op(0, 0, 2, incoming, total)
    back = plane() if upper else None
    exchange((total, rank - 1) if lower else None,
             (back, rank + 1) if upper else None)
    # 3: the lower side writes the totals into its copies
    if upper:
        local_op(top, top, 3, back, None)
    return w


def apply_operator(kernel, env, mesh, variant=0):
    """The assembled SEM operator: w <- Q Q^T semlap(u) -- the element-local
    operator through the drop-in ``interpret`` (in place on env's w), then
    the direct-stiffness summation over *mesh*."""
    from .executor import interpret
    if env.params.get("nelt", mesh.nelt) != mesh.nelt:
        raise InterpError(f"mesh has {mesh.nelt} elements, env "
                          f"{env.params.get('nelt')}")
    out = interpret(kernel, env, inplace=True, variant=variant)
    dssum(out.arrays["w"].data, mesh)
    return out


__all__ = ["BoxMesh", "dssum", "dssum_sharded", "apply_operator",
           "device_local_op"]
