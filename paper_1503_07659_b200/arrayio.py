"""Array files straight to and from HBM.

Same on-disk format as the reference's ``write_array_file`` /
``read_array_file`` (/root/reference/pkg/src/loopforge/interp.py:426-449):
little-endian ``int32 dtype code`` (f32 0, f64 1, i32 2; interp.py:25),
``int32 rank``, ``rank x int32`` shape, then the logical array in C order.
A file written here reads back with the reference's reader and vice versa.

The reference goes file -> numpy -> per-element scatter into its flat
buffers.  Here the payload is read with one ``readinto`` into a pinned host
tensor and copied to the device with one asynchronous H2D copy (and the
reverse for writing), so multi-GiB SEM inputs stream at PCIe speed; the
strided scatter into the kernel's flat layout happens on the device
(``make_device_env``).
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

from ._loopforge import InterpError

_CODE = {"f32": 0, "f64": 1, "i32": 2}
_DTYPE = {0: "f32", 1: "f64", 2: "i32"}
_NP = {"f32": np.float32, "f64": np.float64, "i32": np.int32}
_TORCH = {"f32": torch.float32, "f64": torch.float64, "i32": torch.int32}
_FROM_TORCH = {v: k for k, v in _TORCH.items()}


def read_header(path):
    """(dtype name, shape, payload byte offset)."""
    with open(path, "rb") as f:
        head = f.read(8)
        if len(head) != 8:
            raise InterpError(f"{path}: not an array file (short header)")
        code, rank = struct.unpack("<ii", head)
        if code not in _DTYPE or rank < 0 or rank > 16:
            raise InterpError(f"{path}: bad array header (code {code}, "
                              f"rank {rank})")
        shape = struct.unpack(f"<{rank}i", f.read(4 * rank)) if rank else ()
    return _DTYPE[code], tuple(shape), 8 + 4 * rank


def read_array_file(path, device=None, dtype=None):
    """The array in *path* as a tensor of its logical shape on *device*
    (default: the current CUDA device).  *dtype* ("f32"/"f64"/"i32")
    converts after loading, like the reference's ``np.asarray(src, dtype)``
    in make_env."""
    name, shape, off = read_header(path)
    count = int(np.prod(shape, dtype=np.int64)) if shape else 1
    nbytes = count * np.dtype(_NP[name]).itemsize
    if os.path.getsize(path) != off + nbytes:
        raise InterpError(f"{path}: payload is {os.path.getsize(path) - off}"
                          f" bytes, header says {nbytes}")
    host = torch.empty(count, dtype=_TORCH[name],
                       pin_memory=torch.cuda.is_available())
    with open(path, "rb") as f:
        f.seek(off)
        view = host.numpy().view(np.uint8)
        if f.readinto(memoryview(view)) != nbytes:
            raise InterpError(f"{path}: short read")
    if np.little_endian is False:  # pragma: no cover - big-endian hosts
        host = torch.from_numpy(host.numpy().byteswap())
    dev = device if device is not None else (
        torch.device("cuda", torch.cuda.current_device())
        if torch.cuda.is_available() else torch.device("cpu"))
    out = host.to(dev, non_blocking=True)
    if dtype is not None and _TORCH[dtype] != out.dtype:
        out = out.to(_TORCH[dtype])
    return out.reshape(shape) if shape else out.reshape(())


def write_array_file(path, array, dtype=None):
    """Write a tensor (any device) or numpy array of logical shape."""
    if isinstance(array, np.ndarray) or np.isscalar(array):
        array = torch.from_numpy(np.asarray(array))
    name = dtype or _FROM_TORCH.get(array.dtype)
    if name is None:
        raise InterpError(f"unsupported dtype {array.dtype}")
    t = array.to(_TORCH[name]).contiguous()
    host = torch.empty(t.shape, dtype=t.dtype,
                       pin_memory=torch.cuda.is_available() and t.is_cuda)
    host.copy_(t)
    with open(path, "wb") as f:
        f.write(struct.pack("<ii", _CODE[name], host.dim()))
        f.write(struct.pack(f"<{host.dim()}i", *host.shape))
        f.write(host.numpy().astype(
            np.dtype(_NP[name]).newbyteorder("<"), copy=False).tobytes())
