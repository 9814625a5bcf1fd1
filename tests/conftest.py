import json
import os
import struct
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200, sm_100a)")


_DT = {0: np.float32, 1: np.float64, 2: np.int32}


def read_array_file(path):
    """Reader for the reference's array-file format (interp.py:426-449):
    little-endian (dtype code, rank, shape) header, then the data."""
    with open(path, "rb") as f:
        code, rank = struct.unpack("<ii", f.read(8))
        shape = struct.unpack(f"<{rank}i", f.read(4 * rank)) if rank else ()
        data = np.frombuffer(f.read(), dtype=np.dtype(_DT[code])
                             .newbyteorder("<")).astype(_DT[code])
    return data.reshape(shape)


class Golden:
    def __init__(self, name):
        self.name = name
        self.dir = os.path.join(GOLDEN, name)
        with open(os.path.join(self.dir, "meta.json")) as f:
            self.meta = json.load(f)
        self.params = self.meta["params"]
        self.args = self.meta["args"]

    def inp(self, arg):
        return read_array_file(os.path.join(self.dir, f"{arg}.in.bin"))

    def out(self, arg):
        return read_array_file(os.path.join(self.dir, f"{arg}.out.bin"))

    def source(self):
        from paper_1503_07659_b200 import fixtures
        return getattr(fixtures, self.meta["generator"])(**self.meta["kwargs"])

    def kernels(self):
        from paper_1503_07659_b200 import fixtures
        if self.meta["generator"] == "generic_native":
            return fixtures.generic_native(**self.meta["kwargs"])
        return fixtures.translate(self.source(), f"{self.name}.f")

    def outputs(self):
        return [a for a, m in self.args.items() if m["is_output"]]


def golden_names():
    return sorted(d for d in os.listdir(GOLDEN)
                  if os.path.exists(os.path.join(GOLDEN, d, "meta.json")))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1503_07659_b200 import abi
    abi.load()
    return torch.device("cuda", 0)
