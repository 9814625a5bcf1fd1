"""Multi-process host logic on CPU (gloo, world_size 2): element shards and
the verification-norm all-reduce."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import REPO
from paper_1503_07659_b200.dist import (allreduce_max, allreduce_sum,
                                        shard_params, shard_range)


@pytest.mark.parametrize("nelt,world,block", [(1 << 21, 8, 32), (100, 3, 7),
                                              (65536, 2, 32), (5, 4, 1),
                                              (31, 2, 32)])
def test_shards_partition_elements(nelt, world, block):
    spans = [shard_range(nelt, r, world, block) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == nelt
    for (a, b), (c, _d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    for lo, hi in spans[:-1]:
        assert lo % block == 0 and hi % block == 0


def test_shard_params():
    assert shard_params({"nelt": 64, "q": 1}, "nelt", 32, 64) == \
        {"nelt": 32, "q": 1}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, nelt, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)            # same global problem everywhere
    u = rng.random(nelt * n**3)
    g = rng.random(6 * nelt * n**3)
    d = rng.random(n * n)
    lo, hi = shard_range(nelt, rank, world, 4)
    w = np.zeros_like(u)
    oracle.semlap(w, u, d, g, n, nelt, elems=(lo, hi))
    part = oracle.sumsq(np.ascontiguousarray(w[lo * n**3:hi * n**3]))
    total = allreduce_sum(part)
    worst = allreduce_max(float(rank))
    q.put((rank, total, worst))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_gloo_world2_norm_allreduce(world):
    """world 2 as the contract asks, and 3 / 4 ranks (uneven shards, one
    rank with a partial block) on the same gloo path."""
    n, nelt = 4, 18
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nelt, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    u = rng.random(nelt * n**3)
    g = rng.random(6 * nelt * n**3)
    d = rng.random(n * n)
    w = oracle.semlap(np.zeros_like(u), u, d, g, n, nelt)
    want = float((w * w).sum())
    for _rank, total, worst in res:
        assert abs(total - want) <= 1e-12 * want
        assert worst == world - 1


@pytest.mark.gpu
def test_bench_multi_rank_path_on_one_gpu(tmp_path):
    """bench.py under torchrun with 2 ranks (both on cuda:0, gloo -- NCCL
    refuses two ranks on one GPU): element shards, barriers, max over ranks,
    the all-reduced verification norm and one JSON line from rank 0."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, LFB_BENCH_ONE_DEVICE="1", LFB_BENCH_BACKEND="gloo")
    r = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
         "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
         "--master-port", "29541", os.path.join(REPO, "bench.py"),
         "--gpus", "2", "--workload", "sem65k", "--steps", "3",
         "--warmup", "3", "--no-cpu", "--e2e-nelt", "4096"],
        capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["verify"]["max_err_over_magnitude_head"] <= 1e-12
    assert d["verify"]["max_err_over_magnitude_tail"] <= 1e-12
    assert d["e2e"]["value"] > 0


@pytest.mark.gpu
def test_bench_spawns_its_own_ranks(tmp_path):
    """`python bench.py --gpus 2` WITHOUT torchrun (how the driver's scaling
    run invokes it) starts its own two ranks and reports n_gpus 2 with the
    all-reduced norm and a 2-rank communicator -- never a silent 1-GPU run.
    Both ranks on cuda:0 over gloo (NCCL refuses two ranks on one GPU)."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, LFB_BENCH_ONE_DEVICE="1", LFB_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
         "--workload", "sem65k", "--steps", "3", "--warmup", "3", "--no-cpu",
         "--e2e-nelt", "4096"],
        capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["comm"]["world_size"] == 2
    assert d["comm"]["allreduce_of_ones"] == 2.0
    assert sorted(x["rank"] for x in d["comm"]["ranks"]) == [0, 1]
    assert d["verify"]["max_err_over_magnitude_head"] <= 1e-12
    assert d["e2e"]["verify_tail"]["max_err_over_magnitude"] <= 1e-12


def test_bench_refuses_more_gpus_than_visible():
    """Without enough visible devices `bench.py --gpus 2` fails loudly with
    an error line instead of timing one GPU (CPU container: 0 devices)."""
    import json
    import subprocess
    import sys

    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough devices here")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("LFB_BENCH_ONE_DEVICE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"),
                        "--gpus", "2"], capture_output=True, text=True,
                       timeout=300, env=env, cwd=REPO)
    assert r.returncode != 0
    d = json.loads([l for l in r.stdout.splitlines()
                    if l.startswith("{")][0])
    assert "only" in d["error"]


@pytest.mark.gpu
def test_bench_semop_two_ranks(tmp_path):
    """The assembled operator (semlap + Q Q^T) with its interface exchange
    on 2 ranks (both on cuda:0, gloo): one JSON line, n_gpus 2."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, LFB_BENCH_ONE_DEVICE="1", LFB_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
         "--workload", "semop", "--semop-e", "16", "--steps", "3",
         "--warmup", "3"],
        capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["comm"]["world_size"] == 2
