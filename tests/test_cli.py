"""CLI and array-file I/O (interp.py:426-449) --
SURVEY.md §8(f) row 2.  CPU tests: the file format against the reference's
golden files byte for byte, the front-end modes, the exit codes.  GPU tests:
``run`` on every Fortran golden fixture, outputs bitwise the reference's
interpret() results."""

import filecmp
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import REPO, Golden, golden_names, read_array_file
from paper_1503_07659_b200 import arrayio, fixtures as fx
from paper_1503_07659_b200.cli import main


def _golden_files():
    for name in golden_names():
        d = os.path.join(REPO, "tests", "golden", name)
        for f in sorted(os.listdir(d)):
            if f.endswith(".bin"):
                yield os.path.join(d, f)


@pytest.mark.parametrize("path", list(_golden_files())[:40])
def test_arrayio_reads_and_rewrites_reference_files(path, tmp_path):
    """Files written by the reference's write_array_file read back equal and
    re-write byte for byte."""
    t = arrayio.read_array_file(path, device="cpu")
    ref = read_array_file(path)
    assert t.numpy().shape == ref.shape
    assert t.numpy().tobytes() == ref.tobytes()
    out = tmp_path / "x.bin"
    arrayio.write_array_file(str(out), t)
    assert filecmp.cmp(path, str(out), shallow=False)


def test_arrayio_header_errors(tmp_path):
    from paper_1503_07659_b200._loopforge import InterpError
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x07\x00\x00\x00\x01\x00\x00\x00")
    with pytest.raises(InterpError):
        arrayio.read_array_file(str(bad), device="cpu")
    short = tmp_path / "short.bin"
    arrayio.write_array_file(str(short), np.arange(10, dtype=np.float64))
    short.write_bytes(short.read_bytes()[:-8])
    with pytest.raises(InterpError):
        arrayio.read_array_file(str(short), device="cpu")


def test_arrayio_with_the_reference_reader(tmp_path):
    from paper_1503_07659_b200._loopforge import interp
    a = np.random.default_rng(3).random((3, 5, 7))
    p = tmp_path / "a.bin"
    arrayio.write_array_file(str(p), torch.from_numpy(a))
    assert np.array_equal(interp.read_array_file(str(p)), a)
    q = tmp_path / "b.bin"
    interp.write_array_file(str(q), a.astype(np.float32))
    assert np.array_equal(arrayio.read_array_file(str(q), device="cpu")
                          .numpy(), a.astype(np.float32))


def _src(tmp_path, text, name="k.f"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_cli_translate_dump_check(tmp_path, capsys):
    f = _src(tmp_path, fx.fill_source("f64"))
    assert main(["translate", f, "--target", "opencl"]) == 0
    out = capsys.readouterr().out
    assert "get_group_id(0)" in out and "1 + i_inner + 128 * i_outer <= n" \
        in out
    assert main(["translate", f, "--target", "cuda"]) == 0
    assert "blockIdx.x" in capsys.readouterr().out
    assert main(["dump-ir", f, "--stage", "raw"]) == 0
    assert "kernel: fill" in capsys.readouterr().out
    s = _src(tmp_path, fx.semlap_source(4), "sem.f")
    assert main(["check", s, "--param", "nelt=64"]) == 0
    rep = capsys.readouterr().out
    assert '"workload": "semlap"' in rep and '"npts": 4' in rep


def test_cli_extra_transform_script(tmp_path, capsys):
    """--transforms applies after the embedded blocks."""
    f = _src(tmp_path, fx.fill_source("f64", script=False))
    t = tmp_path / "t.txt"
    t.write_text('fill = lp.split_iname(fill, "i", 128, outer_tag="g.0", '
                 'inner_tag="l.0")\nfill = lp.assume(fill, "n mod 128 = 0")\n')
    assert main(["translate", f, "--target", "opencl"]) == 0
    assert "get_group_id" not in capsys.readouterr().out
    assert main(["translate", f, "--target", "opencl", "--transforms",
                 str(t)]) == 0
    out = capsys.readouterr().out
    assert "get_group_id(0)" in out and "<= n" not in out  # guard elided


def test_cli_user_errors_exit_1(tmp_path, capsys):
    f = _src(tmp_path, fx.fill_source("f64"))
    # run needs its parameter bindings
    assert main(["run", f, "--scalar", "a=1", "--out",
                 f"out={tmp_path}/o.bin"]) == 1
    assert "--param" in capsys.readouterr().err
    bad = _src(tmp_path, "subroutine x(a)\n  real*8 a(\nend\n", "bad.f")
    assert main(["dump-ir", bad]) == 1
    err = capsys.readouterr().err
    assert "bad.f" in err  # diagnostic carries the source span


def test_cli_module_entry_point(tmp_path):
    f = _src(tmp_path, fx.fill_source("f64"))
    r = subprocess.run([sys.executable, "-m", "paper_1503_07659_b200",
                        "dump-ir", f], capture_output=True, text=True,
                       cwd=REPO)
    assert r.returncode == 0 and "kernel: fill" in r.stdout


def _fortran_goldens():
    return [n for n in golden_names()
            if Golden(n).meta["generator"] != "generic_native"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", _fortran_goldens())
def test_cli_run_matches_reference_goldens(cuda, name, tmp_path):
    """run <file> --param ... --in ... --out ...: outputs bitwise the
    reference interpret() golden vectors."""
    g = Golden(name)
    src = _src(tmp_path, g.source(), f"{name}.f")
    argv = ["run", src]
    for k, v in g.params.items():
        argv += ["--param", f"{k}={v}"]
    for a in g.args:
        p = os.path.join(g.dir, f"{a}.in.bin")
        if os.path.exists(p):
            argv += ["--in", f"{a}={p}"]
    outs = g.outputs()
    for a in outs:
        argv += ["--out", f"{a}={tmp_path}/{a}.bin"]
    argv.append("--flat-out")  # the goldens hold the flat buffers
    assert main(argv) == 0
    for a in outs:
        got = read_array_file(f"{tmp_path}/{a}.bin")
        want = g.out(a)
        assert got.shape == want.shape
        assert got.tobytes() == want.tobytes(), a


@pytest.mark.gpu
@pytest.mark.parametrize("src,params", [
    (fx.semlap_source(8, block=2), {"nelt": 6}),
    (fx.matvec_source("f64"), {"n": 256}),
    (fx.axpy_source("f32"), {"n": 333}),
    (fx.gemm_source("f64"), {"m": 40, "n": 24, "l": 48}),
], ids=["semlap8", "matvec", "axpy32", "dgemm"])
def test_cli_check_smoke_engines_agree(cuda, src, params, tmp_path, capsys):
    """check --smoke: hand-written kernel vs generated CUDA on the device,
    same seeded inputs: bitwise, or within the tolerance where the default
    kernel reassociates (matvec split-j, DMMA GEMM)."""
    path = _src(tmp_path, src, "k.f")
    argv = ["check", path, "--smoke"]
    for k, v in params.items():
        argv += ["--param", f"{k}={v}"]
    assert main(argv) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["smoke"]["agree"]
    if "semlap" in src or "axpy" in src:
        assert rep["smoke"]["bitwise"]


@pytest.mark.gpu
def test_cli_run_bounds_check(cuda, tmp_path):
    """run --bounds-check: the checked device build, same bits."""
    g = Golden("gen_dgemm_m20_n12_l40")
    src = _src(tmp_path, g.source(), "dgemm.f")
    argv = ["run", src, "--bounds-check", "--flat-out"]
    for k, v in g.params.items():
        argv += ["--param", f"{k}={v}"]
    for a in g.args:
        p = os.path.join(g.dir, f"{a}.in.bin")
        if os.path.exists(p):
            argv += ["--in", f"{a}={p}"]
    argv += ["--out", f"c={tmp_path}/c.bin"]
    assert main(argv) == 0
    assert read_array_file(f"{tmp_path}/c.bin").tobytes() == \
        g.out("c").tobytes()
