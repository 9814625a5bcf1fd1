"""The C-ABI library loads and exports every symbol include/*.h declares
(CPU only: no compute calls)."""

import ctypes
import os
import re
import subprocess

from paper_1503_07659_b200 import abi
from paper_1503_07659_b200.build import INCLUDE, LIB

HEADER = os.path.join(INCLUDE, "loopforge_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lfb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_entry_points():
    syms = declared_symbols()
    for s in ("lfb_fill_f64", "lfb_axpy_f64", "lfb_matvec_f64",
              "lfb_semlap_f64", "lfb_sgemm_f32", "lfb_dgemm_f64", "lfb_last_error",
              "lfb_abi_version"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build()"
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", LIB],
                        capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", nm), s


def test_bindings_cover_the_header():
    assert set(abi.SIGNATURES) == set(declared_symbols())


def test_abi_version_and_error_text():
    lib = abi.load()
    assert lib.lfb_abi_version() == abi.ABI_VERSION
    # an argument error needs no GPU and sets the thread-local text
    rc = lib.lfb_fill_f64(None, 1.0, 10, None, None)
    assert rc == abi.LFB_ERR_ARG
    assert "null output" in abi.last_error()
    rc = lib.lfb_semlap_f64(None, None, None, None, 10, None, None)
    assert rc == abi.LFB_ERR_ARG


def test_launch_struct_layout(tmp_path):
    """ctypes mirror == the C compiler's layout of struct lfb_launch."""
    fields = [f[0] for f in abi.LfbLaunch._fields_]
    prog = tmp_path / "layout.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "loopforge_b200.h"\n'
        "int main(void){printf(\"%zu\", sizeof(lfb_launch));"
        + "".join(f'printf(" %zu", offsetof(lfb_launch, {f}));'
                  for f in fields) + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["cc", "-I", INCLUDE, "-o", str(exe), str(prog)],
                   check=True)
    got = [int(v) for v in subprocess.run(
        [str(exe)], capture_output=True, text=True).stdout.split()]
    assert got[0] == ctypes.sizeof(abi.LfbLaunch)
    assert got[1:] == [getattr(abi.LfbLaunch, f).offset for f in fields]


def test_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly():
    """No CPU fallback: without the built .so the executor raises."""
    import subprocess
    import sys
    code = ("from paper_1503_07659_b200 import abi\n"
            "abi.LIB = '/nonexistent/libloopforge_b200.so'\n"
            "try:\n"
            "    abi.load()\n"
            "except Exception as e:\n"
            "    print(type(e).__name__, e)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True,
                       text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(
                           os.path.abspath(__file__))))
    assert "InterpError" in r.stdout and "no CPU fallback" in r.stdout
