"""The C-ABI is usable from plain C: examples/listing1.c compiles against
include/jacc.h and links libjacc.so (CPU); on a B200 it runs (gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    import __graft_entry__ as ge
    lib = ge.build_jacc()
    exe = str(tmp_path / "listing1")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "listing1.c"), "-o", exe,
                        "-L", os.path.dirname(lib), "-ljacc",
                        f"-Wl,-rpath,{os.path.dirname(lib)}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3])
def test_c_example_runs(tmp_path, n):
    exe = _build(tmp_path)
    r = subprocess.run([exe, str(n)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "x = 1 4 9" in r.stdout and r.stdout.strip().endswith("ok")
