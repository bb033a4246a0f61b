"""C-ABI checks that need no GPU (-m "not gpu"): the library builds, loads
and exports every entry point include/jacc.h declares; calls without a
runtime fail with JACC_ERR_STATE instead of crashing; host-side logic
(partition) agrees with the oracle."""
import os
import re

import pytest

import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def J():
    import __graft_entry__ as ge
    ge.build_jacc()
    from paper_2110_14340_b200 import jacc
    return jacc


def _declared():
    src = open(os.path.join(ROOT, "include", "jacc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jacc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("jacc_data_create", "jacc_data_delete", "jacc_launch", "jacc_update_host",
              "jacc_update_device", "jacc_wait"):
        assert n in names


def test_library_exports_every_declared_symbol(J):
    for name in _declared():
        assert hasattr(J.lib, name), name
    assert sorted(J.EXPORTS) == _declared()


def test_no_torch_in_the_boundary():
    src = open(os.path.join(ROOT, "include", "jacc.h")).read()
    assert "torch" not in src.lower().replace("/*", "").split("*/")[-1]
    assert "#include <torch" not in src


def test_calls_before_init_return_state(J):
    assert J.jacc_num_devices() == 0
    assert J.lib.jacc_wait(-1) == J.JACC_ERR_STATE
    assert J.lib.jacc_data_delete(None) == J.JACC_ERR_STATE
    assert J.lib.jacc_launch(J.JACC_LOOP_DOT_F64, None, None, 0, -1) == J.JACC_ERR_STATE
    assert J.lib.jacc_finalize() == J.JACC_ERR_STATE
    assert J.lib.jacc_set_merge_policy(0) == J.JACC_ERR_STATE


def test_init_without_gpu_fails_cleanly(J):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st = J.lib.jacc_init(1, None)
    assert st in (J.JACC_ERR_CUDA, J.JACC_ERR_INVALID)
    assert J.jacc_num_devices() == 0


def test_error_strings_stable(J):
    for st, key in ((0, "JACC_OK"), (-1, "INVALID"), (-2, "OVERLAP"), (-3, "NOT_PRESENT"),
                    (-4, "UNKNOWN_LOOP"), (-5, "OOM"), (-6, "CUDA"), (-7, "NCCL"), (-8, "STATE")):
        assert key in J.jacc_error_string(st)


@pytest.mark.parametrize("n", range(1, 10))
def test_runtime_partition_matches_oracle(J, n):
    for E in list(range(0, 50)) + [16384, 8192, 2**28, 2**30, 2**30 + 5]:
        for d in range(n):
            assert J.jacc_partition(E, n, d) == orc.partition(E, n, d), (E, n, d)


def test_partition_rejects_bad_args(J):
    import ctypes
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    for E, n, d in ((-1, 2, 0), (5, 0, 0), (5, 2, 2), (5, 2, -1)):
        assert J.lib.jacc_partition(E, n, d, ctypes.byref(lo), ctypes.byref(hi)) == J.JACC_ERR_INVALID


def test_sass_is_sm100a_and_uses_dmma(J):
    """The fp64 GEMM loop runs on the tensor pipe (DMMA), built as sm_100a SASS."""
    import subprocess
    so = J.LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass


def test_library_exports_only_the_c_abi(J):
    """csrc/exports.map: the C-ABI and nothing else (no C++ runtime, kernel
    wrapper or std:: template symbols leak out of libjacc.so)."""
    import subprocess
    r = subprocess.run(["nm", "-D", "--defined-only", J.lib._name], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("nm unavailable")
    syms = [ln.split()[-1] for ln in r.stdout.splitlines() if ln.strip()]
    assert syms and all(s.startswith("jacc_") for s in syms), [s for s in syms if not s.startswith("jacc_")][:5]
    assert sorted(syms) == _declared()
