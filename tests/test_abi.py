"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every entry point include/duhl.h declares, and fails loudly without a GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "duhl.h")).read()
    return sorted(set(re.findall(r"\b(duhl_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1708_05357_b200 as D
    L = D.lib()
    declared = _declared()
    assert {"duhl_create", "duhl_gaps", "duhl_select", "duhl_scd_epoch", "duhl_duality_gap",
            "duhl_solve"} <= set(declared)
    missing = [f for f in declared if not hasattr(L, f)]
    assert not missing, missing
    assert set(D._abi.FUNCTIONS) == set(declared)


def test_library_is_sm100a():
    import subprocess
    import paper_1708_05357_b200 as D
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", D.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_bulk_async_copy():
    """The SCD kernel stages working-set tiles with cp.async.bulk (SASS UBLKCP)."""
    import subprocess
    import paper_1708_05357_b200 as D
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", D.lib_path()],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in sass


def test_default_config_and_no_gpu_fails_loudly():
    import torch
    import paper_1708_05357_b200 as D
    cfg = D._abi.default_config()
    assert cfg.refresh_fraction == 0.05 and cfg.cert_every == 10 and cfg.seed == 170805357
    if torch.cuda.is_available():
        pytest.skip("GPU present: the no-GPU path is not observable here")
    A = np.ones((4, 4), dtype=np.float32)
    with pytest.raises(D.DuhlError):
        D.create(A, np.ones(4), 0.1, D.LASSO)


def test_invalid_arguments_rejected_before_device():
    import paper_1708_05357_b200 as D
    A = np.ones((4, 4), dtype=np.float32)
    for lam, y, model in [(0.0, np.ones(4), D.LASSO), (-1.0, np.ones(4), D.LASSO),
                          (0.1, np.array([1.0, 2.0, 1.0, -1.0]), D.SVM_DUAL)]:
        with pytest.raises(D.DuhlError) as e:
            D.create(A, y, lam, model)
        assert e.value.status == 2


def test_invalid_csc_rejected_before_device():
    """duhl_create_csc validates the structure on the host (DUHL_E_INVALID, status 2)."""
    import paper_1708_05357_b200 as D
    b = np.ones(5)
    good = (np.array([0, 2, 3]), np.array([0, 3], np.int32), np.array([1.0, 2.0], np.float32))
    cases = [
        (np.array([0, 2, 3]), np.array([3, 0, 1], np.int32), np.ones(3, np.float32)),   # unsorted rows
        (np.array([0, 2, 3]), np.array([0, 5, 1], np.int32), np.ones(3, np.float32)),   # row >= d
        (np.array([0, 2, 1]), np.array([0, 1, 1], np.int32), np.ones(3, np.float32)),   # col_ptr decreasing
        (np.array([1, 2, 3]), np.array([0, 1, 1], np.int32), np.ones(3, np.float32)),   # col_ptr[0] != 0
        (np.array([0, 2, 3]), np.array([0, 1, 1], np.int32),
         np.array([1.0, np.nan, 1.0], np.float32)),                                    # non-finite value
    ]
    for cp, ri, va in cases:
        with pytest.raises(D.DuhlError) as e:
            D.create_csc(cp, ri, va, 5, b, 0.1, D.LASSO)
        assert e.value.status == 2
    with pytest.raises(D.DuhlError) as e:           # lambda must be > 0
        D.create_csc(*good, 5, b, 0.0, D.LASSO)
    assert e.value.status == 2


def _build_abi_check(tmp_path):
    """Compile tests/c/abi_check.c (plain C11) against include/duhl.h, linked to libduhl.so."""
    import subprocess
    import paper_1708_05357_b200 as D
    lib = D.lib_path()
    exe = str(tmp_path / "abi_check")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_check.c"), "-o", exe,
                           "-L", os.path.dirname(lib), "-lduhl", "-lm",
                           f"-Wl,-rpath,{os.path.dirname(lib)}"])
    return exe


def test_c_program_compiles_against_header_and_runs(tmp_path):
    """A C caller compiles against include/duhl.h alone and links libduhl.so; without a GPU
    duhl_create returns DUHL_E_CUDA and the host-only calls (config, group) work."""
    import subprocess
    import torch
    exe = _build_abi_check(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present: the GPU run is tests/test_gpu_edge.py::test_c_program_solves_P1")
    r = subprocess.run([exe, "0"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
