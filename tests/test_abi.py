"""Host-side checks of the C ABI (-m "not gpu"): the library builds, loads, exports
every symbol include/maspcg.h declares, validates arguments before touching a
device, and shares no code with the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "maspcg.h")


@pytest.fixture(scope="module")
def L():
    from paper_2303_03398_b200 import build, maspcg
    build.build()
    return maspcg.lib()


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"MASPCG_API\s+[\w\s\*]+?\b(maspcg_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("maspcg_create", "maspcg_set_grid", "maspcg_set_workspace", "maspcg_set_coefficients",
                 "maspcg_set_bc_r", "maspcg_solve", "maspcg_apply", "maspcg_destroy", "maspcg_last_error",
                 "maspcg_local_extent", "maspcg_workspace_bytes"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    from paper_2303_03398_b200 import maspcg
    names = declared_functions()
    for n in names:
        assert hasattr(L, n), n
    # the binding's signature table covers exactly the header
    assert sorted(maspcg.SIGNATURES) == names


def test_no_torch_types_in_the_abi():
    src = open(HEADER).read()
    assert "torch" not in src.split("*/", 1)[1].lower() or "at::" not in src
    assert "at::Tensor" not in src and "c10" not in src


def test_version_and_argument_validation_without_gpu(L):
    from paper_2303_03398_b200 import maspcg
    assert L.maspcg_version().decode().startswith("maspcg")
    ctx = ctypes.c_void_p()
    # argument errors are detected before any device call
    assert L.maspcg_create(0, 4, 4, 0, 1, None, 0, ctypes.byref(ctx)) == maspcg.E_INVALID
    assert L.maspcg_create(4, 4, 6, 0, 4, b"x" * 128, 0, ctypes.byref(ctx)) == maspcg.E_INVALID  # 6 % 4
    assert b"divisible" in L.maspcg_last_error(None)
    assert L.maspcg_create(4, 4, 8, 0, 2, None, 0, ctypes.byref(ctx)) == maspcg.E_INVALID     # no unique id
    assert L.maspcg_create(4, 4, 8, 2, 2, b"x" * 128, 0, ctypes.byref(ctx)) == maspcg.E_INVALID  # rank
    assert L.maspcg_create(2000, 2000, 600, 0, 1, None, 0, ctypes.byref(ctx)) == maspcg.E_INVALID  # > 2^31
    assert L.maspcg_destroy(None) == maspcg.OK
    assert L.maspcg_solve(None, None, None, 1e-10, 10, None, None, None) == maspcg.E_INVALID


def test_no_cpu_fallback_without_gpu(L):
    """On a host without a GPU, a valid create must fail with E_CUDA (nothing runs on the CPU)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2303_03398_b200 import maspcg
    ctx = ctypes.c_void_p()
    st = L.maspcg_create(4, 4, 8, 0, 1, None, 0, ctypes.byref(ctx))
    assert st == maspcg.E_CUDA
    with pytest.raises(maspcg.MaspcgError):
        maspcg.Solver(4, 4, 8, [1, 2, 3, 4, 5], [0, .5, 1, 2, 3], [0, 1, 2, 3, 4, 5, 6, 6.283185307179586, 7])


def test_oracle_and_product_share_no_code():
    """The oracle (oracle/) and the CUDA path (paper_2303_03398_b200/, include/) never include,
    import or link each other; only the seeded input generators are common."""
    prod_files = []
    for d in ("paper_2303_03398_b200", "include"):
        for dirpath, _, files in os.walk(os.path.join(ROOT, d)):
            prod_files += [os.path.join(dirpath, f) for f in files if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp"))]
    for f in prod_files:
        s = open(f).read()
        assert "masoracle" not in s, f
        assert not re.search(r"^\s*(import|from)\s+oracle\b", s, re.M), f
    for dirpath, _, files in os.walk(os.path.join(ROOT, "oracle")):
        for fn in files:
            if fn.endswith((".py", ".c", ".h")):
                s = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r'#\s*include\s*[<"][^>"]*(maspcg\.h|\.cuh)', s), fn
                assert not re.search(r"^\s*(import|from)\s+paper_2303_03398_b200", s, re.M), fn
                assert not re.search(r"CDLL\([^)]*maspcg|-lmaspcg", s), fn
