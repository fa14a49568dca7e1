"""CPU checks of the drop-in boundary: the C ABI library loads and exports
every entry point include/seethrough_b200.h declares (no compute calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seethrough_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:const\s+)?\w+\*?\s+\*?(st_\w+)\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2003_11076_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_entry_points():
    names = declared()
    for must in ("st_solve", "st_synthesize", "st_e_step", "st_m_step", "st_e_step_at",
                 "st_descriptors", "st_bilinear", "st_mu_raster", "st_support_build",
                 "st_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header(lib):
    from paper_2003_11076_b200 import _native
    assert set(_native.exported_symbols()) == set(declared())


def test_struct_layouts_match_the_header(lib):
    """The ctypes mirrors have the size the compiled library gives each struct."""
    from paper_2003_11076_b200 import _native as N
    mirrors = (N.StRig, N.StParams, N.StStats, N.StFrame, N.StTri, N.StCams, N.StFramePlan,
               N.StScene)
    for which, cls in enumerate(mirrors):
        assert ctypes.sizeof(cls) == N.lib().st_struct_size(which), cls.__name__
    assert N.lib().st_struct_size(99) == -1
    assert ctypes.sizeof(N.StStats) == 8 + 3 * N.MAX_ITERS * 8 + 7 * 8 + 4 * 8 + 4 * 4 + 2 * 8


def test_version_and_error_calls_need_no_gpu(lib):
    lib.st_version.restype = ctypes.c_int
    assert lib.st_version() >= 10000
    lib.st_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.st_last_error(), bytes)


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import numpy as np
    import paper_2003_11076_b200 as st
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        st.e_step(np.zeros((1, 3, 16)), np.ones((1, 3), bool), np.full((1, 3), 0.5),
                  st.SolverParams())
