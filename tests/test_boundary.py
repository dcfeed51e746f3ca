"""The drop-in boundary: C-ABI exports, ctypes signatures, Python API names.

No GPU needed: the library must load (it links cudart statically and only
touches the device when a kernel is launched) and export every symbol that
include/rskel.h declares.
"""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "rskel.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_09417_b200 import _build, _lib

    if not os.path.exists(_lib.LIB_PATH):
        _build.build()
    return _lib.load()


def test_header_declares_the_hot_path():
    names = header_functions()
    for must in ("rs_sketch_gemm", "rs_panel_lupp", "rs_schur_block", "rs_absorb_block",
                 "rs_scatter_interp", "rs_gather_rows", "rs_dgemm", "rs_rank_update"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_ctypes_table_matches_header():
    from paper_2310_09417_b200 import _lib

    assert sorted(_lib.SIGNATURES) == header_functions()


def test_abi_version_and_status_strings(lib):
    assert lib.rs_abi_version() == 2
    assert lib.rs_status_string(0) == b"ok"
    assert b"capacity" in lib.rs_status_string(-3)
    assert lib.rs_workspace_bytes() > (1 << 20)


def test_python_api_mirrors_reference_hot_path_names():
    import paper_2310_09417_b200 as rs

    # hot-path names of /root/reference/pkg/src/randskel/__init__.py:9-84
    for name in ("RngStream", "SketchSpec", "GaussianSketch", "make_gaussian", "make_sketch",
                 "apply_sketch", "rand_lupp", "column_id", "rand_lupp_adaptive", "SkeletonResult",
                 "ErrorTrace", "TraceRecord", "STATUS_OK", "STATUS_NOT_CONVERGED",
                 "STATUS_RANK_EXHAUSTED", "STATUS_ILL_CONDITIONED", "DimensionError",
                 "RankDeficientError", "SingularError", "NumericalError"):
        assert hasattr(rs, name), name
    assert issubclass(rs.DimensionError, ValueError)
    assert issubclass(rs.RankDeficientError, RuntimeError)
    assert rs.RankDeficientError(3).step == 3


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_2310_09417_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "randskel_oracle" not in src and "oracle/" not in src, f
