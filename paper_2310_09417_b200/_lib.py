"""ctypes binding of librskel.so (the C ABI declared in include/rskel.h).

This is the only place Python touches the native library.  Device buffers are
passed as raw pointers (``tensor.data_ptr()``) and streams as
``cudaStream_t`` handles; there are no torch types in the ABI.  A missing or
broken library raises :class:`DeviceError` -- there is no CPU fallback.
"""

import ctypes
import os

from .errors import DeviceError

_PKG_DIR = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_LIB = os.path.join(_PKG_DIR, "librskel.so")
# experiment builds (tools/build_*_variants.sh) can be loaded in place of the library
LIB_PATH = os.environ.get("RSKEL_LIB_PATH") or _DEFAULT_LIB

_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_c_double = ctypes.c_double
_p = ctypes.c_void_p

# name -> (restype, argtypes); must match include/rskel.h
SIGNATURES = {
    "rs_abi_version": (_c_int, []),
    "rs_status_string": (ctypes.c_char_p, [_c_int]),
    "rs_workspace_bytes": (ctypes.c_size_t, []),
    "rs_launch_count": (ctypes.c_ulonglong, []),
    "rs_dgemm": (_c_int, [_c_int, _c_int, _c_int, _c_double, _p, _c_ll, _c_int, _p, _p, _c_ll, _p,
                          _c_double, _p, _c_ll, _p, _p, _c_ll, _p, _p]),
    "rs_gemm_chunk": (_c_int, [_c_ll]),
    "rs_dgemm_ex": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _p, _c_ll, _c_int, _p, _p, _c_ll,
                             _p, _c_double, _p, _c_ll, _p, _p, _c_ll, _p, _p]),
    "rs_sketch_gemm": (_c_int, [_c_int, _c_int, _c_int, _p, _c_ll, _c_int, _p, _c_ll, _p, _c_ll,
                                _p, _p]),
    "rs_panel_lupp": (_c_int, [_p, _c_ll, _c_int, _c_int, _p, _p, _p, _p]),
    "rs_schur_block": (_c_int, [_c_int, _c_int, _c_int, _p, _c_ll, _p, _p, _c_ll, _p, _c_ll, _p, _p, _p]),
    "rs_absorb_block": (_c_int, [_c_int, _c_int, _c_int, _p, _c_ll, _p, _p, _c_ll, _p, _p, _p, _p, _p]),
    "rs_absorb_schur": (_c_int, [_c_int, _c_int, _c_int, _p, _c_ll, _p, _p, _c_ll, _p, _p, _p, _p, _c_ll,
                                 _p, _p, _p, _p]),
    "rs_rank_update": (_c_int, [_c_int, _c_int, _c_int, _p, _c_ll, _p, _c_ll, _p, _p, _c_ll, _p, _p,
                                _c_ll, _p]),
    "rs_scatter_interp":(_c_int, [_p, _c_ll, _p, _c_int, _c_int, _p, _c_ll, _p]),
    "rs_gather_rows": (_c_int, [_p, _c_ll, _p, _c_int, _c_int, _p, _c_ll, _p]),
    "rs_sumsq": (_c_int, [_p, _c_ll, _c_int, _c_int, _p, _p, _p]),
    "rs_trinv": (_c_int, [_p, _c_ll, _c_ll, _p, _c_int, _c_int, _c_int, _p, _c_ll, _p]),
    "rs_perm_update": (_c_int, [_p, _p, _c_int, _c_int, _p, _p]),
    "rs_transpose": (_c_int, [_p, _c_ll, _c_int, _c_int, _p, _c_ll, _p]),
    "rs_jacobi_round": (_c_int, [_p, _c_ll, _c_int, _p, _c_ll, _c_int, _p, _c_int, _c_double, _p, _p]),
    "rs_pinv_scale": (_c_int, [_p, _c_ll, _c_int, _p, _c_ll, _c_int, _c_double, _p, _p]),
    "rs_norm1": (_c_int, [_p, _c_ll, _c_int, _c_int, _p, _p]),
    "rs_cholesky": (_c_int, [_p, _c_ll, _c_int, _p, _p]),
    "rs_trsv_cols": (_c_int, [_p, _c_ll, _c_int, _c_int, _c_int, _p, _p]),
    "rs_what": (_c_int, [_p, _c_ll, _p, _c_int, _p, _c_int, _p, _c_ll, _p]),
    "rs_srtt_dense": (_c_int, [_c_int, _c_int, _p, _p, _p, _c_double, _p, _c_ll, _p]),
    "rs_sparse_sign_dense": (_c_int, [_c_int, _c_int, _c_int, _p, _p, _c_double, _p, _c_ll, _p]),
    "rs_srtt_workspace_bytes": (_c_ll, [_c_ll, _c_int]),
    "rs_srtt_apply": (_c_int, [_c_ll, _c_int, _c_int, _p, _c_ll, _c_int, _p, _p, _p, _c_double, _p, _c_ll, _p, _c_ll,
                               _p]),
    "rs_sparse_sign_plan_bytes": (_c_ll, [_c_int, _c_int]),
    "rs_sparse_sign_apply": (_c_int, [_c_ll, _c_int, _c_int, _c_int, _p, _c_ll, _c_int, _p, _p, _c_double, _p, _c_ll,
                                      _p, _p, _p]),
    "rs_jacobi_sweep": (_c_int, [_p, _c_ll, _c_int, _p, _c_ll, _c_int, _p, _c_int, _c_int, _c_double, _p, _p, _p]),
    "rs_gather2d": (_c_int, [_p, _c_ll, _c_ll, _p, _c_int, _p, _c_int, _p, _c_ll, _p]),
    "rs_gaussian_workspace_bytes": (ctypes.c_size_t, [_c_ll]),
    "rs_gaussian": (_c_int, [ctypes.c_ulonglong, ctypes.c_ulonglong, _c_ll, _c_double, _p, _p,
                             ctypes.c_size_t, _p, _p]),
    "rs_iota": (_c_int, [_p, _c_int, _p]),
    "rs_shard_maps": (_c_int, [_p, _c_int, _c_int, _c_ll, _c_ll, _p, _p, _c_int, _c_int, _p, _p, _p, _p, _p,
                               _p, _p, _p, _c_int, _p]),
    "rs_shard_max_count": (_c_int, [_p, _c_int, _c_int, _p, _c_int, _p, _p]),
    "rs_scatter_rows": (_c_int, [_p, _c_ll, _p, _c_int, _c_int, _p, _c_ll, _p]),
    "rs_scatter_interp_local": (_c_int, [_p, _c_ll, _p, _c_int, _p, _c_int, _c_ll, _c_ll, _p, _c_ll, _p]),
    "rs_oz_chunk": (_c_int, [_c_ll]),
    "rs_oz_digits_bytes": (ctypes.c_size_t, [_c_int, _c_ll, _c_int, _c_int]),
    "rs_oz_slice": (_c_int, [_p, _c_int, _c_ll, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _p,
                             _p, _p, _p, _p]),
    "rs_oz_gemm": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _p, _p, _c_int, _p, _p, _c_int,
                            _c_double, _p, _c_ll, _p, _c_ll, _p, _p]),
    "rs_uniform": (_c_int, [ctypes.c_ulonglong, ctypes.c_ulonglong, _c_ll, _p, _p]),
    "rs_hadamard_init": (_c_int, [_p, _c_ll, _c_int, _c_double, _p, _p]),
    "rs_fwht_rows": (_c_int, [_p, _c_ll, _c_int, _c_double, _p, _p]),
    "rs_kahan": (_c_int, [_p, _c_ll, _c_int, _p, _c_double, _p]),
    "rs_chan": (_c_int, [_p, _c_ll, _c_int, _p]),
    "rs_axpy_cast": (_c_int, [_p, _p, _c_double, _c_ll, _p, _p, _p]),
}

ABI_VERSION = 2

_lib = None


def load(path=LIB_PATH):
    """Load (once) and type the shared library; raise DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(
            f"{path} is missing: build it with `python -m paper_2310_09417_b200._build` "
            "(nvcc, sm_100a); the skeleton path has no CPU fallback"
        )
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - environment specific
        raise DeviceError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rs_abi_version() != ABI_VERSION:
        raise DeviceError("librskel.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def check(status, what):
    if status != 0:
        msg = load().rs_status_string(status).decode()
        raise DeviceError(f"{what} failed: {msg} (status {status})")


def call(name, *args):
    """Invoke ``name`` and raise DeviceError on a non-zero status."""
    status = getattr(load(), name)(*args)
    check(status, name)
