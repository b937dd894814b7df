"""ctypes binding of libfdmd.so (C ABI declared in include/fdmd.h).

The library is built in-tree (`python -c "import __graft_entry__ as g; g.build()"`
or `make -C paper_2502_05339_b200/csrc`). There is no fallback: if the shared
object is missing every compute entry point raises `NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConvergenceError, FlowDmdError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfdmd.so")

FDMD_OK = 0
FDMD_ERR_INVALID = -1
FDMD_ERR_CUDA = -2
FDMD_ERR_SOLVER = -3
FDMD_ERR_WORKSPACE = -4

F32, F64 = 0, 1
ROW, COL = 0, 1

# name -> (restype, argtypes); must match include/fdmd.h exactly
_c = ctypes
_vp, _i, _i64, _sz, _d, _u64 = _c.c_void_p, _c.c_int, _c.c_int64, _c.c_size_t, _c.c_double, _c.c_uint64
SIGNATURES = {
    "fdmd_version": (_i, []),
    "fdmd_last_error": (_c.c_char_p, []),
    "fdmd_device_info": (_i, [_i, _c.POINTER(_i), _c.POINTER(_i), _c.POINTER(_i)]),
    "fdmd_tall_gemm_workspace": (_sz, [_i64, _i]),
    "fdmd_tall_gemm": (_i, [_vp, _i, _i, _i64, _vp, _i64, _vp, _i, _i, _i64, _i64, _i, _i, _i,
                            _vp, _i64, _vp, _sz, _vp]),
    "fdmd_tall_gemm_planes": (_i, [_vp, _i, _i64, _vp, _i64, _vp, _vp, _i64, _d, _i64, _i, _i, _i, _vp]),
    "fdmd_tall_gram_bordered_workspace": (_sz, [_i64, _i]),
    "fdmd_tall_gram_bordered": (_i, [_vp, _i, _i64, _vp, _i64, _d, _i64, _i, _vp, _sz, _vp]),
    "fdmd_tc_decode_pairstats": (_i, [_vp, _vp, _i64, _i64, _i, _vp, _vp, _i, _i, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "fdmd_svd_small": (_i, [_vp, _i64, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "fdmd_gram_plan_info": (_i, [_i64, _i, _i, _i, _i, _vp, _vp, _i]),
    "fdmd_tall_tdot_workspace": (_sz, [_i64, _i]),
    "fdmd_tall_tdot": (_i, [_vp, _i, _i64, _vp, _i64, _i64, _i, _vp, _d, _vp, _sz, _vp]),
    "fdmd_tall_gram_workspace": (_sz, [_i64, _i, _i]),
    "fdmd_tall_gram": (_i, [_vp, _i, _i, _i64, _vp, _i, _i, _i64, _vp, _i64, _d, _i64, _i, _i, _i,
                            _vp, _sz, _vp]),
    "fdmd_decode": (_i, [_vp, _i, _i64, _vp, _i, _vp, _i64, _i64, _i, _i, _vp]),
    "fdmd_colmajor_dot_workspace": (_sz, [_i64, _i, _i]),
    "fdmd_colmajor_dot": (_i, [_vp, _i, _i64, _vp, _i, _i64, _i64, _i, _i, _vp, _vp, _sz, _vp]),
    "fdmd_table_apply": (_i, [_vp, _i, _i64, _vp, _vp, _vp, _vp, _i, _i64, _i64, _i, _vp]),
    "fdmd_table_apply_inplace": (_i, [_vp, _i, _i64, _i, _vp, _vp, _vp, _i, _i64, _vp]),
    "fdmd_residual_workspace": (_sz, [_i64]),
    "fdmd_residual": (_i, [_vp, _i, _i64, _vp, _i, _i64, _vp, _i, _i, _i64, _vp, _vp, _sz, _vp]),
    "fdmd_geev": (_i, [_i, _vp, _vp, _vp, _vp]),
    "fdmd_copy2d": (_i, [_vp, _i64, _vp, _i64, _i64, _i64, _i, _vp]),
    "fdmd_dmma_peak": (_i, [_d, _c.POINTER(_d)]),
    "fdmd_split_basis": (_i, [_vp, _i64, _i64, _i, _c.c_float, _vp, _vp, _i64, _vp]),
    "fdmd_split_coef": (_i, [_vp, _i, _i, _i, _c.c_float, _vp, _vp, _i, _vp, _vp]),
    "fdmd_split_rows_f64": (_i, [_vp, _i64, _i64, _i, _d, _vp, _vp, _i64, _vp]),
    "fdmd_split_rows": (_i, [_vp, _i, _i64, _i64, _i, _d, _vp, _vp, _i64, _vp]),
    "fdmd_pair_stats_workspace": (_sz, [_i64, _i]),
    "fdmd_pair_stats": (_i, [_vp, _i64, _i64, _i, _i64, _vp, _vp, _sz, _vp]),
    "fdmd_tc_decode": (_i, [_vp, _vp, _i64, _i64, _i, _vp, _vp, _i, _i, _vp, _vp, _i64, _vp]),
    "fdmd_tc_decode_ex": (_i, [_vp, _vp, _i64, _i64, _i, _vp, _vp, _i, _i, _vp, _vp, _i64, _i, _vp]),
    "fdmd_tc_decode_planes": (_i, [_vp, _vp, _i64, _i64, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _i64, _c.c_float, _i,
                                   _vp]),
    "fdmd_mac_decode": (_i, [_vp, _i, _i64, _i, _vp, _i, _i, _i, _vp, _vp]),
    "fdmd_mac_advect": (_i, [_vp, _i, _i, _i, _d, _d, _vp, _vp, _vp]),
    "fdmd_mac_inject": (_i, [_vp, _i, _i, _i, _i, _i64, _i64, _vp, _vp]),
    "fdmd_mac_project": (_i, [_vp, _vp, _i, _i, _i, _d, _vp, _vp]),
    "fdmd_sol_mask": (_i, [_vp, _i, _i, _vp, _i, _vp]),
    "fdmd_sol_advect": (_i, [_vp, _vp, _i, _i, _i, _d, _d, _i, _vp, _vp, _vp]),
    "fdmd_sol_emit": (_i, [_vp, _vp, _i, _i, _d, _d, _d, _d, _d, _d, _vp]),
    "fdmd_sol_buoyancy": (_i, [_vp, _vp, _vp, _i, _i, _d, _d, _d, _vp]),
    "fdmd_sol_vorticity": (_i, [_vp, _i, _i, _d, _d, _d, _vp, _vp]),
    "fdmd_sol_reduce": (_i, [_vp, _vp, _vp, _i64, _i, _vp, _vp, _vp]),
    "fdmd_sol_rhs": (_i, [_vp, _i, _i, _d, _vp, _i, _d, _vp, _vp, _vp, _vp]),
    "fdmd_sol_poisson": (_i, [_vp, _i, _i, _d, _vp, _i, _vp, _vp]),
    "fdmd_sol_cg_step": (_i, [_vp, _vp, _vp, _vp, _d, _i64, _vp]),
    "fdmd_sol_cg_dir": (_i, [_vp, _vp, _d, _i64, _vp]),
    "fdmd_sol_cg_single": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _d, _vp, _i, _d, _i, _vp, _vp]),
    "fdmd_sol_pressure_apply": (_i, [_vp, _vp, _i, _i, _d, _vp, _i, _vp]),
    "fdmd_rsvd": (_i, [_vp, _i, _i64, _i64, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i64, _vp]),
    "fdmd_ctx_create": (_i, [_i, _i, _c.POINTER(_vp)]),
    "fdmd_ctx_destroy": (_i, [_vp]),
    "fdmd_mat_upload": (_i, [_vp, _vp, _i, _i64, _i64, _i64, _c.POINTER(_vp)]),
    "fdmd_mat_free": (_i, [_vp]),
    "fdmd_dmd_fit": (_i, [_vp, _vp, _d, _i, _i, _i, _vp, _i, _i, _vp, _vp, _vp, _vp, _c.POINTER(_vp)]),
    "fdmd_dmdc_fit": (_i, [_vp, _vp, _vp, _i, _d, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _c.POINTER(_vp)]),
    "fdmd_model_info": (_i, [_vp, _c.POINTER(_i64), _c.POINTER(_i), _c.POINTER(_d), _c.POINTER(_i)]),
    "fdmd_model_history": (_i, [_vp, _vp, _i]),
    "fdmd_model_phi_to_host": (_i, [_vp, _vp, _i64, _i64, _vp]),
    "fdmd_encode": (_i, [_vp, _vp, _vp, _vp]),
    "fdmd_model_decode": (_i, [_vp, _vp, _vp, _i, _vp]),
    "fdmd_model_free": (_i, [_vp]),
    "fdmd_synth3d": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _d, _u64, _i64, _i64, _vp, _i, _i64, _vp]),
}


class NativeLibraryError(FlowDmdError, RuntimeError):
    """libfdmd.so is missing or failed to load; there is no CPU fallback."""


class DeviceError(FlowDmdError, RuntimeError):
    """A CUDA runtime failure inside libfdmd."""


_lock = threading.Lock()
_lib = None


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeLibraryError(
                        f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
                try:
                    handle = ctypes.CDLL(LIB_PATH)
                except OSError as exc:
                    raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def check(rc: int, what: str = ""):
    if rc == FDMD_OK:
        return
    msg = lib().fdmd_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == FDMD_ERR_INVALID:
        raise ValueError(text)
    if rc == FDMD_ERR_SOLVER:
        raise ConvergenceError(text)
    raise DeviceError(text)


def call(name: str, *args):
    rc = getattr(lib(), name)(*args)
    check(rc, name)
