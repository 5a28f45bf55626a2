"""ctypes binding of the C ABI (include/rsvd_b200.h) — the only way the
package reaches native code. There is no CPU fallback: if the library is
missing, importing the device layer raises."""

from __future__ import annotations

import ctypes
import os

from .errors import ConvergenceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librsvd_b200.so")

RSVD_OK, RSVD_ERR_INVALID, RSVD_ERR_CONVERGENCE, RSVD_ERR_CUDA = 0, 1, 2, 3
F32, F64 = 0, 1
GEMM_AUTO, GEMM_SIMT, GEMM_TC_3XTF32, GEMM_DMMA, GEMM_SKINNY = 0, 1, 2, 3, 4

_i64, _u64, _int, _dbl, _vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p

_SIGS = {
    "rsvd_last_error": ([], ctypes.c_char_p),
    "rsvd_abi_version": ([], _int),
    "rsvd_sm_count": ([], _int),
    "rsvd_gauss_fill": ([_i64, _u64, _vp, ctypes.POINTER(_u64)], _int),
    "rsvd_gemm_nn": ([_int, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp, _int, _vp, _vp], _int),
    "rsvd_gemm_tn_ws_bytes": ([_int, _i64, _i64, _i64, _int], _i64),
    "rsvd_gemm_tn": ([_int, _int, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp, _vp, _vp,
                      _i64, _int, _vp, _vp], _int),
    "rsvd_oz_planes_bytes": ([_i64, _i64], _i64),
    "rsvd_oz_num_planes": ([], _int),
    "rsvd_oz_prepare": ([_i64, _i64, _vp, _i64, _vp, _vp, _vp], _int),
    "rsvd_oz_prepare_rows": ([_i64, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp], _int),
    "rsvd_oz_gemm_ws_bytes": ([_int, _i64, _i64, _i64], _i64),
    "rsvd_oz_gemm": ([_int, _i64, _i64, _i64, _dbl, _vp, _vp, _vp, _i64, _dbl, _vp, _i64, _vp, _i64, _vp, _vp],
                     _int),
    "rsvd_oz_basis_planes": ([], _int),
    "rsvd_oz_basis_bytes": ([_i64, _i64], _i64),
    "rsvd_oz_basis_ws_bytes": ([_i64], _i64),
    "rsvd_oz_basis_slice": ([_i64, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _vp], _int),
    "rsvd_oz_gemm_planes": ([_int, _i64, _i64, _i64, _dbl, _vp, _int, _i64, _i64, _vp, _int, _vp, _i64, _dbl, _vp,
                             _i64, _vp, _i64, _vp, _vp], _int),
    "rsvd_spmm_csr": ([_int, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _vp, _i64, _vp], _int),
    "rsvd_spmm_nnz_plan": ([_i64, _int, _i64, _vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _vp, _i64, _vp, _vp, _i64, _vp, _vp,
                            _i64, _vp, _vp, _i64, _vp], _int),
    "rsvd_spmm_slab": ([_i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp], _int),
    "rsvd_spmm_csr_plan": ([_int, _int, _i64, _i64, _vp, _vp, _vp, _i64, _dbl, _dbl, _vp, _i64, _i64, _vp, _vp, _vp,
                            _vp, _i64, _vp, _vp, _vp, _i64, _vp], _int),
    "rsvd_csr_transpose": ([_int, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "rsvd_chol_deflate_ws_bytes": ([_i64], _i64),
    "rsvd_chol_deflate": ([_i64, _vp, _i64, _vp, _dbl, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp], _int),
    "rsvd_mask_cols": ([_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp], _int),
    "rsvd_insert_fill": ([_int, _i64, _i64, _vp, _i64, _vp, _vp, _u64, _i64, _i64, _vp, _vp], _int),
    "rsvd_fill_stream": ([_i64, _i64, _u64, _vp, _vp], _int),
    "rsvd_jacobi_ws_bytes": ([_i64], _i64),
    "rsvd_jacobi_sweeps": ([_i64, _vp, _i64, _vp, _i64, _dbl, _int, _vp, _vp, _vp, _i64, _vp], _int),
    "rsvd_eig_select": ([_i64, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp], _int),
    "rsvd_syev_topk_ws_bytes": ([_i64, _i64], _i64),
    "rsvd_syev_topk": ([_i64, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp], _int),
    "rsvd_colreduce_ws_bytes": ([_i64, _i64], _i64),
    "rsvd_colreduce": ([_int, _int, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp], _int),
    "rsvd_canonicalize_signs": ([_int, _i64, _i64, _vp, _i64, _vp, _i64, _vp], _int),
    "rsvd_col_absargmax": ([_int, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _vp], _int),
    "rsvd_flip_by_sign": ([_int, _i64, _i64, _vp, _i64, _vp, _vp], _int),
    "rsvd_split_planes_bytes": ([_i64, _i64], _i64),
    "rsvd_split_planes": ([_i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp], _int),
    "rsvd_gemm_nn_f32_emit": ([_i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp, _vp, _i64, _vp, _vp,
                               _vp], _int),
    "rsvd_gemm_tn_f32_planes": ([_int, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp, _vp, _vp,
                                 _i64, _vp, _vp], _int),
    "rsvd_gemm_tn_f32_planes_ok": ([_i64, _i64, _i64, _vp, _i64], _int),
    "rsvd_convert": ([_int, _int, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp], _int),
    "rsvd_gather_rows": ([_int, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp], _int),
    "rsvd_scatter_rows": ([_int, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp], _int),
    "rsvd_sqrt_clip": ([_i64, _vp, _vp, _vp], _int),
    "rsvd_ortho_error": ([_i64, _vp, _i64, _vp, _vp], _int),
    "rsvd_cond_begin": ([_vp, _vp, _vp, _vp], _int),
    "rsvd_handle_create": ([_int, _vp], _int),
    "rsvd_handle_destroy": ([_vp], _int),
    "rsvd_handle_device": ([_vp, _vp], _int),
    "rsvd_handle_world": ([_vp, _vp, _vp], _int),
    "rsvd_handle_set_comm": ([_vp, _vp, _int, _int], _int),
    "rsvd_nccl_unique_id": ([_vp, _i64], _int),
    "rsvd_handle_init_comm": ([_vp, _vp, _i64, _int, _int], _int),
    "rsvd_handle_allreduce_sum": ([_vp, _vp, _i64, _int, _vp], _int),
    "rsvd_cond_end": ([_vp], _int),
}

_lib = None


def load():
    """Load librsvd_b200.so (building it first only if sources are present and
    it is missing). Raises ImportError when the native library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        try:
            from .build import build

            build()
        except Exception as exc:  # pragma: no cover - depends on toolchain
            raise ImportError(f"librsvd_b200.so is not built and could not be built: {exc}") from exc
    L = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def exported_symbols():
    return list(_SIGS)


def last_error():
    return load().rsvd_last_error().decode(errors="replace")


def check(status, what=""):
    if status == RSVD_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == RSVD_ERR_INVALID:
        raise ValueError(msg)
    if status == RSVD_ERR_CONVERGENCE:
        raise ConvergenceError(msg)
    raise RuntimeError(msg)
