"""ctypes binding of libsdfgb200.so (include/sdfgb200.h).

The reference binds its generated library the same way (``ctypes.CDLL`` +
``getattr(lib, code.name)``, codegen.py:866-874).  The library is built
in-tree (``__graft_entry__.build()`` / ``make -C paper_1902_10345_b200/csrc``);
when it is missing the backend fails loudly -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsdfgb200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "sdfgb200.h")

OK, ERR_INVALID, ERR_CUDA, ERR_OOB, ERR_WORKSPACE = 0, 1, 2, 3, 4
PREC_FP32, PREC_NATIVE = 0, 1
CMP = {"<": 0, "<=": 1, ">": 2, ">=": 3, "==": 4, "!=": 5}
QUERY_ORDERED = 0x100  # include/sdfgb200.h: OR into op for input-order survivors
GEMM_B_SPLIT = 1  # include/sdfgb200.h: sdfgb_gemm_f32_ex flag, B already split in the workspace

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_INT = ctypes.c_int
_F64 = ctypes.c_double
_SZ = ctypes.c_size_t

SIGNATURES = {
    "sdfgb_abi_version": (_INT, []),
    "sdfgb_last_error": (ctypes.c_char_p, []),
    "sdfgb_device_count": (_INT, [_P]),
    "sdfgb_host_alloc": (_INT, [_P, _SZ]),
    "sdfgb_host_free": (_INT, [_P]),
    "sdfgb_last_status": (_INT, []),
    "sdfgb_host_threads": (_INT, []),
    "sdfgb_host_convert": (_I64, [_INT, _P, _P, _I64, _I64, _I64]),
    "sdfgb_hist_f32": (_INT, [_P, _I64, _F64, _F64, _P, _I64, _P, _P]),
    "sdfgb_hist_f64": (_INT, [_P, _I64, _F64, _F64, _P, _I64, _P, _P]),
    "sdfgb_hist_i64": (_INT, [_P, _I64, _P, _I64, _P, _P]),
    "sdfgb_query_workspace_bytes": (_SZ, [_I64, _INT]),
    "sdfgb_query_f32": (_INT, [_P, _I64, _INT, _F64, _P, _P, _P, _SZ, _P]),
    "sdfgb_query_f64": (_INT, [_P, _I64, _INT, _F64, _P, _P, _P, _SZ, _P]),
    "sdfgb_spmv_csr_f32": (_INT, [_P, _P, _P, _P, _P, _I64, _P]),
    "sdfgb_spmv_csr_f64": (_INT, [_P, _P, _P, _P, _P, _I64, _P]),
    "sdfgb_nccl_available": (_INT, []),
    "sdfgb_enable_peer_access": (_INT, [_INT]),
    "sdfgb_nccl_unique_id": (_INT, [_P]),
    "sdfgb_nccl_comm_init": (_INT, [_P, _INT, _P, _INT]),
    "sdfgb_nccl_comm_destroy": (_INT, [_P]),
    "sdfgb_hist_mgpu_workspace_bytes": (_SZ, [_I64]),
    "sdfgb_hist_f32_mgpu": (_INT, [_P, _I64, _F64, _F64, _P, _I64, _P, _P, _SZ, _P, _P]),
    "sdfgb_hist_f32_p2p": (_INT, [_P, _I64, _F64, _F64, _P, _P, _INT, _I64, _P]),
    "sdfgb_query_f32_p2p": (_INT, [_P, _I64, _INT, _F64, _P, _P, _P, _SZ, _P]),
    "sdfgb_query_f32_mgpu": (_INT, [_P, _I64, _INT, _F64, _P, _P, _P, _P, _P, _SZ, _P, _P]),
    "sdfgb_spmv_csr_f32_mgpu": (_INT, [_P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P]),
    "sdfgb_jacobi2d_f32_mgpu": (_INT, [_P, _I64, _I64, _I64, _I64, _I64, _F64, _P, _P]),
    "sdfgb_gemm_f32_mgpu": (_INT, [_P, _I64, _P, _I64, _I64, _I64, _P, _P, _P, _P, _SZ, _P, _P, _P]),
    "sdfgb_jacobi2d_f32": (_INT, [_P, _I64, _I64, _F64, _P, _P, _INT, _P]),
    "sdfgb_jacobi2d_f64": (_INT, [_P, _I64, _I64, _F64, _P, _P, _INT, _P]),
    "sdfgb_jacobi2d_step_f32": (_INT, [_P, _P, _I64, _I64, _I64, _I64, _I64, _F64, _P, _P, _INT, _P]),
    "sdfgb_jacobi2d_rect_f32": (_INT, [_P, _I64, _I64, _I64, _F64, _P, _P, _INT, _P]),
    "sdfgb_jacobi2d_block_f32": (_INT, [_P, _P, _I64, _I64, _I64, _F64, _P]),
    "sdfgb_jacobi2d_band_f32": (_INT, [_P, _P, _I64, _I64, _I64, _I64, _I64, _F64, _P]),
    "sdfgb_jacobi2d_band_mirror_f32": (_INT, [_P, _P, _I64, _I64, _I64, _I64, _I64, _F64, _P, _I64, _I64, _P]),
    "sdfgb_flag_signal": (_INT, [_P, _INT, _P]),
    "sdfgb_flag_wait": (_INT, [_P, _INT, _P]),
    "sdfgb_debug_strip_tiles": (_I64, [_I64, _I64, _I64, _I64, _I64, _P, _I64]),
    "sdfgb_probe_gather_f32": (_INT, [_P, _P, _P, _I64, _P, _P]),
    "sdfgb_gemm_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "sdfgb_gemm_f32": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P, _SZ, _P]),
    "sdfgb_gemm_f32_ex": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P, _SZ, _INT, _P]),
    "sdfgb_gemm_f32_simt": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "sdfgb_gemm_f64": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "sdfgb_host_histogram": (_INT, [_P, _P, _I64, _I64, _I64, _F64, _F64, _INT]),
    "sdfgb_host_histogram_i64": (_INT, [_P, _P, _I64, _I64, _I64]),
    "sdfgb_host_query": (_INT, [_P, _P, _P, _P, _I64, _INT, _INT]),
    "sdfgb_host_spmv": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _INT]),
    "sdfgb_host_jacobi2d": (_INT, [_P, _I64, _I64, _F64, _P, _P, _INT, _INT]),
    "sdfgb_host_matmul": (_INT, [_P, _P, _P, _I64, _I64, _I64]),
    "sdfgb_host_matmul_f64": (_INT, [_P, _P, _P, _I64, _I64, _I64]),
}


class BackendUnavailable(RuntimeError):
    """libsdfgb200.so is missing or cannot be loaded (no CPU fallback)."""


class BackendError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_lock = threading.Lock()
_lib = None


def load(path: str = None):
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # SDFGB_LIB: an alternative build of the same library (kernel
        # experiments under tools/); the default is the in-tree build
        path = path or os.environ.get("SDFGB_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise BackendUnavailable(
                f"{path} is not built; run __graft_entry__.build() (make -C paper_1902_10345_b200/csrc)")
        try:
            L = ctypes.CDLL(path)
        except OSError as exc:
            raise BackendUnavailable(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.sdfgb_abi_version() != 1:
            raise BackendUnavailable("libsdfgb200 ABI mismatch")
        _lib = L
        return L


def header_symbols(path: str = HEADER) -> list:
    """Entry points declared in include/sdfgb200.h."""
    import re
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sdfgb_[a-z0-9_]+)\s*\(", text)))


def check(rc: int) -> None:
    """Raise for a non-zero status, mapping codes onto the reference's
    exception vocabulary (see errors.py)."""
    if rc == OK:
        return
    from . import errors
    msg = (load().sdfgb_last_error() or b"").decode(errors="replace")
    if rc == ERR_OOB:
        raise errors.OutOfBoundsError(msg)
    if rc == ERR_INVALID:
        raise errors.CodegenError(msg)
    raise errors.ExecutionError(f"[code {rc}] {msg}")
