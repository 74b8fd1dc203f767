"""ctypes declarations of the libfls C ABI (include/fls.h).  Argument marshalling only.

Loading fails loudly (FlsError / OSError) when libfls.so is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# FLS_LIB selects a tuning-variant build (tools/variant_sweep.sh); default = the product build
LIB_PATH = os.environ.get("FLS_LIB") or os.path.join(HERE, "libfls.so")
HEADER = os.path.join(ROOT, "include", "fls.h")

FLS_MAX_DIM = 8
FLS_MAX_TERMS = 64
FLS_MAX_FIELDS = 4
FLS_COL_MAJOR = 0
FLS_ROW_MAJOR = 1
FLS_IPC_HANDLE_BYTES = 64
FLS_COMM_ID_BYTES = 128
FLS_TSQR_AUTO = 0
FLS_TSQR_P2P = 1
FLS_TSQR_NCCL = 2

STATUS = {0: "FLS_OK", 1: "FLS_EINVAL", 2: "FLS_ENOMEM", 3: "FLS_ECUDA", 4: "FLS_ECUSOLVER",
          5: "FLS_ENCCL", 6: "FLS_ENONFINITE", 7: "FLS_ERANK", 8: "FLS_EUNSUPPORTED"}


class FlsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class fls_term(C.Structure):
    _fields_ = [("alpha", C.c_int32 * FLS_MAX_DIM), ("coef", C.c_double), ("field", C.c_int32)]


class fls_operator(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n_terms", C.c_int32), ("terms", C.POINTER(fls_term))]


class fls_block(C.Structure):
    _fields_ = [("X", C.c_void_p), ("n_points", C.c_int64), ("op", C.POINTER(fls_operator)),
                ("coef_fields", C.c_void_p), ("n_fields", C.c_int32), ("weight", C.c_double),
                ("values", C.c_void_p)]


FLS_NL_POLY = 1
FLS_NL_EXP = 2
FLS_NL_UDU = 3


class fls_nonlinearity(C.Structure):
    _fields_ = [("kind", C.c_int32), ("degree", C.c_int32), ("a", C.c_double * 8)]


# int32 allgather(void *user, const void *send, void *recv, int64 bytes)
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)


class fls_host_coll(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", HOST_ALLGATHER)]


_SIGS = {
    "fls_last_error": (C.c_char_p, []),
    "fls_status_string": (C.c_char_p, [C.c_int]),
    "fls_api_version": (C.c_int, []),
    "fls_ctx_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "fls_ctx_destroy": (C.c_int, [C.c_void_p]),
    "fls_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fls_sync": (C.c_int, [C.c_void_p]),
    "fls_ctx_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "fls_ctx_timing_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "fls_features": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64,
                               C.c_void_p, C.c_void_p]),
    "fls_assemble": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                               C.POINTER(fls_block), C.c_int32, C.c_int64, C.c_int64, C.c_void_p,
                               C.c_int64, C.c_int32, C.c_void_p]),
    "fls_features_assemble": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64,
                                        C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(fls_block),
                                        C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                        C.c_int32, C.c_void_p]),
    "fls_features_blocks": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_uint64, C.c_void_p, C.c_void_p]),
    "fls_qr_factor": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                C.POINTER(C.c_void_p)]),
    "fls_qr_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                               C.c_int64]),
    "fls_qr_destroy": (C.c_int, [C.c_void_p]),
    "fls_nl_residual": (C.c_int, [C.c_void_p, C.POINTER(fls_nonlinearity), C.c_int64, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    "fls_sample_box": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_uint64, C.c_uint64, C.c_void_p]),
    "fls_sample_faces": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_void_p,
                                   C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "fls_features_transform": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    "fls_bandwidth_grad": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                     C.c_int64, C.c_int32, C.POINTER(fls_block), C.c_int32,
                                     C.c_void_p, C.c_void_p]),
    "fls_nl_residual2": (C.c_int, [C.c_void_p, C.POINTER(fls_nonlinearity), C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "fls_axpy": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "fls_assemble_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64,
                                    C.c_int32, C.POINTER(fls_block), C.c_int32, C.c_int64,
                                    C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]),
    "fls_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                            C.c_void_p, C.POINTER(C.c_double)]),
    "fls_solve_mu": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                               C.c_void_p, C.POINTER(C.c_double)]),
    "fls_comm_unique_id": (C.c_int, [C.c_void_p]),
    "fls_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    "fls_comm_init_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(fls_host_coll)]),
    "fls_comm_destroy": (C.c_int, [C.c_void_p]),
    "fls_comm_config": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "fls_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32)]),
    "fls_solve_stacked": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_double, C.c_void_p, C.POINTER(C.c_double)]),
    "fls_geqrf": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]),
    "fls_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "fls_ipc_open": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "fls_ipc_close": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fls_qr_r": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                           C.c_int64]),
    "fls_frob2": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                            C.POINTER(C.c_double)]),
    "fls_eval_block": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                                 C.c_void_p, C.POINTER(fls_block), C.c_void_p]),
    "fls_eval": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                           C.c_void_p, C.POINTER(fls_operator), C.c_void_p, C.c_int64, C.c_void_p]),
}

_lib = None


def header_symbols() -> list:
    """every function declared in include/fls.h"""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fls_[a-z0-9_]+)\s*\(", txt)))


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FlsError(3, f"libfls.so not built at {LIB_PATH}; run "
                              "`python -m paper_2602_10541_b200.build` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def check(status: int):
    if status != 0:
        msg = load().fls_last_error()
        raise FlsError(status, msg.decode() if msg else "")
