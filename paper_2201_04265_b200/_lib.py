"""ctypes binding of libldpc_b200.so -- argument marshalling only.

Every function here has the name of the C entry point it forwards to
(include/ldpc.h); tensors are passed as raw device pointers, the stream as the
current torch CUDA stream.  There is no fallback: if the library is missing
or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LDPC_LIB_PATH") or os.path.join(_HERE, "libldpc_b200.so")   # override: A/B of builds

# symbols declared in include/ldpc.h (a CPU test checks the two lists agree)
EXPORTED = [
    "ldpc_make_H", "ldpc_code_from_csr", "ldpc_code_from_alist", "ldpc_code_write_alist", "ldpc_make_G",
    "ldpc_make_G_device_workspace_bytes", "ldpc_make_G_device", "ldpc_code_query", "ldpc_code_copy_H",
    "ldpc_code_copy_csr", "ldpc_code_copy_perm", "ldpc_code_copy_P", "ldpc_code_bind_device",
    "ldpc_code_free", "ldpc_status_str", "ldpc_encode", "ldpc_decode_workspace_bytes", "ldpc_decode",
    "ldpc_decode_variant", "ldpc_decode_simulate",
    "ldpc_gen_info", "ldpc_channel", "ldpc_count_errors", "ldpc_partition", "ldpc_debug_phi", "ldpc_debug_psi", "ldpc_debug_check_row",
]


class LdpcError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed: {msg} (status {status})")
        self.status = status


class CodeInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("k", C.c_int32), ("rank", C.c_int32),
                ("nnz", C.c_int32), ("max_row_deg", C.c_int32), ("max_col_deg", C.c_int32),
                ("wc", C.c_int32), ("wr", C.c_int32), ("gallager", C.c_int32),
                ("design_rate", C.c_double), ("device_bytes", C.c_size_t)]


class DecodeOpts(C.Structure):
    _fields_ = [("max_iter", C.c_int32), ("early_term", C.c_int32), ("variant", C.c_int32),
                ("reserved", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
        sig = {
            "ldpc_make_H": [i32, i32, i32, u64, vp],
            "ldpc_code_from_csr": [i32, i32, vp, vp, vp],
            "ldpc_code_from_alist": [C.c_char_p, sz, vp],
            "ldpc_code_write_alist": [vp, C.c_char_p, sz, vp],
            "ldpc_make_G": [vp],
            "ldpc_make_G_device_workspace_bytes": [vp, vp],
            "ldpc_make_G_device": [vp, vp, sz, vp],
            "ldpc_code_query": [vp, vp],
            "ldpc_code_copy_H": [vp, vp],
            "ldpc_code_copy_csr": [vp, vp, vp],
            "ldpc_code_copy_perm": [vp, vp],
            "ldpc_code_copy_P": [vp, vp],
            "ldpc_code_bind_device": [vp, vp, sz, vp],
            "ldpc_encode": [vp, vp, vp, i64, vp],
            "ldpc_decode_workspace_bytes": [vp, i64, vp, vp],
            "ldpc_decode_variant": [vp, i64, vp, vp],
            "ldpc_decode": [vp, vp, i64, vp, vp, vp, vp, vp, vp, sz, vp],
            "ldpc_decode_simulate": [vp, u64, i64, i64, C.c_double, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp],
            "ldpc_gen_info": [u64, i64, i64, i32, vp, vp],
            "ldpc_channel": [vp, u64, i64, i64, vp, C.c_double, vp, vp],
            "ldpc_count_errors": [vp, vp, vp, vp, vp, vp, i64, vp, vp],
            "ldpc_partition": [i64, i32, vp, vp],
            "ldpc_debug_phi": [vp, vp, i64, vp],
            "ldpc_debug_psi": [vp, vp, i64, i32, vp],
            "ldpc_debug_check_row": [vp, vp, i64, i32, i32, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.ldpc_code_free.argtypes = [vp]
        L.ldpc_code_free.restype = None
        L.ldpc_status_str.argtypes = [C.c_int]
        L.ldpc_status_str.restype = C.c_char_p
        _lib = L
    return _lib


def check(fn: str, status: int) -> None:
    if status != 0:
        raise LdpcError(fn, status, lib().ldpc_status_str(status).decode())


def call(fn: str, *args) -> None:
    check(fn, getattr(lib(), fn)(*args))
