"""paper_2201_04265_b200 -- B200-native batched Sum-Product LDPC decoding.

Thin Python binding over the C ABI of ``libldpc_b200.so`` (include/ldpc.h).
Functions keep the C names; they marshal torch tensors to raw pointers and
pass the current CUDA stream.  Every step of the hot path runs in the
library's CUDA kernels; there is no CPU fallback.  PyTorch is used for device
memory and streams only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import CodeInfo, DecodeOpts, LdpcError, call, lib

__all__ = [
    "Code", "LdpcError", "ldpc_make_H", "ldpc_code_from_csr", "ldpc_make_G", "ldpc_code_query",
    "ldpc_code_copy_H", "ldpc_code_copy_csr", "ldpc_code_copy_perm", "ldpc_code_copy_P",
    "ldpc_code_bind_device", "ldpc_encode", "ldpc_decode_workspace_bytes", "ldpc_decode",
    "ldpc_gen_info", "ldpc_channel", "ldpc_count_errors", "ldpc_partition", "ldpc_debug_phi", "ldpc_debug_psi",
    "ldpc_debug_check_row", "words",
]


def words(bits: int) -> int:
    """uint32 words holding `bits` packed bits."""
    return (int(bits) + 31) // 32


def _ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())


def _stream(stream=None) -> C.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _np(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


class Code:
    """Owns an ``ldpc_code*`` (host) and, once bound, its device image (a torch
    uint8 buffer that must outlive every launch using the code)."""

    def __init__(self, handle: C.c_void_p):
        self.handle = handle
        self.device_buffer = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().ldpc_code_free(h)
            except Exception:
                pass
            self.handle = None

    @property
    def info(self) -> CodeInfo:
        return ldpc_code_query(self)

    def __getattr__(self, name):
        if name in ("n", "m", "k", "rank", "nnz", "max_row_deg", "max_col_deg", "wc", "wr", "design_rate"):
            return getattr(ldpc_code_query(self), name)
        raise AttributeError(name)


# ---------------------------------------------------------------- codes
def ldpc_make_H(n: int, wc: int, wr: int, seed: int) -> Code:
    h = C.c_void_p()
    call("ldpc_make_H", int(n), int(wc), int(wr), C.c_uint64(int(seed)), C.byref(h))
    return Code(h)


def ldpc_code_from_csr(m: int, n: int, row_ptr, col_idx) -> Code:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    if ci.size == 0:
        ci = np.zeros(1, np.int32)
    h = C.c_void_p()
    call("ldpc_code_from_csr", int(m), int(n), _np(rp), _np(ci), C.byref(h))
    return Code(h)


def ldpc_code_from_alist(text) -> Code:
    """MacKay alist text (str or bytes) -> code."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    call("ldpc_code_from_alist", C.c_char_p(b), C.c_size_t(len(b)), C.byref(h))
    return Code(h)


def ldpc_code_write_alist(code: Code) -> str:
    """Code -> MacKay alist text."""
    n = C.c_size_t(0)
    call("ldpc_code_write_alist", code.handle, None, C.c_size_t(0), C.byref(n))
    buf = C.create_string_buffer(n.value + 1)
    call("ldpc_code_write_alist", code.handle, buf, C.c_size_t(n.value + 1), C.byref(n))
    return buf.raw[:n.value].decode()


def ldpc_make_G(code: Code) -> Code:
    call("ldpc_make_G", code.handle)
    return code


def ldpc_make_G_device(code: Code, device=None, stream=None) -> Code:
    """make_G on the GPU (same result as ldpc_make_G); workspace from torch."""
    import torch
    n = C.c_size_t(0)
    call("ldpc_make_G_device_workspace_bytes", code.handle, C.byref(n))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = torch.empty(max(int(n.value), 256), dtype=torch.uint8, device=dev)
    call("ldpc_make_G_device", code.handle, _ptr(ws), C.c_size_t(ws.numel()), _stream(stream))
    return code


def ldpc_code_query(code: Code) -> CodeInfo:
    info = CodeInfo()
    call("ldpc_code_query", code.handle, C.byref(info))
    return info


def ldpc_code_copy_H(code: Code) -> np.ndarray:
    i = ldpc_code_query(code)
    out = np.zeros((i.m, i.n), dtype=np.uint8)
    call("ldpc_code_copy_H", code.handle, _np(out))
    return out


def ldpc_code_copy_csr(code: Code):
    i = ldpc_code_query(code)
    rp = np.zeros(i.m + 1, dtype=np.int32)
    ci = np.zeros(max(i.nnz, 1), dtype=np.int32)
    call("ldpc_code_copy_csr", code.handle, _np(rp), _np(ci))
    return rp, ci[: i.nnz]


def ldpc_code_copy_perm(code: Code) -> np.ndarray:
    i = ldpc_code_query(code)
    out = np.zeros(i.n, dtype=np.int32)
    call("ldpc_code_copy_perm", code.handle, _np(out))
    return out


def ldpc_code_copy_P(code: Code) -> np.ndarray:
    """P packed by parity column: uint32 [(n-k), ceil(k/32)]."""
    i = ldpc_code_query(code)
    out = np.zeros((i.n - i.k, words(i.k)), dtype=np.uint32)
    if out.size:
        call("ldpc_code_copy_P", code.handle, _np(out))
    return out


def ldpc_code_bind_device(code: Code, device="cuda", stream=None) -> Code:
    import torch
    nbytes = int(ldpc_code_query(code).device_bytes)
    buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % 256
    view = buf[off: off + nbytes]
    call("ldpc_code_bind_device", code.handle, C.c_void_p(view.data_ptr()), C.c_size_t(nbytes), _stream(stream))
    code.device_buffer = buf     # keeps the image alive as long as the code
    return code


# ---------------------------------------------------------------- hot path
def ldpc_encode(code: Code, d_info, d_cw, frames: int, stream=None) -> None:
    call("ldpc_encode", code.handle, _ptr(d_info), _ptr(d_cw), int(frames), _stream(stream))


def _opts(max_iter: int, early_term: bool, variant: int) -> DecodeOpts:
    return DecodeOpts(int(max_iter), int(bool(early_term)), int(variant), 0)


def ldpc_decode_variant(code: Code, frames: int, max_iter: int = 50, early_term: bool = False,
                        variant: int = 0) -> int:
    o = _opts(max_iter, early_term, variant)
    out = C.c_int32(0)
    call("ldpc_decode_variant", code.handle, int(frames), C.byref(o), C.byref(out))
    return int(out.value)


def ldpc_decode_workspace_bytes(code: Code, frames: int, max_iter: int = 50, early_term: bool = False,
                                variant: int = 0) -> int:
    o = _opts(max_iter, early_term, variant)
    out = C.c_size_t(0)
    call("ldpc_decode_workspace_bytes", code.handle, int(frames), C.byref(o), C.byref(out))
    return int(out.value)


def ldpc_decode(code: Code, d_llr, frames: int, d_bits, d_syndrome_ok, d_iters, d_posterior=None,
                d_ws=None, max_iter: int = 50, early_term: bool = False, variant: int = 0,
                stream=None) -> None:
    o = _opts(max_iter, early_term, variant)
    ws_bytes = 0 if d_ws is None else d_ws.numel() * d_ws.element_size()
    call("ldpc_decode", code.handle, _ptr(d_llr), int(frames), C.byref(o), _ptr(d_bits),
         _ptr(d_syndrome_ok), _ptr(d_iters), _ptr(d_posterior), _ptr(d_ws), C.c_size_t(ws_bytes),
         _stream(stream))


def ldpc_decode_simulate(code: Code, seed: int, frame0: int, frames: int, sigma: float, d_info, d_cw,
                         d_bits, d_syndrome_ok, d_iters, d_counters6, d_ws=None, max_iter: int = 50,
                         early_term: bool = False, variant: int = 0, stream=None) -> None:
    """Fused channel -> decode -> count (ldpc.h); counters are ADDED to d_counters6."""
    o = _opts(max_iter, early_term, variant)
    ws_bytes = 0 if d_ws is None else d_ws.numel() * d_ws.element_size()
    call("ldpc_decode_simulate", code.handle, C.c_uint64(int(seed)), int(frame0), int(frames), float(sigma),
         _ptr(d_info), _ptr(d_cw), C.byref(o), _ptr(d_bits), _ptr(d_syndrome_ok), _ptr(d_iters),
         _ptr(d_counters6), _ptr(d_ws), C.c_size_t(ws_bytes), _stream(stream))


def ldpc_gen_info(seed: int, frame0: int, frames: int, k: int, d_info, stream=None) -> None:
    call("ldpc_gen_info", C.c_uint64(int(seed)), int(frame0), int(frames), int(k), _ptr(d_info),
         _stream(stream))


def ldpc_channel(code: Code, seed: int, frame0: int, frames: int, d_cw, sigma: float, d_llr,
                 stream=None) -> None:
    call("ldpc_channel", code.handle, C.c_uint64(int(seed)), int(frame0), int(frames), _ptr(d_cw),
         float(sigma), _ptr(d_llr), _stream(stream))


def ldpc_count_errors(code: Code, d_info, d_bits, d_cw, d_syndrome_ok, d_iters, frames: int,
                      d_counters6, stream=None) -> None:
    call("ldpc_count_errors", code.handle, _ptr(d_info), _ptr(d_bits), _ptr(d_cw),
         _ptr(d_syndrome_ok), _ptr(d_iters), int(frames), _ptr(d_counters6), _stream(stream))


def ldpc_partition(l: int, nproc: int):
    counts = np.zeros(nproc, dtype=np.int64)
    displs = np.zeros(nproc, dtype=np.int64)
    call("ldpc_partition", int(l), int(nproc), _np(counts), _np(displs))
    return counts, displs


def ldpc_debug_phi(d_x, d_y, count: int, stream=None) -> None:
    call("ldpc_debug_phi", _ptr(d_x), _ptr(d_y), int(count), _stream(stream))


def ldpc_debug_psi(d_y, d_out, count: int, tier: int = 0, stream=None) -> None:
    call("ldpc_debug_psi", _ptr(d_y), _ptr(d_out), int(count), int(tier), _stream(stream))


def ldpc_debug_check_row(d_x, d_e, rows: int, degree: int, vote: bool = True, stream=None) -> None:
    call("ldpc_debug_check_row", _ptr(d_x), _ptr(d_e), int(rows), int(degree), int(bool(vote)), _stream(stream))


# ---------------------------------------------------------------- convenience
@dataclass
class DecodeOut:
    bits: "object"
    syndrome_ok: "object"
    iters: "object"
    posterior: "object"
    workspace: "object" = None     # kept alive with the outputs (the launch may still be running)


def decode(code: Code, llr, max_iter: int = 50, early_term: bool = False, posterior: bool = False,
           variant: int = 0, stream=None) -> DecodeOut:
    """Allocate outputs (torch, on llr's device) and run ldpc_decode."""
    import torch
    frames = llr.shape[0]
    n = ldpc_code_query(code).n
    dev = llr.device
    bits = torch.empty((frames, words(n)), dtype=torch.int32, device=dev)
    syn = torch.empty(frames, dtype=torch.uint8, device=dev)
    its = torch.empty(frames, dtype=torch.int32, device=dev)
    post = torch.empty((frames, n), dtype=torch.float32, device=dev) if posterior else None
    wsb = ldpc_decode_workspace_bytes(code, frames, max_iter, early_term, variant)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev) if wsb else None
    ldpc_decode(code, llr, frames, bits, syn, its, post, ws, max_iter, early_term, variant, stream)
    if ws is not None and stream is not None:
        ws.record_stream(stream)     # the caching allocator must not reuse it before `stream` finishes
    return DecodeOut(bits, syn, its, post, ws)
