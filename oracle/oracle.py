"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle (qc_oracle.c).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg, where it is the checker or the timed CPU
baseline, never the product.  The product package (paper_2306_12063_b200)
does not import this module.

`decode_batch(h, llrs, max_iters, early_term, workers)` mirrors the reference's
`_kernels.decode_batch_f32 / _i16` (`/root/reference/pkg/src/qcldpc/_kernels.py:17-186`)
plus the contiguous worker chunking of `decoder.decode_block`
(`decoder.py:217-258`); `encode_packed(mm, info_bytes, word_bits)` mirrors
`encoder.encode_packed` (`encoder.py:166-199`).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None


def build(force: bool = False) -> Path:
    src = _HERE / "qc_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(_LIB_PATH))
        P = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        for name in ("oracle_decode_f32", "oracle_decode_i16"):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = [P, P, i32, i32, i32, i32, P, i64, i32, i32, P, P, P, P, i32]
        L.oracle_encode_packed.restype = C.c_int
        L.oracle_encode_packed.argtypes = [P, i32, i32, i32, i32, i32, i32, P, i64, P]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def decode_batch(h, llrs: np.ndarray, max_iters: int = 10, early_term: bool = True,
                 workers: int | None = None, want_post: bool = False):
    """Decode a (W, N) float32 or int16 block; returns (hard u8, iters i32, conv u8[, post])."""
    llrs = np.ascontiguousarray(llrs)
    if llrs.dtype not in (np.float32, np.int16) or llrs.ndim != 2 or llrs.shape[1] != h.n:
        raise ValueError("llrs must be (W, N) float32 or int16")
    w = llrs.shape[0]
    hard = np.empty((w, h.n), np.uint8)
    iters = np.empty(w, np.int32)
    conv = np.empty(w, np.uint8)
    post = np.empty_like(llrs) if want_post else None
    rp = np.ascontiguousarray(h.row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(h.row_cols, dtype=np.int32)
    fn = lib().oracle_decode_f32 if llrs.dtype == np.float32 else lib().oracle_decode_i16
    rc = fn(_ptr(rp), _ptr(ci), h.m, h.n, h.m // h.z, h.z, _ptr(llrs), w, int(max_iters),
            1 if early_term else 0, _ptr(hard), _ptr(iters), _ptr(conv), _ptr(post),
            int(workers or os.cpu_count() or 1))
    if rc != 0:
        raise RuntimeError(f"oracle decode failed: {rc}")
    return (hard, iters, conv, post) if want_post else (hard, iters, conv)


def find_y(mm) -> tuple[int, int]:
    hb = mm.entries[:, mm.kb]
    inner = [i for i in range(1, mm.mb - 1) if hb[i] >= 0]
    if len(inner) != 1:
        raise ValueError("h_b column needs exactly one interior entry")
    return inner[0], int(hb[inner[0]])


def encode_packed(mm, info_bytes: np.ndarray, word_bits: int | None = None) -> np.ndarray:
    """(W, K/8) MSB-first info bytes -> (W, N/8) codeword bytes."""
    info = np.ascontiguousarray(info_bytes, dtype=np.uint8)
    if info.ndim == 1:
        info = info[None]
    if word_bits is None:
        word_bits = next((wb for wb in (32, 16, 8) if mm.z % wb == 0), 8)
    y, hb = find_y(mm)
    out = np.empty((info.shape[0], mm.n // 8), np.uint8)
    ent = np.ascontiguousarray(mm.entries, dtype=np.int32)
    rc = lib().oracle_encode_packed(_ptr(ent), mm.mb, mm.nb, mm.z, word_bits, y, hb,
                                    _ptr(info), info.shape[0], _ptr(out))
    if rc != 0:
        raise ValueError("oracle encode_packed rejected the code (z % 8 or word size)")
    return out
