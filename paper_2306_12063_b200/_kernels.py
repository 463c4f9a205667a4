"""Drop-in for the reference's compiled decode loops (`qcldpc._kernels`).

`decode_batch_f32` / `decode_batch_i16` keep the reference's exact ten-argument
signature (`/root/reference/pkg/src/qcldpc/_kernels.py:17-19, 103-105`):

    (row_ptr, col_idx, mb, z, llrs, max_iters, early_term, hard, iters, conv)

with caller-owned numpy outputs written in place.  Instead of numba loops they
call libqcb200's `qc_decode_batch_{f32,i16}_host`, which recovers the
circulant shift table from the CSR, uploads the LLR block, runs the sm_100a
decoder and copies hard decisions / iteration counts / convergence flags back.
ctypes releases the GIL for the duration of the call, matching the
reference's `nogil=True`.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def _run(fn_name: str, dtype, row_ptr, col_idx, mb, z, llrs, max_iters, early_term,
         hard, iters, conv) -> None:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    vals = np.ascontiguousarray(llrs, dtype=dtype)
    if vals.ndim != 2:
        raise ValueError("llrs must be a (W, N) block")
    w, n = vals.shape
    for name, arr, dt, shape in (("hard", hard, np.uint8, (w, n)), ("iters", iters, np.int32, (w,)),
                                 ("conv", conv, np.uint8, (w,))):
        if not (isinstance(arr, np.ndarray) and arr.dtype == dt and arr.shape == shape
                and arr.flags.c_contiguous and arr.flags.writeable):
            raise ValueError(f"{name} must be a writeable C-contiguous {np.dtype(dt).name} array of shape {shape}")
    fn = getattr(_lib.lib(), fn_name)
    _lib.check(fn(rp.ctypes.data, rp.shape[0], ci.ctypes.data, ci.shape[0], int(mb), int(z),
                  vals.ctypes.data, w, n, int(max_iters), int(early_term),
                  hard.ctypes.data, iters.ctypes.data, conv.ctypes.data), fn_name)


def decode_batch_f32(row_ptr, col_idx, mb, z, llrs, max_iters, early_term, hard, iters, conv):
    _run("qc_decode_batch_f32_host", np.float32, row_ptr, col_idx, mb, z, llrs, max_iters,
         early_term, hard, iters, conv)


def decode_batch_i16(row_ptr, col_idx, mb, z, llrs, max_iters, early_term, hard, iters, conv):
    _run("qc_decode_batch_i16_host", np.int16, row_ptr, col_idx, mb, z, llrs, max_iters,
         early_term, hard, iters, conv)
