"""ctypes binding of libqcb200.so (the C ABI in include/qcb200.h).

This is the only way the package reaches the device: there is no CPU
fallback.  If the library is missing or fails to load, every codec call
raises `NativeLibraryError` loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (CodecError, DeviceError, MalformedHb, NativeLibraryError,
                     SizeMismatch, UnsupportedCode, UnsupportedZ)

LIB_PATH = Path(os.environ.get("QCB_LIB") or Path(__file__).resolve().parent / "libqcb200.so")

QC_OK = 0
QC_EINVAL = -1
QC_EUNSUPPORTED = -2
QC_ENOMEM = -3
QC_EMALFORMED = -4
QC_EUNALIGNED = -5

_lock = threading.Lock()
_lib = None

P = C.c_void_p
i32, i64 = C.c_int32, C.c_int64

# (name, restype, argtypes) for every symbol declared in include/qcb200.h
SIGNATURES = {
    "qc_version": (C.c_int, []),
    "qc_last_error": (C.c_char_p, []),
    "qc_code_create": (C.c_int, [i32, i32, i32, P, P]),
    "qc_code_from_csr": (C.c_int, [P, i64, P, i64, i32, i32, i32, P]),
    "qc_code_destroy": (C.c_int, [P]),
    "qc_code_info": (C.c_int, [P, P, P, P, P, P, P]),
    "qc_decode_f32": (C.c_int, [P, P, i64, i32, i32, P, i32, P, P, P, P]),
    "qc_decode_i16": (C.c_int, [P, P, i64, i32, i32, P, i32, P, P, P, P]),
    "qc_decode_grouped_f32": (C.c_int, [P, i32, i32, i32, i32, P]),
    "qc_decode_grouped_i16": (C.c_int, [P, i32, i32, i32, i32, P]),
    "qc_decode_batch_f32_host": (C.c_int, [P, i64, P, i64, i32, i32, P, i64, i64, i32, i32, P, P, P]),
    "qc_decode_batch_i16_host": (C.c_int, [P, i64, P, i64, i32, i32, P, i64, i64, i32, i32, P, P, P]),
    "qc_encode_packed": (C.c_int, [P, P, i64, P, P]),
    "qc_encode_packed_host": (C.c_int, [P, P, i64, P]),
    "qc_encode_bits": (C.c_int, [P, P, i64, P, P]),
    "qc_encode_array": (C.c_int, [P, P, i64, P, P]),
    "qc_frames_info": (C.c_int, [C.c_uint64, C.c_uint32, i64, i64, i32, P, P]),
    "qc_channel_llr": (C.c_int, [P, i64, i32, C.c_double, P, C.c_uint64, C.c_uint32, i64, i32, C.c_double,
                                 P, P]),
    "qc_quantize_llr": (C.c_int, [P, i64, i32, C.c_double, P, P]),
    "qc_count_errors": (C.c_int, [P, i32, P, P, i64, i32, i32, i32, P, P]),
    "qc_pack_records": (C.c_int, [P, P, P, i64, i32, P, P]),
}


class DecodeJob(C.Structure):
    """Mirror of qc_decode_job_t."""
    _fields_ = [("code", P), ("llr", P), ("w", i64), ("hard", P), ("iters", P),
                ("conv", P), ("post_out", P)]


def lib():
    """Load libqcb200.so once; raise NativeLibraryError if it is not there."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryError(
                    f"{LIB_PATH} not built; run `python -m paper_2306_12063_b200._build` "
                    "(there is no CPU fallback)")
            try:
                L = C.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    """Translate a qcb200 status into the reference's exception types."""
    if rc == QC_OK:
        return
    msg = (lib().qc_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == QC_EUNALIGNED:
        raise UnsupportedZ(text)
    if rc == QC_EMALFORMED:
        raise MalformedHb(text)
    if rc == QC_EUNSUPPORTED:
        raise UnsupportedCode(text)
    if rc == QC_EINVAL:
        raise SizeMismatch(text) if "length" in text or "shape" in text else ValueError(text)
    if rc == QC_ENOMEM:
        raise MemoryError(text)
    if rc > 0:
        raise DeviceError(text)
    raise CodecError(text)


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())


class Code:
    """Owned qc_code_t handle for one (mb x nb, Z) shift table."""

    def __init__(self, shifts: np.ndarray, z: int):
        tab = np.ascontiguousarray(shifts, dtype=np.int32)
        mb, nb = tab.shape
        h = C.c_void_p()
        check(lib().qc_code_create(mb, nb, int(z), tab.ctypes.data, C.byref(h)), "qc_code_create")
        self._h = h
        self.mb, self.nb, self.z = mb, nb, int(z)
        self.n = nb * int(z)
        info = [i32() for _ in range(6)]
        check(lib().qc_code_info(h, *[C.byref(x) for x in info]), "qc_code_info")
        self.edges = info[3].value
        self.max_row_degree = info[4].value
        self.specialised = bool(info[5].value)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.qc_code_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None


class DeviceCall:
    """Context for one stream-ordered library call on CUDA tensors.

    The C side launches on whatever device is current, so the call runs under
    `torch.cuda.device(device)`; `stream` (default: that device's current
    stream) must live on the same device.  Tensors handed to the kernel that
    the caching allocator could recycle while it still runs on a side stream
    (contiguous temporaries, fresh outputs) are registered with `keep()`:
    when the call's stream is not the current stream, they are marked as used
    on it (`record_stream`) so their memory is not reused early.

        with DeviceCall(t.device, stream, t, *others) as call:
            out = torch.empty(...); call.keep(out)
            check(lib().qc_x(..., call.stream_ptr))
    """

    def __init__(self, device, stream=None, *tensors):
        import torch
        dev = torch.device(device)
        if dev.type != "cuda":
            raise ValueError(f"expected a CUDA device, got {dev}")
        if dev.index is None:                  # "cuda" = the current device
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        for t in tensors:
            if t is not None and t.device != self.device:
                raise ValueError(f"all tensors of one call must be on {self.device}, got {t.device}")
        self._stream = stream
        self._keep = [t for t in tensors if t is not None]

    def __enter__(self):
        import torch
        self._guard = torch.cuda.device(self.device)
        self._guard.__enter__()
        cur = torch.cuda.current_stream(self.device)
        self.stream = self._stream if self._stream is not None else cur
        if self.stream.device != self.device:
            self._guard.__exit__(None, None, None)
            raise ValueError(f"stream is on {self.stream.device}, tensors on {self.device}")
        self._side = self.stream != cur
        self.stream_ptr = C.c_void_p(self.stream.cuda_stream)
        return self

    def keep(self, *tensors):
        for t in tensors:
            if t is not None:
                if t.device != self.device:
                    raise ValueError(f"all tensors of one call must be on {self.device}, got {t.device}")
                self._keep.append(t)

    def __exit__(self, et, ev, tb):
        try:
            if et is None and self._side:
                for t in self._keep:
                    t.record_stream(self.stream)
        finally:
            self._guard.__exit__(et, ev, tb)
        return False
