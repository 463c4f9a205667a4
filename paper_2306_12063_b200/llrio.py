"""Wire formats either side of the decoder.

* The `LLR0` container (/root/reference/pkg/src/qcldpc/decoder.py:261-301):
  16-byte header (magic "LLR0", uint32 N, uint32 count, uint8 arithmetic
  0 = float32 / 1 = fixed16, 3 pad bytes) then count*N little-endian
  values.  `write_llr_file` / `read_llr_file` mirror the reference (same
  errors); `read_llr_file_device` reads the payload straight into pinned host
  memory and hands it to the GPU without a numpy copy.
* Decode records (the CLI `decode` output, cli.py:169-183): per codeword
  packbits(hard) | min(iterations, 255) | converged.  `decode_llr_file` does
  the whole CLI step with the decoder writing bit-packed hard decisions and
  one device kernel (qc_pack_records) assembling the records, so only the
  records cross PCIe.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from . import _lib
from .decoder import Arithmetic, DecoderConfig, LlrBlock, code_handle, decode_batch
from .errors import CorruptFile, SizeMismatch

_LLR_MAGIC = b"LLR0"
_LLR_HEADER = struct.Struct("<4sIIB3x")


def write_llr_file(path, block: LlrBlock) -> None:
    vals = block.values
    if vals.ndim == 1:
        vals = vals.reshape(1, -1)
    if vals.ndim != 2:
        raise SizeMismatch("LLR files hold a (count, N) block")
    count, n = vals.shape
    code = 0 if block.arithmetic is Arithmetic.Float32 else 1
    wire = vals.astype("<f4" if code == 0 else "<i2")
    with open(path, "wb") as f:
        f.write(_LLR_HEADER.pack(_LLR_MAGIC, n, count, code))
        f.write(wire.tobytes())


def _read_header(f, path):
    head = f.read(_LLR_HEADER.size)
    if len(head) != _LLR_HEADER.size:
        raise CorruptFile(f"{path}: truncated header")
    magic, n, count, code = _LLR_HEADER.unpack(head)
    if magic != _LLR_MAGIC:
        raise CorruptFile(f"{path}: bad magic {magic!r}")
    if code not in (0, 1):
        raise CorruptFile(f"{path}: unknown arithmetic code {code}")
    return n, count, Arithmetic.Float32 if code == 0 else Arithmetic.Fixed16


def read_llr_file(path) -> LlrBlock:
    with open(path, "rb") as f:
        n, count, arith = _read_header(f, path)
        payload = f.read()
    wire = "<f4" if arith is Arithmetic.Float32 else "<i2"
    expect = count * n * np.dtype(wire).itemsize
    if len(payload) != expect:
        raise CorruptFile(f"{path}: payload {len(payload)} B, header says {expect} B")
    vals = np.frombuffer(payload, dtype=wire).reshape(count, n)
    return LlrBlock(vals.astype(arith.dtype), arith)


def read_llr_file_device(path, device=None):
    """(values as a CUDA tensor (count, N), arithmetic): payload read into a
    pinned buffer, copied to the device asynchronously on the current stream."""
    import torch
    with open(path, "rb") as f:
        n, count, arith = _read_header(f, path)
        item = 4 if arith is Arithmetic.Float32 else 2
        expect = count * n * item
        left = os.fstat(f.fileno()).st_size - _LLR_HEADER.size
        if left != expect:
            raise CorruptFile(f"{path}: payload {left} B, header says {expect} B")
        dt = torch.float32 if item == 4 else torch.int16
        pinned = torch.empty((count, n), dtype=dt, pin_memory=True)
        view = memoryview(pinned.numpy()).cast("B")
        got = f.readinto(view) if expect else 0
        if got != expect:
            raise CorruptFile(f"{path}: short read {got} of {expect} B")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    return pinned.to(dev, non_blocking=True), arith


def pack_records_device(hard_packed, iters, conv, n: int, stream=None):
    """(W, ceil(N/8)+2) uint8 CUDA tensor of CLI decode records."""
    import torch
    w = iters.shape[0]
    with _lib.DeviceCall(iters.device, stream, hard_packed, conv) as call:
        hp, it, cv = hard_packed.contiguous(), iters.contiguous(), conv.contiguous()
        out = torch.empty((w, (n + 7) // 8 + 2), dtype=torch.uint8, device=iters.device)
        call.keep(hp, it, cv, out)
        _lib.check(_lib.lib().qc_pack_records(_lib.ptr(hp), _lib.ptr(it), _lib.ptr(cv), w, n, _lib.ptr(out),
                                              call.stream_ptr), "pack_records")
    return out


def decode_llr_file(code, path_in, path_out, cfg: DecoderConfig | None = None, arith: str | None = None) -> int:
    """The CLI `decode` step (cli.py:169-183) on the GPU: LLR0 in, records out."""
    c = code_handle(code)
    vals, file_arith = read_llr_file_device(path_in)
    if vals.shape[1] != c.n:
        raise CorruptFile(f"{path_in}: N={vals.shape[1]} but code has N={c.n}")
    if arith is not None and arith != file_arith.value:
        raise CorruptFile(f"{path_in}: holds {file_arith.value}, --arith says {arith}")
    base = cfg or DecoderConfig()
    cfg = DecoderConfig(max_iterations=base.max_iterations, q_b=base.q_b, arithmetic=file_arith,
                        early_termination=base.early_termination)
    if vals.shape[0] == 0:
        open(path_out, "wb").close()
        return 0
    hard, iters, conv = decode_batch(code, vals, cfg, hard_packed=True)
    rec = pack_records_device(hard, iters, conv, c.n).cpu().numpy()
    with open(path_out, "wb") as f:
        f.write(rec.tobytes())
    return 0


__all__ = ["decode_llr_file", "pack_records_device", "read_llr_file", "read_llr_file_device",
           "write_llr_file"]
