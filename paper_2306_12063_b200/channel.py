"""BPSK/AWGN channel, Monte-Carlo waterfall and throughput runs on the GPU.

Mirror of the reference's `qcldpc.chansim` (/root/reference/pkg/src/qcldpc/
chansim.py) -- same names, arguments, dataclasses, CSV format, stop rule and
errors -- with the whole info -> encode -> BPSK -> AWGN -> LLR -> decode ->
count chain on the device:

* `frames="reference"` draws every frame's info bits and noise on the host
  exactly like the reference (`frame_rng`, `_gen_batch`, chansim.py:65-67,
  126-133, numpy's Philox) and runs the rest on the GPU.  The channel/LLR
  kernel repeats the reference's float64 arithmetic operation by operation,
  the decoder is bit-exact, so the WaterfallTable equals the reference's
  (tests/test_gpu_channel.py checks it against tables the reference produced).
* `frames="device"` (default) also draws the frames on the GPU, from a
  counter-based Philox4x32-10 stream keyed by (seed, point, frame): no host
  work and no PCIe traffic per frame, results independent of chunking and GPU
  count, but a different random stream than numpy's -- parity is statistical
  (the reference's calibrated operating points, test_acceptance.py:159-179).

Stopping is decided on the reference's 256-frame batch boundaries
(BATCH_FRAMES, chansim.py:153-176) from per-batch counters computed on the
device, so the GPU may decode a whole chunk of batches at once and still stop
exactly where the reference's sequential loop would.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .codebook import ModelMatrix
from .decoder import (Arithmetic, DecoderConfig, LlrBlock, code_handle, decode_batch,
                      quantize_llr)
from .errors import DivByZeroSigma, SizeMismatch

BATCH_FRAMES = 256


# --- host-side mirrors of the reference's channel helpers (chansim.py:26-67) ----

def ebn0_to_sigma2(ebn0_db: float, rate: float) -> float:
    """Noise variance for unit-energy BPSK at a given Eb/N0 and code rate."""
    if not 0.0 < rate <= 1.0:
        raise ValueError(f"rate {rate} outside (0, 1]")
    return 1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))


@dataclass(frozen=True)
class ChannelConfig:
    ebn0_db: float
    rate: float
    seed: int = 0
    sigma2: float = field(init=False)

    def __post_init__(self):
        object.__setattr__(self, "sigma2", ebn0_to_sigma2(self.ebn0_db, self.rate))


def bpsk_modulate(bits: np.ndarray) -> np.ndarray:
    """Map bit 0 to +1.0 and bit 1 to -1.0."""
    return 1.0 - 2.0 * np.asarray(bits, dtype=np.float64)


def awgn(symbols: np.ndarray, sigma2: float, rng: np.random.Generator) -> np.ndarray:
    if sigma2 < 0:
        raise ValueError("sigma2 must be >= 0")
    if sigma2 == 0:
        return np.asarray(symbols, dtype=np.float64).copy()
    return symbols + math.sqrt(sigma2) * rng.standard_normal(np.shape(symbols))


def llr_from_samples(samples: np.ndarray, sigma2: float) -> LlrBlock:
    """Channel LLR 2y/sigma^2 for BPSK over AWGN."""
    if sigma2 <= 0:
        raise DivByZeroSigma(f"sigma2 = {sigma2}")
    vals = (2.0 / sigma2) * np.asarray(samples, dtype=np.float64)
    return LlrBlock(vals.astype(np.float32), Arithmetic.Float32)


def frame_rng(seed: int, point: int, frame: int) -> np.random.Generator:
    """Counter-keyed numpy stream of one frame (the reference's frame recipe)."""
    return np.random.Generator(np.random.Philox(key=[seed, (point << 40) | frame]))


def gen_batch_host(mm: ModelMatrix, seed: int, point: int, start: int, count: int):
    """Info bits and noise for frames [start, start+count), one key per frame
    (host, numpy: identical to the reference's _gen_batch)."""
    info = np.empty((count, mm.k), dtype=np.uint8)
    noise = np.empty((count, mm.n), dtype=np.float64)
    for i in range(count):
        g = frame_rng(seed, point, start + i)
        info[i] = g.integers(0, 2, size=mm.k, dtype=np.uint8)
        noise[i] = g.standard_normal(mm.n)
    return info, noise


@dataclass(frozen=True)
class WaterfallPoint:
    ebn0_db: float
    frames: int
    bits_decoded: int
    bit_errors: int
    frame_errors: int
    avg_iterations: float

    @property
    def ber(self) -> float:
        return self.bit_errors / self.bits_decoded if self.bits_decoded else 0.0

    @property
    def fer(self) -> float:
        return self.frame_errors / self.frames if self.frames else 0.0


@dataclass
class WaterfallTable:
    points: list[WaterfallPoint]

    CSV_HEADER = "ebn0_db,frames,bits,bit_errors,frame_errors,ber,fer,avg_iters"

    def to_csv(self) -> str:
        lines = [self.CSV_HEADER]
        for p in self.points:
            lines.append("%.6g,%d,%d,%d,%d,%.6g,%.6g,%.6g" % (
                p.ebn0_db, p.frames, p.bits_decoded, p.bit_errors,
                p.frame_errors, p.ber, p.fer, p.avg_iterations))
        return "\n".join(lines) + "\n"


@dataclass
class ThroughputReport:
    arithmetic: Arithmetic
    workers: int
    pool: str
    frames: int
    info_bits: int
    seconds: float
    mbps: float

    CSV_HEADER = "arithmetic,workers,pool,frames,info_bits,seconds,mbps"

    def csv_line(self) -> str:
        return "%s,%d,%s,%d,%d,%.6g,%.6g" % (
            self.arithmetic.value, self.workers, self.pool, self.frames,
            self.info_bits, self.seconds, self.mbps)

    def summary(self) -> str:
        return (f"{self.arithmetic.value} workers={self.workers} pool={self.pool}: "
                f"{self.info_bits} info bits in {self.seconds:.3f} s "
                f"= {self.mbps:.2f} Mbps")


# --- device operations (CUDA torch tensors, stream ordered) ----------------------

def encode_array_device(code, info_bits, stream=None):
    """Bit-per-byte encoder on the device (encoder.encode_array, any Z):
    (W, K) uint8 CUDA tensor -> (W, N) uint8."""
    import torch
    c = code_handle(code)
    k = c.n - c.mb * c.z
    if info_bits.dim() != 2 or info_bits.shape[1] != k or info_bits.dtype != torch.uint8 or not info_bits.is_cuda:
        raise SizeMismatch(f"info bits must be a (W, {k}) uint8 CUDA tensor")
    with _lib.DeviceCall(info_bits.device, stream) as call:
        t = info_bits.contiguous()
        out = torch.empty((t.shape[0], c.n), dtype=torch.uint8, device=t.device)
        call.keep(t, out)
        _lib.check(_lib.lib().qc_encode_array(c.handle, _lib.ptr(t), t.shape[0], _lib.ptr(out), call.stream_ptr),
                   "encode_array")
    return out


def frames_info_device(seed: int, point: int, frame0: int, w: int, k: int, device, stream=None):
    """Info bits of frames [frame0, frame0+w) from the device Philox stream."""
    import torch
    with _lib.DeviceCall(device, stream) as call:
        out = torch.empty((w, k), dtype=torch.uint8, device=device)
        call.keep(out)
        _lib.check(_lib.lib().qc_frames_info(seed & (2**64 - 1), point, frame0, w, k, _lib.ptr(out),
                                             call.stream_ptr), "frames_info")
    return out


def channel_llr_device(cw_bits, sigma2: float, arithmetic: Arithmetic = Arithmetic.Float32, *,
                       q_b: int = 10, l_clip: float = 24.0, noise=None, seed: int = 0, point: int = 0,
                       frame0: int = 0, stream=None):
    """_llr_batch on the device: BPSK + AWGN + LLR (+ quantize_llr for Fixed16).

    `noise` (W, N) float64 CUDA tensor: the reference's samples (bit-exact
    LLRs); None: device Philox noise for frames frame0.. of `point`."""
    import torch
    if sigma2 <= 0:
        raise DivByZeroSigma(f"sigma2 = {sigma2}")
    fixed = arithmetic is Arithmetic.Fixed16
    with _lib.DeviceCall(cw_bits.device, stream, noise) as call:
        t = cw_bits.contiguous()
        w, n = t.shape
        out = torch.empty((w, n), dtype=torch.int16 if fixed else torch.float32, device=t.device)
        nz = None
        if noise is not None:
            nz = noise.contiguous()
            if nz.shape != t.shape or nz.dtype != torch.float64:
                raise SizeMismatch("noise must be a float64 tensor shaped like the codeword bits")
        call.keep(t, out, nz)
        _lib.check(_lib.lib().qc_channel_llr(_lib.ptr(t), w, n, float(sigma2), _lib.ptr(nz), seed & (2**64 - 1),
                                             point, frame0, q_b if fixed else 0, float(l_clip), _lib.ptr(out),
                                             call.stream_ptr), "channel_llr")
    return out


def quantize_llr_device(x, q_b: int = 10, l_clip: float = 24.0, stream=None):
    """decoder.quantize_llr on a float32 CUDA tensor -> int16 tensor."""
    import torch
    if not 1 <= q_b <= 14:
        raise ValueError("q_b must stay in [1, 14]")
    if x.dtype != torch.float32:
        raise SizeMismatch("quantize_llr_device wants float32")
    with _lib.DeviceCall(x.device, stream) as call:
        t = x.contiguous()
        out = torch.empty(t.shape, dtype=torch.int16, device=t.device)
        call.keep(t, out)
        _lib.check(_lib.lib().qc_quantize_llr(_lib.ptr(t), t.numel(), q_b, float(l_clip), _lib.ptr(out),
                                              call.stream_ptr), "quantize_llr")
    return out


def count_errors_device(hard, info_bits, iters, k: int, *, batch: int = BATCH_FRAMES, hard_packed: bool = False,
                        n: int | None = None, stream=None):
    """Per `batch` frames: (bit errors over the K info bits, frame errors,
    iteration sum) as a (ceil(W/batch), 3) int64 CUDA tensor."""
    import torch
    w = info_bits.shape[0]
    n = n if n is not None else (hard.shape[1] if not hard_packed else hard.shape[1] * 8)
    with _lib.DeviceCall(info_bits.device, stream, hard, iters) as call:
        h, inf, it = hard.contiguous(), info_bits.contiguous(), iters.contiguous()
        sums = torch.empty(((w + batch - 1) // batch, 3), dtype=torch.int64, device=info_bits.device)
        call.keep(h, inf, it, sums)
        _lib.check(_lib.lib().qc_count_errors(_lib.ptr(h), 1 if hard_packed else 0, _lib.ptr(inf), _lib.ptr(it),
                                              w, n, k, batch, _lib.ptr(sums), call.stream_ptr), "count_errors")
    return sums


# --- waterfall -------------------------------------------------------------------

def _walk_batches(sums: np.ndarray, counts: list[int], state: list[int], min_errors: int,
                  min_frames: int) -> bool:
    """Apply the reference's per-batch accumulation and stop test
    (chansim.py:166-176) to consecutive batches; state = [frames, bit_errors,
    frame_errors, iter_sum] is updated in place.  True = stop here."""
    for (be, fe, it), cnt in zip(sums.tolist(), counts):
        state[1] += be
        state[2] += fe
        state[3] += it
        state[0] += cnt
        if state[1] >= min_errors and state[0] >= min_frames:
            return True
    return False


def _point_distributed(chunk_sums, chunk: int, max_frames: int, min_errors: int, min_frames: int,
                       group=None, device=None) -> list[int]:
    """One SNR point's frame loop over consecutive `chunk`-frame chunks.

    `chunk_sums(f0, count)` returns the (ceil(count/256), 3) int64 per-batch
    counters of frames [f0, f0+count).  With a torch.distributed group of W
    ranks, rank r computes chunks r, r+W, ... of each round, the rounds'
    counters are all-gathered (the path's only collective) and every rank walks
    the batches in frame order with the reference's stop rule -- so the
    result is identical for any number of ranks.  Returns [frames, bit_errors,
    frame_errors, iter_sum]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if world > 1 else 0
    nb = chunk // BATCH_FRAMES
    state = [0, 0, 0, 0]                          # frames, bit_errors, frame_errors, iter_sum
    start = 0                                     # first frame of this round
    while True:
        if max_frames - start <= 0:
            break
        f0 = start + rank * chunk
        count = max(0, min(chunk, max_frames - f0))
        mine = torch.zeros((nb, 3), dtype=torch.int64, device=device)
        if count > 0:
            s = chunk_sums(f0, count)
            mine[: s.shape[0]] = s
        if world > 1:
            allc = torch.empty((world * nb, 3), dtype=torch.int64, device=device)
            dist.all_gather_into_tensor(allc, mine, group=group)
        else:
            allc = mine
        sums = allc.cpu().numpy()
        counts = []
        for r in range(world):
            c_r = max(0, min(chunk, max_frames - (start + r * chunk)))
            counts += [max(0, min(BATCH_FRAMES, c_r - b * BATCH_FRAMES)) for b in range(nb)]
        # batches past max_frames have count 0: the reference loop has stopped there
        n_valid = sum(1 for c in counts if c > 0)
        if _walk_batches(sums[:n_valid], counts[:n_valid], state, min_errors, min_frames):
            break
        start += world * chunk
    return state


def run_waterfall(code: ModelMatrix, cfg: DecoderConfig, snrs_db, min_errors: int = 10000,
                  max_frames: int = 1_000_000, seed: int = 0, workers: int = 1, min_frames: int = 1,
                  pool: str = "simple", *, frames: str = "device", chunk_frames: int = 1 << 16,
                  device=None, group=None) -> WaterfallTable:
    """Simulate info->encode->BPSK->AWGN->LLR->decode per SNR point on the GPU.

    A point stops at the first 256-frame batch boundary where bit_errors >=
    min_errors and frames >= min_frames, or when frames reaches max_frames
    (the reference's rule).  `workers` / `pool` are accepted for signature
    compatibility; the device replaces the worker pool.  Under
    torch.distributed (one process per GPU) pass `group` (e.g.
    torch.distributed.group.WORLD): the chunks of frames are spread over the
    group's ranks and the table is the same as on one GPU."""
    import torch
    if min_errors < 1:
        raise ValueError("min_errors must be >= 1")
    if frames not in ("device", "reference"):
        raise ValueError("frames must be 'device' or 'reference'")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    chunk = max(BATCH_FRAMES, chunk_frames // BATCH_FRAMES * BATCH_FRAMES)
    if frames == "reference":
        chunk = min(chunk, 8 * BATCH_FRAMES)      # host generation dominates; keep the overshoot small
    points = []
    for p_idx, ebn0 in enumerate(snrs_db):
        sigma2 = ebn0_to_sigma2(ebn0, code.rate.fraction)

        def chunk_sums(f0, count, p_idx=p_idx, sigma2=sigma2):
            if frames == "device":
                info = frames_info_device(seed, p_idx, f0, count, code.k, dev)
                noise = None
            else:
                hi, hn = gen_batch_host(code, seed, p_idx, f0, count)
                info = torch.from_numpy(hi).to(dev)
                noise = torch.from_numpy(hn).to(dev)
            cw = encode_array_device(code, info)
            llr = channel_llr_device(cw, sigma2, cfg.arithmetic, q_b=cfg.q_b, noise=noise, seed=seed,
                                     point=p_idx, frame0=f0)
            hard, iters, _ = decode_batch(code, llr, cfg)
            return count_errors_device(hard, info, iters, code.k)

        state = _point_distributed(chunk_sums, chunk, max_frames, min_errors, min_frames, group=group, device=dev)
        fr = state[0]
        points.append(WaterfallPoint(ebn0_db=float(ebn0), frames=fr, bits_decoded=fr * code.k,
                                     bit_errors=state[1], frame_errors=state[2],
                                     avg_iterations=state[3] / fr if fr else 0.0))
    return WaterfallTable(points)


def run_throughput_bench(code: ModelMatrix, cfg: DecoderConfig, workers: int = 1, pool: str = "cuda",
                         frames: int = 1000, seed: int = 0, ebn0_db: float = 2.0) -> ThroughputReport:
    """Time the decoder only (chansim.py:186-215): 10 iterations, early
    termination off, frames generated and one warm-up call untimed; the whole
    batch is one device call, timed with CUDA events."""
    import torch
    bench_cfg = replace(cfg, max_iterations=10, early_termination=False)
    if frames <= 0:
        return ThroughputReport(bench_cfg.arithmetic, workers, pool, 0, 0, 0.0, 0.0)
    dev = torch.device("cuda", torch.cuda.current_device())
    sigma2 = ebn0_to_sigma2(ebn0_db, code.rate.fraction)
    info = frames_info_device(seed, 0, 0, frames, code.k, dev)
    llr = channel_llr_device(encode_array_device(code, info), sigma2, bench_cfg.arithmetic, q_b=bench_cfg.q_b,
                             seed=seed)
    out = decode_batch(code, llr, bench_cfg)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    decode_batch(code, llr, bench_cfg, out=out)
    b.record()
    b.synchronize()
    seconds = a.elapsed_time(b) * 1e-3
    bits = frames * code.k
    mbps = bits / seconds / 1e6 if seconds > 0 else 0.0
    return ThroughputReport(bench_cfg.arithmetic, workers, pool, frames, bits, seconds, mbps)


__all__ = [
    "BATCH_FRAMES", "ChannelConfig", "ThroughputReport", "WaterfallPoint", "WaterfallTable", "awgn",
    "bpsk_modulate", "channel_llr_device", "count_errors_device", "ebn0_to_sigma2", "encode_array_device",
    "frame_rng", "frames_info_device", "gen_batch_host", "llr_from_samples", "quantize_llr",
    "quantize_llr_device", "run_throughput_bench", "run_waterfall",
]
