"""BASELINE.json workloads and seeded synthetic channel inputs.

The five configurations of `/root/repo/BASELINE.json`:

  C1  Wi-Fi 648 R1/2,  f32, 10 it, W = 1024,      Eb/N0 2.0 dB
  C2  WiMAX 2304 R1/2, f32, 10 it, W = 65536,     Eb/N0 1.5 dB   (bench default)
  C3  Wi-Fi 1944 R5/6, i16,  8 it, W = 262144,    Eb/N0 4.0 dB
  C4  18 codes mixed,  f32, 10 it, W = 18 x 16384, Eb/N0 3.0 dB
  C5  WiMAX 2304 R3/4A, i16, 10 it, W = 2^22,     Eb/N0 2.0 dB (+ packed encode)

Inputs follow the reference channel (chansim.py:26-62, test_acceptance.py:45-54):
seeded uniform info bits, systematic encoding, BPSK (0 -> +1), AWGN with
sigma^2 = 1 / (2 R 10^(EbN0/10)), LLR = 2y/sigma^2 in float64, then float32 or
quantize_llr(q_b=10).  No public dataset is involved.

BASELINE-sized batches are generated on the device by `shard_llrs`, keyed by
the GLOBAL frame index of the job: frame f of code ci gets its info bits and
its AWGN samples from the counter-based Philox streams of the device channel
(`qc_frames_info` / `qc_channel_llr`, keyed by (seed, ci, f)), is encoded by
the device `encode_array`, and quantised exactly like `quantize_llr`.  A rank
that owns frames [lo, hi) therefore holds exactly the rows [lo, hi) of the
one-GPU batch, so hard decisions are comparable across GPU counts.  Decoding
runs a fixed number of iterations, so the work does not depend on the data.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import codebook as CB
from .decoder import Arithmetic, DecoderConfig
from .encoder import encode_array, make_plan


@dataclass(frozen=True)
class Workload:
    key: str
    codes: tuple            # ((standard, n_bits, rate), ...)
    fixed: bool
    iters: int
    w_per_code: int
    ebn0_db: float
    seed: int
    strong: bool = False    # True: w_per_code is the job total, sharded over the ranks

    @property
    def arithmetic(self) -> Arithmetic:
        return Arithmetic.Fixed16 if self.fixed else Arithmetic.Float32

    def config(self) -> DecoderConfig:
        return DecoderConfig(max_iterations=self.iters, arithmetic=self.arithmetic,
                             early_termination=False)

    def model_matrices(self):
        return [CB.get_model_matrix(*c) for c in self.codes]

    @property
    def w_total(self) -> int:
        return self.w_per_code * len(self.codes)

    def for_rank(self, rank: int, world: int) -> "Workload":
        """This rank's share: the whole per-GPU batch (weak scaling) or its
        contiguous shard of the job total (strong scaling, shard.shard_range)."""
        if not self.strong or world == 1:
            return self
        from dataclasses import replace
        from .shard import shard_range
        lo, hi = shard_range(self.w_per_code, rank, world)
        return replace(self, w_per_code=hi - lo)


ALL_18 = tuple([("wifi", n, r) for n in (648, 1296, 1944) for r in ("1/2", "2/3", "3/4", "5/6")]
               + [("wimax", 2304, r) for r in ("1/2", "2/3A", "2/3B", "3/4A", "3/4B", "5/6")])

WORKLOADS = {
    "C1": Workload("C1", (("wifi", 648, "1/2"),), False, 10, 1024, 2.0, 1),
    "C2": Workload("C2", (("wimax", 2304, "1/2"),), False, 10, 65536, 1.5, 2),
    "C3": Workload("C3", (("wifi", 1944, "5/6"),), True, 8, 262144, 4.0, 3),
    "C4": Workload("C4", ALL_18, False, 10, 16384, 3.0, 4),
    # BASELINE config 5: 2^22 codewords sharded across 1/2/4/8 GPUs (strong scaling)
    "C5": Workload("C5", (("wimax", 2304, "3/4A"),), True, 10, 1 << 22, 2.0, 5, True),
}


def sigma2(ebn0_db: float, rate: float) -> float:
    """chansim.ebn0_to_sigma2 (/root/reference/pkg/src/qcldpc/chansim.py:26-30)."""
    return 1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))


def host_llrs(mm, w: int, ebn0_db: float, seed, fixed: bool):
    """Exact host generation (reference recipe), returns (llr, info bits)."""
    from .decoder import quantize_llr
    rng = np.random.default_rng(seed)
    info = rng.integers(0, 2, size=(w, mm.k), dtype=np.uint8)
    cw = encode_array(make_plan(mm), info)
    s2 = sigma2(ebn0_db, mm.rate.fraction)
    y = (1.0 - 2.0 * cw) + rng.standard_normal(cw.shape) * math.sqrt(s2)
    llr = (2.0 / s2) * y
    return (quantize_llr(llr).values if fixed else llr.astype(np.float32)), info


def frame_range(wl: Workload, rank: int, world: int) -> tuple[int, int]:
    """Global frames [lo, hi) of each code that `rank` decodes: its contiguous
    shard of the job total (strong scaling, C5) or its own block of W frames
    (weak scaling: rank r takes frames [r W, (r+1) W))."""
    if wl.strong:
        from .shard import shard_range
        return shard_range(wl.w_per_code, rank, world)
    return rank * wl.w_per_code, (rank + 1) * wl.w_per_code


def shard_info(wl: Workload, ci: int, lo: int, hi: int, device):
    """Info bits (hi-lo, K) of global frames [lo, hi) of code ci (device Philox stream)."""
    from .channel import frames_info_device
    mm = wl.model_matrices()[ci]
    return frames_info_device(wl.seed, ci, lo, hi - lo, mm.k, device)


def shard_llrs(wl: Workload, ci: int, lo: int, hi: int, device, chunk: int = 1 << 16):
    """(hi-lo, N) channel LLRs of global frames [lo, hi) of code ci, generated on
    `device`: Philox info bits -> encode_array -> BPSK/AWGN (Philox noise keyed
    by frame) -> float32 or quantize_llr(q_b=10).  Identical rows for a frame
    whichever rank / shard generates it."""
    import torch
    from .channel import channel_llr_device, encode_array_device
    mm = wl.model_matrices()[ci]
    s2 = sigma2(wl.ebn0_db, mm.rate.fraction)
    out = torch.empty((hi - lo, mm.n), dtype=torch.int16 if wl.fixed else torch.float32, device=device)
    for f0 in range(lo, hi, chunk):
        f1 = min(hi, f0 + chunk)
        cw = encode_array_device(mm, shard_info(wl, ci, f0, f1, device))
        out[f0 - lo:f1 - lo] = channel_llr_device(cw, s2, wl.arithmetic, seed=wl.seed, point=ci, frame0=f0)
    return out
