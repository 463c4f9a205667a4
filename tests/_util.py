"""Test helpers: golden fixture loading and seeded channel inputs.

Input generation mirrors the reference acceptance builder
(`/root/reference/pkg/tests/test_acceptance.py:45-54`) using the package's
host-side encoder, so tests on the GPU box need no reference checkout.
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np

from paper_2306_12063_b200 import codebook as CB

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden_cases(prefix: str):
    return sorted(p.name for p in GOLDEN.glob(f"{prefix}_*.npz"))


def load_case(name: str):
    z = np.load(GOLDEN / name)
    d = {k: z[k] for k in z.files}
    mm = CB.get_model_matrix(str(d["standard"]), int(d["n_bits"]), str(d["rate"]))
    d["mm"] = mm
    d["h"] = CB.expand(mm)
    d["hard"] = np.unpackbits(d["hard_packed"], axis=-1, count=mm.n)
    return d


def sigma2(ebn0_db: float, rate: float) -> float:
    """chansim.ebn0_to_sigma2 (/root/reference/pkg/src/qcldpc/chansim.py:26-30)."""
    return 1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))


def noisy_llrs(mm, frames: int, ebn0_db: float, seed: int, fixed: bool = False):
    """Seeded BPSK/AWGN channel LLRs 2y/sigma^2 (reference test_acceptance.py:45-54).

    Returns (llr values, info bits, codeword bits); int16 LLRs go through
    quantize_llr(q_b=10) exactly like the reference's fixed-point inputs.
    """
    from paper_2306_12063_b200 import decoder as D, encoder as E
    rng = np.random.default_rng(seed)
    info = rng.integers(0, 2, size=(frames, mm.k), dtype=np.uint8)
    cw = E.encode_array(E.make_plan(mm), info)
    s2 = sigma2(ebn0_db, mm.rate.fraction)
    y = (1.0 - 2.0 * cw) + rng.standard_normal(cw.shape) * math.sqrt(s2)
    llr = (2.0 / s2) * y
    vals = D.quantize_llr(llr).values if fixed else llr.astype(np.float32)
    return vals, info, cw


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def acceptance_case(fixed: bool):
    """The reference's decoder-oracle acceptance case
    (/root/reference/pkg/tests/test_acceptance.py:139-156): WiMAX 576 R1/2,
    1000 frames at 1.8 dB, seed 1004, 10 iterations with early termination.
    Returns (h, llr values, hard, iters, conv); the LLRs are regenerated with the
    reference recipe and checked against the fixture's SHA-256."""
    import hashlib
    z = np.load(GOLDEN / "acceptance_decoder_oracle.npz")
    mm = CB.get_model_matrix("wimax", 576, "1/2")
    vals, _, _ = noisy_llrs(mm, int(z["frames"]), float(z["ebn0_db"]), int(z["seed"]), fixed)
    tag = "i16" if fixed else "f32"
    assert hashlib.sha256(vals.tobytes()).digest() == z[f"llr_sha256_{tag}"].tobytes(), \
        "LLR recipe drifted from the reference's (numpy generator / encoder / quantizer)"
    hard = np.unpackbits(z[f"hard_packed_{tag}"], axis=-1, count=mm.n)
    return CB.expand(mm), vals, hard, z[f"iters_{tag}"], z[f"conv_{tag}"]
