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
