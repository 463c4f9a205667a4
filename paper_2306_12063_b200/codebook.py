"""Code selection: the 802.11 (Wi-Fi) and 802.16 (WiMAX) QC-LDPC families.

Host-side mirror of the reference's `qcldpc.codebook`
(`/root/reference/pkg/src/qcldpc/codebook.py`), same names and semantics:

* `get_model_matrix(standard, n_bits, rate)` (ref `codebook.py:203-214`)
* `scale_model_matrix(base, z)` (ref `:217-229`): floor(p*z/96), or p mod z
  for WiMAX rate 2/3A
* `expand(mm)` -> `SparseParityCheck` CSR (ref `:232-266`)
* `supported_codes()` (ref `:317-324`)

What changes on B200: the decoder never walks `expand`'s CSR.  A code is
handed to the device as its mb x nb shift table (`ModelMatrix.entries`),
which `libqcb200` turns into a per-tier (block column, shift) descriptor
living in kernel-parameter constant memory (see `_lib.Code`).  `expand`
stays for the drop-in `_kernels` signature (which passes CSR) and for the
host-side syndrome helpers.

The base matrices come from `data/base_matrices.json`, converted from the
reference's tables by `tools/import_tables.py`.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache
from pathlib import Path

import numpy as np

from .errors import BadZ, UnsupportedCode


class Standard(Enum):
    Wifi = "wifi"
    Wimax = "wimax"


class Rate(Enum):
    R12 = "1/2"
    R23A = "2/3A"
    R23B = "2/3B"
    R34A = "3/4A"
    R34B = "3/4B"
    R56 = "5/6"

    @property
    def fraction(self) -> float:
        num, den = self.value.rstrip("AB").split("/")
        return int(num) / int(den)


WIFI_Z = {648: 27, 1296: 54, 1944: 81}
WIFI_RATES = (Rate.R12, Rate.R23A, Rate.R34A, Rate.R56)
WIMAX_Z = tuple(range(24, 97, 4))
WIMAX_Z0 = 96
NB = 24
_KB = {Rate.R12: 12, Rate.R23A: 16, Rate.R23B: 16, Rate.R34A: 18,
       Rate.R34B: 18, Rate.R56: 20}


def parse_standard(value) -> Standard:
    if isinstance(value, Standard):
        return value
    for s in Standard:
        if str(value).lower() == s.value:
            return s
    raise UnsupportedCode(f"unknown standard {value!r}")


def parse_rate(value, standard: Standard | None = None) -> Rate:
    """'1/2', '2/3', '2/3B', '3/4a', '5/6' ...; bare 2/3 and 3/4 mean the A variant."""
    if isinstance(value, Rate):
        rate = value
    else:
        key = str(value).upper()
        key = {"2/3": "2/3A", "3/4": "3/4A"}.get(key, key)
        matches = [r for r in Rate if r.value == key]
        if not matches:
            raise UnsupportedCode(f"unknown rate {value!r}")
        rate = matches[0]
    if standard is Standard.Wifi and rate not in WIFI_RATES:
        raise UnsupportedCode(f"wifi defines no {rate.value} code")
    return rate


@dataclass(frozen=True)
class ModelMatrix:
    """mb x nb shift table: -1 = zero block, s >= 0 = identity rotated by s."""

    standard: Standard
    rate: Rate
    z: int
    nb: int
    kb: int
    entries: np.ndarray

    def __post_init__(self):
        e = np.ascontiguousarray(self.entries, dtype=np.int32)
        e.flags.writeable = False
        object.__setattr__(self, "entries", e)
        if e.shape != (self.mb, self.nb):
            raise ValueError(f"entries shape {e.shape} != ({self.mb}, {self.nb})")
        if e.min() < -1 or e.max() >= self.z:
            raise ValueError("entries must lie in [-1, z)")

    @property
    def mb(self) -> int:
        return self.nb - self.kb

    @property
    def n(self) -> int:
        return self.nb * self.z

    @property
    def k(self) -> int:
        return self.kb * self.z

    @property
    def m(self) -> int:
        return self.mb * self.z

    @property
    def edges(self) -> int:
        return int((self.entries >= 0).sum()) * self.z


@dataclass(frozen=True)
class SparseParityCheck:
    """Expanded H as CSR in both orientations (reference layout, ref `:122-155`)."""

    n: int
    k: int
    m: int
    z: int
    row_ptr: np.ndarray
    row_cols: np.ndarray
    col_ptr: np.ndarray
    col_rows: np.ndarray

    def row(self, m: int) -> np.ndarray:
        return self.row_cols[self.row_ptr[m]:self.row_ptr[m + 1]]

    def col(self, n: int) -> np.ndarray:
        return self.col_rows[self.col_ptr[n]:self.col_ptr[n + 1]]

    @property
    def row_degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    @property
    def col_degrees(self) -> np.ndarray:
        return np.diff(self.col_ptr)

    @property
    def max_row_degree(self) -> int:
        return int(self.row_degrees.max())

    @property
    def edges(self) -> int:
        return int(self.row_cols.shape[0])


_DATA = Path(__file__).with_name("data") / "base_matrices.json"


@lru_cache(maxsize=None)
def _base_tables() -> dict:
    return json.loads(_DATA.read_text())["matrices"]


def _table_name(standard: Standard, n_bits: int, rate: Rate) -> str:
    if standard is Standard.Wifi:
        return f"wifi_n{n_bits}_r" + rate.value.rstrip("AB").replace("/", "")
    return "wimax_r" + rate.value.replace("/", "").lower()


@lru_cache(maxsize=None)
def _load(name: str) -> ModelMatrix:
    rec = _base_tables()[name]
    return ModelMatrix(parse_standard(rec["standard"]), parse_rate(rec["rate"]),
                       rec["z"], rec["nb"], rec["kb"],
                       np.array(rec["entries"], dtype=np.int32))


def get_model_matrix(standard, n_bits: int, rate) -> ModelMatrix:
    """Look a code up by (standard, N, rate); WiMAX is scaled from its Z=96 base."""
    standard = parse_standard(standard)
    rate = parse_rate(rate, standard)
    if standard is Standard.Wifi:
        if n_bits not in WIFI_Z:
            raise UnsupportedCode(f"wifi defines no N={n_bits} code")
        return _load(_table_name(standard, n_bits, rate))
    if n_bits % NB or n_bits // NB not in WIMAX_Z:
        raise UnsupportedCode(f"wimax defines no N={n_bits} code")
    return scale_model_matrix(_load(_table_name(standard, n_bits, rate)), n_bits // NB)


def scale_model_matrix(base: ModelMatrix, z_target: int) -> ModelMatrix:
    """802.16e shift scaling from the Z0=96 base (ref `codebook.py:217-229`)."""
    if base.standard is not Standard.Wimax or base.z != WIMAX_Z0:
        raise BadZ("scaling starts from the Z=96 wimax base matrix")
    if z_target not in WIMAX_Z:
        raise BadZ(f"z={z_target} not in the supported 24..96 step 4 table")
    e = base.entries.astype(np.int64)
    pos = e > 0
    if base.rate is Rate.R23A:
        scaled = np.where(pos, e % z_target, e)
    else:
        scaled = np.where(pos, (e * z_target) // WIMAX_Z0, e)
    return ModelMatrix(base.standard, base.rate, z_target, base.nb, base.kb,
                       scaled.astype(np.int32))


def expand(mm: ModelMatrix) -> SparseParityCheck:
    """CSR of H: block (i, j) with shift e >= 0 puts a one at (iZ + r, jZ + (r+e) mod Z)."""
    z, e = mm.z, mm.entries
    r = np.arange(z, dtype=np.int64)
    row_blocks, col_blocks = [], []
    for i in range(mm.mb):
        js = np.nonzero(e[i] >= 0)[0]
        row_blocks.append((js[None, :] * z + (r[:, None] + e[i, js][None, :]) % z).reshape(-1))
    for j in range(mm.nb):
        is_ = np.nonzero(e[:, j] >= 0)[0]
        col_blocks.append((is_[None, :] * z + (r[:, None] - e[is_, j][None, :]) % z).reshape(-1))
    row_deg = np.repeat((e >= 0).sum(axis=1), z)
    col_deg = np.repeat((e >= 0).sum(axis=0), z)
    row_ptr = np.concatenate([[0], np.cumsum(row_deg)]).astype(np.int32)
    col_ptr = np.concatenate([[0], np.cumsum(col_deg)]).astype(np.int32)
    return SparseParityCheck(
        n=mm.n, k=mm.k, m=mm.m, z=z, row_ptr=row_ptr,
        row_cols=np.concatenate(row_blocks).astype(np.int32),
        col_ptr=col_ptr, col_rows=np.concatenate(col_blocks).astype(np.int32))


def supported_codes():
    """(standard, N, rate) for all 126 codes: 12 Wi-Fi + 19 Z values x 6 WiMAX rates."""
    for n_bits in WIFI_Z:
        for rate in WIFI_RATES:
            yield Standard.Wifi, n_bits, rate
    for z in WIMAX_Z:
        for rate in Rate:
            yield Standard.Wimax, NB * z, rate


def shift_table_from_csr(row_ptr: np.ndarray, row_cols: np.ndarray, mb: int, z: int,
                         n: int) -> np.ndarray:
    """Recover the mb x nb shift table from the reference kernel's CSR arguments.

    The drop-in `_kernels.decode_batch_*` receives `(row_ptr, col_idx, mb, z)`
    exactly like the reference (`_kernels.py:17-19`).  Row i*Z of tier i lists
    column j*Z + e for every block (i, j) with shift e, so e = col mod Z and
    j = col // Z.  The table is then checked against every row of the CSR;
    a CSR that is not a QC expansion raises ValueError (the GPU path has no
    generic-sparse fallback).
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    cols = np.asarray(row_cols, dtype=np.int64)
    if z < 1 or n % z or row_ptr.shape[0] != mb * z + 1:
        raise ValueError("CSR shape does not match mb*z rows")
    nb = n // z
    tab = np.full((mb, nb), -1, dtype=np.int32)
    for i in range(mb):
        first = cols[row_ptr[i * z]:row_ptr[i * z + 1]]
        js, es = first // z, first % z
        if np.any(np.diff(js) <= 0):
            raise ValueError(f"tier {i}: columns not in ascending distinct block order")
        tab[i, js] = es
    r = np.arange(z, dtype=np.int64)
    for i in range(mb):
        js = np.nonzero(tab[i] >= 0)[0]
        want = (js[None, :] * z + (r[:, None] + tab[i, js][None, :]) % z).reshape(-1)
        got = cols[row_ptr[i * z]:row_ptr[(i + 1) * z]]
        deg = np.diff(row_ptr[i * z:(i + 1) * z + 1])
        if np.any(deg != js.size) or got.shape != want.shape or np.any(got != want):
            raise ValueError(f"tier {i}: CSR is not a quasi-cyclic expansion")
    return tab
