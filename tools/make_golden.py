"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Runs only in the build container, where `/root/reference` exists: it imports
the reference package (`/root/reference/pkg/src/qcldpc`) and its test-side
oracle (`/root/reference/pkg/tests/_reference.py`) and records their outputs
on seeded inputs.  The GPU box never reads `/root/reference`; it only reads
the committed fixtures.

Fixtures
--------
decode_<case>.npz   LLR block + reference `decode_block` outputs (hard bits
                    packed MSB-first, iterations, converged) and, for the
                    first few codewords, the final posteriors from the
                    white-box oracle `init_state` + `tier_update` sweeps with
                    the reference stop rule (pkg/tests/test_decoder.py:179-198).
special_<case>.npz  hostile inputs (int16 wrap, -32768, +/-0.0, inf, NaN):
                    reference kernel outputs only (tier_update's np.argmin
                    treats NaN differently from the kernel, so posteriors
                    are pinned for the finite cases only).
encode_packed.npz   reference `encode_packed` on seeded info words for
                    byte-aligned WiMAX codes, several word sizes.
kat.npz             known answers: degree-3 row by hand (test_decoder.py:74-91),
                    quantizer points (test_decoder.py:274-289).
acceptance_decoder_oracle.npz
                    the reference's decoder-oracle acceptance case
                    (pkg/tests/test_acceptance.py:139-156): WiMAX 576 R1/2,
                    1000 frames at 1.8 dB, seed 1004, default DecoderConfig
                    (10 iterations, early termination), Fixed16 and Float32;
                    decode_block outputs (checked here against the explicit-
                    message `_reference.ref_decode`, as that test does) plus the
                    SHA-256 of the LLR block, which the tests regenerate with
                    the same numpy recipe instead of storing 3 MB of LLRs.

Usage:  python tools/make_golden.py [kat|encode|special|decode|acceptance ...]
"""

from __future__ import annotations

import math
import zlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import qcldpc as R  # noqa: E402
import _reference as RR  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def noisy(mm, frames, ebn0_db, seed, fixed):
    """Mirror of the reference acceptance input builder (test_acceptance.py:45-54)."""
    rng = np.random.default_rng(seed)
    info = rng.integers(0, 2, size=(frames, mm.k), dtype=np.uint8)
    cw = R.encode_array(R.make_plan(mm), info)
    sigma2 = 1.0 / (2.0 * mm.rate.fraction * 10.0 ** (ebn0_db / 10.0))
    y = (1.0 - 2.0 * cw) + rng.standard_normal(cw.shape) * math.sqrt(sigma2)
    llr = (2.0 / sigma2) * y
    vals = R.quantize_llr(llr).values if fixed else llr.astype(np.float32)
    return vals, info, cw


def tier_sweeps(h, vals, arith, max_iters, early):
    """White-box posteriors: init_state + tier_update, stop rule of the kernel."""
    st = R.init_state(h, R.LlrBlock(vals, arith))
    it, ok = 0, False
    for k in range(max_iters):
        for t in range(h.m // h.z):
            R.tier_update(st, h, t)
        it = k + 1
        ok = R.syndrome_check(h, (st.posterior <= 0).astype(np.uint8))
        if ok and early:
            break
    return st.posterior.copy(), it, ok


def ref_decode(h, vals, arith, max_iters, early):
    cfg = R.DecoderConfig(max_iterations=max_iters, arithmetic=arith, early_termination=early)
    res = R.decode_block(h, R.LlrBlock(vals, arith), cfg, workers=8, pool="mtx")
    hard = np.stack([r.hard_bits for r in res]) if res else np.zeros((0, h.n), np.uint8)
    iters = np.array([r.iterations for r in res], np.int32)
    conv = np.array([r.converged for r in res], np.uint8)
    return hard, iters, conv


DECODE_CASES = [
    # name, std, N, rate, fixed, ebn0, iters, early, frames, post_frames
    ("wimax576_r12_f32_et", "wimax", 576, "1/2", False, 1.8, 10, True, 48, 6),
    ("wimax576_r12_i16_et", "wimax", 576, "1/2", True, 1.8, 10, True, 48, 6),
    ("wifi648_r12_f32_c1", "wifi", 648, "1/2", False, 2.0, 10, False, 32, 4),
    ("wifi648_r34_f32_noet", "wifi", 648, "3/4", False, 2.5, 5, False, 16, 4),
    ("wimax2304_r12_f32_c2", "wimax", 2304, "1/2", False, 1.5, 10, False, 16, 2),
    ("wifi1944_r56_i16_c3", "wifi", 1944, "5/6", True, 4.0, 8, False, 16, 2),
    ("wimax2304_r34a_i16_c5", "wimax", 2304, "3/4A", True, 2.0, 10, False, 16, 2),
    ("wifi1296_r23_f32_et", "wifi", 1296, "2/3", False, 2.5, 10, True, 16, 2),
    ("wimax1056_r23b_i16_et", "wimax", 1056, "2/3B", True, 2.5, 10, True, 16, 2),
    ("wimax960_r56_f32_et", "wimax", 960, "5/6", False, 4.0, 10, True, 16, 2),
    ("wimax672_r34b_f32_noet", "wimax", 672, "3/4B", False, 3.0, 7, False, 16, 2),
    ("wimax1920_r23a_i16_et", "wimax", 1920, "2/3A", True, 2.5, 10, True, 16, 2),
]


def make_decode():
    for name, std, n, rate, fixed, ebn0, iters, early, frames, npost in DECODE_CASES:
        mm = R.get_model_matrix(std, n, rate)
        h = R.expand(mm)
        arith = R.Arithmetic.Fixed16 if fixed else R.Arithmetic.Float32
        vals, info, cw = noisy(mm, frames, ebn0, seed=zlib.crc32(name.encode()) % 100003, fixed=fixed)
        hard, it, conv = ref_decode(h, vals, arith, iters, early)
        post = []
        for w in range(npost):
            p, i2, ok2 = tier_sweeps(h, vals[w], arith, iters, early)
            assert np.array_equal((p <= 0).astype(np.uint8), hard[w]) and i2 == it[w] and ok2 == conv[w]
            post.append(p)
        # independent explicit-message oracle agrees too (pkg/tests/_reference.py:122-130)
        for w in range(min(frames, 8)):
            hh, ii, cc = RR.ref_decode(h, vals[w], iters, early)
            assert np.array_equal(hh, hard[w]) and ii == it[w] and cc == conv[w]
        np.savez_compressed(
            OUT / f"decode_{name}.npz", standard=std, n_bits=n, rate=rate,
            arithmetic="fixed16" if fixed else "float32", ebn0_db=ebn0,
            max_iters=iters, early_term=int(early), llr=vals,
            hard_packed=np.packbits(hard, axis=-1), iters=it, conv=conv,
            post=np.stack(post), info=np.packbits(info, axis=-1))
        print(name, "conv", conv.mean(), "iters", it.mean())


def make_special():
    rng = np.random.default_rng(2024)
    cases = {}
    # int16 wrap-heavy: full-range values incl. -32768 on a high-rate code
    mm = R.get_model_matrix("wifi", 1944, "5/6")
    v = rng.integers(-32768, 32768, size=(12, mm.n), dtype=np.int64).astype(np.int16)
    v[:, ::97] = -32768
    v[0, :] = -32768
    v[1, :] = 32767
    cases["i16_fullrange_wifi1944_r56"] = (mm, v, R.Arithmetic.Fixed16, 8, False, True)
    mm2 = R.get_model_matrix("wimax", 576, "1/2")
    v2 = rng.integers(-4000, 4000, size=(12, mm2.n), dtype=np.int64).astype(np.int16) * 8
    cases["i16_large_wimax576_r12_et"] = (mm2, v2, R.Arithmetic.Fixed16, 10, True, True)
    v3 = np.zeros((4, mm2.n), np.int16)
    v3[1] = 1
    v3[2] = -1
    cases["i16_zeros_wimax576"] = (mm2, v3, R.Arithmetic.Fixed16, 4, True, True)
    # float specials: signed zeros, exact ties, infinities and NaN
    f = rng.standard_normal((12, mm2.n)).astype(np.float32) * 3
    f[0] = 0.0
    f[1] = -0.0
    f[2, ::3] = -0.0
    f[3] = np.round(f[3])          # many exact ties
    f[4] = np.sign(f[4]) * 2.0     # all-equal magnitudes
    f[5, 7] = np.inf
    f[6, 11] = -np.inf
    f[7, 5] = np.nan
    f[8] *= np.float32(1e37)       # overflow to inf inside the iterations
    f[9, ::2] = np.float32(3.4e38)
    cases["f32_specials_wimax576_r12"] = (mm2, f, R.Arithmetic.Float32, 6, False, False)
    fe = f.copy()
    cases["f32_specials_wimax576_r12_et"] = (mm2, fe, R.Arithmetic.Float32, 6, True, False)
    g = rng.standard_normal((8, mm2.n)).astype(np.float32)
    g[0] = 0.0
    g[1, ::2] = -0.0
    g[2] = np.round(g[2] * 2) / 2
    cases["f32_zeros_ties_wimax576_r12"] = (mm2, g, R.Arithmetic.Float32, 5, False, True)
    for name, (mm, vals, arith, iters, early, with_post) in cases.items():
        h = R.expand(mm)
        hard, it, conv = ref_decode(h, vals, arith, iters, early)
        extra = {}
        if with_post:
            extra["post"] = np.stack([tier_sweeps(h, vals[w], arith, iters, early)[0]
                                      for w in range(vals.shape[0])])
            assert np.array_equal((extra["post"] <= 0).astype(np.uint8), hard)
        std = mm.standard.value
        np.savez_compressed(OUT / f"special_{name}.npz", standard=std, n_bits=mm.n,
                            rate=mm.rate.value, arithmetic=arith.value, max_iters=iters,
                            early_term=int(early), llr=vals,
                            hard_packed=np.packbits(hard, axis=-1), iters=it, conv=conv, **extra)
        print(name, "iters", it, "conv", conv)


def make_encode():
    rng = np.random.default_rng(1003)
    arrs = {}
    for n, rate in [(2304, "3/4A"), (2304, "1/2"), (2304, "5/6"), (576, "1/2"), (576, "5/6"),
                    (1536, "3/4B"), (768, "2/3A"), (960, "2/3B"), (1920, "3/4A"), (1152, "1/2")]:
        mm = R.get_model_matrix("wimax", n, rate)
        info = rng.integers(0, 2, size=(64, mm.k), dtype=np.uint8)
        ib = R.pack_bits(info)
        for wb in (8, 16, 32):
            if mm.z % wb:
                continue
            cw = R.encode_packed(R.make_plan(mm, R.EncoderVariant.Packed, word_bits=wb), ib)
            assert np.array_equal(cw, R.pack_bits(R.encode_array(R.make_plan(mm), info)))
            arrs[f"cw_{n}_{rate.replace('/', '')}_{wb}"] = cw
        arrs[f"info_{n}_{rate.replace('/', '')}"] = ib
    np.savez_compressed(OUT / "encode_packed.npz", **arrs)
    print("encode fixtures", len(arrs))


def make_kat():
    toy = R.ModelMatrix(R.Standard.Wimax, R.Rate.R12, 1, 3, 2, np.array([[0, 0, 0]], np.int32))
    h = R.expand(toy)
    st = R.init_state(h, R.LlrBlock(np.array([3.0, -1.0, 2.0], np.float32)))
    R.tier_update(st, h, 0)
    st16 = R.init_state(h, R.LlrBlock(np.array([3, -1, 2], np.int16), R.Arithmetic.Fixed16))
    R.tier_update(st16, h, 0)
    q = R.quantize_llr(np.array([0.0, 24.0, -24.0, 100.0, -100.0, 12.0, -12.0])).values
    q4 = R.quantize_llr(np.array([24.0, 3.2, -24.0]), q_b=4).values
    zero = R.decode(h, R.LlrBlock(np.zeros(3, np.float32)), R.DecoderConfig(max_iterations=3))
    # edge_i16: the int16 tier update on [-32768, 5, 7] (min1 = -32768)
    ste = R.init_state(h, R.LlrBlock(np.array([-32768, 5, 7], np.int16), R.Arithmetic.Fixed16))
    R.tier_update(ste, h, 0)
    np.savez(OUT / "kat.npz",
             deg3_post_f32=st.posterior, deg3_min1=st.min1, deg3_min2=st.min2,
             deg3_argmin=st.argmin, deg3_sign_bits=st.sign_bits, deg3_sign_prod=st.sign_prod,
             deg3_post_i16=st16.posterior, quant_in=np.array([0.0, 24.0, -24.0, 100.0, -100.0, 12.0, -12.0]),
             quant_out=q, quant4_out=q4, zero_hard=zero.hard_bits, zero_iters=zero.iterations,
             zero_conv=int(zero.converged), wrap_post=ste.posterior, wrap_min1=ste.min1,
             wrap_min2=ste.min2)
    print("kat", st.posterior, ste.posterior, ste.min1)


def make_acceptance():
    import hashlib
    mm = R.get_model_matrix(R.Standard.Wimax, 576, R.Rate.R12)
    h = R.expand(mm)
    arrs = {}
    for arith, fixed in ((R.Arithmetic.Fixed16, True), (R.Arithmetic.Float32, False)):
        vals, _, _ = noisy(mm, 1000, 1.8, 1004, fixed)
        hard, iters, conv = ref_decode(h, vals, arith, 10, True)
        for w in range(vals.shape[0]):     # the reference test's own oracle comparison
            eh, ei, ec = RR.ref_decode(h, vals[w])
            assert np.array_equal(hard[w], eh) and iters[w] == ei and bool(conv[w]) == bool(ec), w
        tag = "i16" if fixed else "f32"
        arrs[f"llr_sha256_{tag}"] = np.frombuffer(hashlib.sha256(vals.tobytes()).digest(), np.uint8)
        arrs[f"hard_packed_{tag}"] = np.packbits(hard, axis=-1)
        arrs[f"iters_{tag}"] = iters
        arrs[f"conv_{tag}"] = conv
    np.savez_compressed(OUT / "acceptance_decoder_oracle.npz", standard="wimax", n_bits=576, rate="1/2",
                        frames=1000, ebn0_db=1.8, seed=1004, max_iters=10, early_term=1, **arrs)
    print("acceptance: 1000 frames x 2 arithmetics equal to _reference.ref_decode")


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    steps = {"kat": make_kat, "encode": make_encode, "special": make_special, "decode": make_decode,
             "acceptance": make_acceptance}
    for name in (sys.argv[1:] or list(steps)):
        steps[name]()
