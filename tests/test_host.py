"""CPU-side checks: the C ABI library, the host mirror of the reference API
(codebook / validation / quantizer / white-box tier update), no GPU needed."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import _lib
from tests._util import golden_cases, load_case

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "qcb200.h").read_text()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(qc_\w+)\(", header, re.M))
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.qc_version() == 110


def test_code_handles_without_gpu():
    # host-only entry points work with no device present
    for std, n, rate in P.supported_codes():
        mm = P.get_model_matrix(std, n, rate)
        c = _lib.Code(mm.entries, mm.z)
        assert c.specialised and c.n == mm.n and c.edges == mm.edges
        assert c.max_row_degree == int((mm.entries >= 0).sum(axis=1).max())
    toy = _lib.Code(np.array([[0, 0, 0]]), 1)
    assert not toy.specialised
    with pytest.raises(P.UnsupportedCode):
        _lib.Code(np.zeros((1, 40), np.int32), 4)        # row degree 40 > 32
    with pytest.raises(ValueError):
        _lib.Code(np.array([[0, 5, 0]]), 4)               # shift outside [-1, z)


def test_csr_recovery_matches_model_matrix():
    L = _lib.lib()
    for std, n, rate in list(P.supported_codes())[::7]:
        mm = P.get_model_matrix(std, n, rate)
        h = P.expand(mm)
        out = C.c_void_p()
        rc = L.qc_code_from_csr(h.row_ptr.ctypes.data, h.row_ptr.size, h.row_cols.ctypes.data,
                                h.row_cols.size, mm.mb, mm.z, mm.n, C.byref(out))
        assert rc == 0
        L.qc_code_destroy(out)
        tab = P.codebook.shift_table_from_csr(h.row_ptr, h.row_cols, mm.mb, mm.z, mm.n)
        assert np.array_equal(tab, mm.entries)
    # a non-QC CSR is refused (no generic-sparse fallback)
    mm = P.get_model_matrix("wimax", 576, "1/2")
    h = P.expand(mm)
    bad = h.row_cols.copy()
    bad[5], bad[6] = bad[6], bad[5]
    out = C.c_void_p()
    assert L.qc_code_from_csr(h.row_ptr.ctypes.data, h.row_ptr.size, bad.ctypes.data, bad.size,
                              mm.mb, mm.z, mm.n, C.byref(out)) == _lib.QC_EUNSUPPORTED
    with pytest.raises(ValueError):
        P.codebook.shift_table_from_csr(h.row_ptr, bad, mm.mb, mm.z, mm.n)


def test_decoder_validation_matches_reference_order():
    h = P.expand(P.get_model_matrix("wimax", 576, "1/2"))
    cfg = P.DecoderConfig()
    with pytest.raises(ValueError):
        P.DecoderConfig(max_iterations=0)
    with pytest.raises(ValueError):
        P.DecoderConfig(q_b=15)
    with pytest.raises(P.ArithmeticMismatch):
        P.decode(h, P.LlrBlock(np.zeros(h.n, np.float32)), P.DecoderConfig(arithmetic=P.Arithmetic.Fixed16))
    with pytest.raises(P.SizeMismatch):
        P.decode(h, P.LlrBlock(np.zeros(h.n - 1, np.float32)), cfg)
    with pytest.raises(P.SizeMismatch):
        P.decode(h, P.LlrBlock(np.zeros((2, h.n), np.float32)), cfg)
    with pytest.raises(P.SizeMismatch):
        P.decode_block(h, P.LlrBlock(np.zeros(h.n, np.float32)), cfg)
    with pytest.raises(ValueError):
        P.decode_block(h, P.LlrBlock(np.zeros((2, h.n), np.float32)), cfg, workers=0)
    with pytest.raises(ValueError):
        P.decode_block(h, P.LlrBlock(np.zeros((2, h.n), np.float32)), cfg, pool="x")
    assert P.decode_block(h, P.LlrBlock(np.empty((0, h.n), np.float32)), cfg) == []


def test_quantizer_reference_points(golden_dir):
    kat = np.load(golden_dir / "kat.npz")
    q = P.quantize_llr(kat["quant_in"])
    assert q.arithmetic is P.Arithmetic.Fixed16
    assert np.array_equal(q.values, kat["quant_out"])
    assert np.array_equal(q.values, [0, 1023, -1023, 1023, -1023, 512, -512])
    assert np.array_equal(P.quantize_llr(np.array([24.0, 3.2, -24.0]), q_b=4).values, kat["quant4_out"])


def test_white_box_tier_update_known_answers(golden_dir):
    kat = np.load(golden_dir / "kat.npz")
    toy = P.ModelMatrix(P.Standard.Wimax, P.Rate.R12, 1, 3, 2, np.array([[0, 0, 0]]))
    h = P.expand(toy)
    st = P.init_state(h, P.LlrBlock(np.array([3.0, -1.0, 2.0], np.float32)))
    P.tier_update(st, h, 0)
    assert st.min1[0] == 1.0 and st.min2[0] == 2.0 and st.argmin[0] == 1
    assert st.sign_bits[0] == 0b010 and st.sign_prod[0] == 1
    assert np.array_equal(st.messages(h, 0), [-1.0, 2.0, -1.0])
    assert np.array_equal(st.posterior, kat["deg3_post_f32"])
    st = P.init_state(h, P.LlrBlock(np.array([-32768, 5, 7], np.int16), P.Arithmetic.Fixed16))
    P.tier_update(st, h, 0)
    assert np.array_equal(st.posterior, kat["wrap_post"]) and st.min1[0] == kat["wrap_min1"][0]


@pytest.mark.parametrize("name", golden_cases("decode")[:4])
def test_white_box_sweeps_reproduce_reference_posteriors(name):
    d = load_case(name)
    h, llr = d["h"], d["llr"]
    arith = P.Arithmetic.Float32 if llr.dtype == np.float32 else P.Arithmetic.Fixed16
    st = P.init_state(h, P.LlrBlock(llr[0], arith))
    it, ok = 0, False
    for k in range(int(d["max_iters"])):
        for t in range(h.m // h.z):
            P.tier_update(st, h, t)
        it = k + 1
        ok = P.syndrome_check(h, (st.posterior <= 0).astype(np.uint8))
        if ok and d["early_term"]:
            break
    assert it == d["iters"][0] and ok == bool(d["conv"][0])
    assert np.array_equal(st.posterior, d["post"][0])


def test_encoder_plans_and_rotations():
    mm = P.get_model_matrix("wimax", 2304, "3/4B")
    assert P.find_y(mm) == (2, 80)
    assert P.find_y(P.get_model_matrix("wimax", 576, "1/2")) == (5, 0)
    with pytest.raises(P.UnsupportedZ):
        P.make_plan(P.get_model_matrix("wifi", 648, "1/2"), P.EncoderVariant.Packed)
    with pytest.raises(P.UnsupportedZ):
        P.make_plan(P.get_model_matrix("wimax", 576, "1/2"), P.EncoderVariant.Packed, word_bits=16)
    a = np.array([0b10110001, 0b01011100, 0b11100111], dtype=np.uint8)
    out = P.cyclic_shift_packed(a, 3, 24)
    assert out[0] == ((a[2] << 5) & 0xFF) | (a[0] >> 3)
    rng = np.random.default_rng(7)
    for wb, dt in ((8, np.uint8), (16, np.uint16), (32, np.uint32)):
        x = rng.integers(0, 1 << wb, size=64 // wb, dtype=np.uint64).astype(dt)
        assert np.array_equal(P.cyclic_shift_inverse(P.cyclic_shift_packed(x, 13, 64), 13, 64), x)


def test_array_encoder_solves_parity_for_every_code():
    rng = np.random.default_rng(41)
    for std, n, rate in P.supported_codes():
        mm = P.get_model_matrix(std, n, rate)
        h = P.expand(mm)
        info = rng.integers(0, 2, size=(3, mm.k), dtype=np.uint8)
        cw = P.encode_array(P.make_plan(mm), info)
        assert not P.row_parities(h, cw).any(), (std, n, rate)
        assert np.array_equal(cw[:, :mm.k], info)


def test_channel_abi_validates_before_touching_the_device():
    # argument checks run on the host and return before any CUDA call, so
    # they are exercised here without a GPU (capi.cu qc_channel_llr ...).
    L = _lib.lib()
    buf = C.c_void_p(1)          # never dereferenced: every call fails first
    cases = [
        (L.qc_channel_llr, (buf, 4, 96, 0.0, None, 1, 0, 0, 0, 1.0, buf, None), "sigma2"),
        (L.qc_channel_llr, (buf, 4, 95, 1.0, None, 1, 0, 0, 0, 1.0, buf, None), "bad shape"),
        (L.qc_channel_llr, (buf, -1, 96, 1.0, None, 1, 0, 0, 0, 1.0, buf, None), "bad shape"),
        (L.qc_channel_llr, (buf, 4, 96, 1.0, None, 1, 0, 0, 15, 1.0, buf, None), "q_b"),
        (L.qc_channel_llr, (buf, 4, 96, 1.0, None, 1, 0, 0, 6, 0.0, buf, None), "l_clip"),
        (L.qc_channel_llr, (None, 4, 96, 1.0, None, 1, 0, 0, 0, 1.0, buf, None), "NULL"),
        (L.qc_quantize_llr, (buf, 8, 0, 1.0, buf, None), "q_b"),
        (L.qc_quantize_llr, (buf, 8, 6, -1.0, buf, None), "l_clip"),
        (L.qc_quantize_llr, (buf, -8, 6, 1.0, buf, None), "count"),
        (L.qc_count_errors, (buf, 1, buf, buf, 4, 96, 97, 256, buf, None), "bad shape"),
        (L.qc_count_errors, (buf, 1, buf, buf, 4, 96, 48, 0, buf, None), "bad shape"),
        (L.qc_count_errors, (buf, 1, None, buf, 4, 96, 48, 256, buf, None), "NULL"),
        (L.qc_pack_records, (buf, buf, buf, 4, 0, buf, None), "bad shape"),
        (L.qc_pack_records, (buf, None, buf, 4, 96, buf, None), "NULL"),
        (L.qc_frames_info, (1, 0, -1, 4, 48, buf, None), "negative"),
        (L.qc_frames_info, (1, 0, 0, 4, 48, None, None), "NULL"),
        (L.qc_encode_bits, (None, buf, 4, buf, None), "NULL"),
    ]
    for fn, args, why in cases:
        assert fn(*args) == _lib.QC_EINVAL, (fn.__name__, args)
        assert why in L.qc_last_error().decode(), (fn.__name__, L.qc_last_error())
    # empty work is a successful no-op
    assert L.qc_channel_llr(None, 0, 96, 1.0, None, 1, 0, 0, 0, 1.0, None, None) == 0
    assert L.qc_quantize_llr(None, 0, 6, 1.0, None, None) == 0
    assert L.qc_pack_records(None, None, None, 0, 96, None, None) == 0
    assert L.qc_frames_info(1, 0, 0, 0, 48, None, None) == 0


def test_device_call_refuses_non_cuda_devices():
    """_lib.DeviceCall guards every library call: CUDA device only, and every
    tensor of one call on that device (calls run on the tensors'
    device, not whatever device happens to be current)."""
    import torch
    from paper_2306_12063_b200 import _lib
    with pytest.raises(ValueError):
        _lib.DeviceCall("cpu")
    with pytest.raises(ValueError):
        _lib.DeviceCall("cuda:0", None, torch.zeros(2))


def test_bench_ring_of_batches_exceeds_l2():
    """bench.py steps a workload smaller than L2 (C1) through a ring of distinct
    batches: never reused inside warm-up + timed steps unless the ring already holds
    more than 2 x L2 of inputs."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("qcb_bench", Path(__file__).resolve().parents[1] / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    c1 = 1024 * (648 * 5 + 5)                                  # C1: LLR in + hard out + iters / conv
    for warmup, steps in ((5, 20), (10, 100), (5, 400), (3, 1)):
        n = bench.ring_slots(c1, warmup, steps)
        assert n * c1 > 2 * bench.L2_BYTES
        assert n >= min(warmup + steps, 256)
    assert bench.ring_slots(100_000, 5, 20) * 100_000 > 2 * bench.L2_BYTES   # tiny batches: above the cap
    assert bench.ring_slots(c1, 5, 20) == 25 or bench.ring_slots(c1, 5, 20) * c1 > 2 * bench.L2_BYTES
