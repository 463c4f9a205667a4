"""GPU tests of the device channel, waterfall loop and wire formats
 against fixtures produced by the REFERENCE
(tools/make_golden_channel.py) and the reference's statistical pins."""

import json
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2306_12063_b200 as P  # noqa: E402
from paper_2306_12063_b200 import channel as CH, llrio  # noqa: E402
from tests._util import GOLDEN  # noqa: E402

pytestmark = pytest.mark.gpu


def _cases(prefix, ext):
    return sorted(p.name for p in GOLDEN.glob(f"{prefix}_*.{ext}"))


@pytest.mark.parametrize("name", _cases("channel", "npz"))
def test_device_encoder_and_channel_bit_exact_with_reference(name):
    z = np.load(GOLDEN / name)
    mm = P.get_model_matrix(str(z["std"]), int(z["n"]), str(z["rate"]))
    info = torch.from_numpy(z["info"]).cuda()
    cw = CH.encode_array_device(mm, info)
    assert np.array_equal(cw.cpu().numpy(), z["cw"])
    noise = torch.from_numpy(z["noise"]).cuda()
    s2 = float(z["sigma2"])
    f32 = CH.channel_llr_device(cw, s2, P.Arithmetic.Float32, noise=noise).cpu().numpy()
    assert np.array_equal(f32.view(np.uint32), z["llr_f32"].view(np.uint32))
    i16 = CH.channel_llr_device(cw, s2, P.Arithmetic.Fixed16, q_b=10, noise=noise).cpu().numpy()
    assert np.array_equal(i16, z["llr_i16"])


def test_device_array_encoder_all_codes():
    rng = np.random.default_rng(77)
    for std, n, rate in P.supported_codes():
        mm = P.get_model_matrix(std, n, rate)
        info = rng.integers(0, 2, size=(37, mm.k), dtype=np.uint8)
        got = CH.encode_array_device(mm, torch.from_numpy(info).cuda()).cpu().numpy()
        assert np.array_equal(got, P.encode_array(P.make_plan(mm), info)), (std, n, rate)


def test_device_quantizer_matches_host_quantizer():
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(1 << 16) * 20).astype(np.float32)
    lim_over = 1023 / 24.0
    ties = ((np.arange(-2000, 2000) + 0.5) / lim_over).astype(np.float32)    # near half-way points
    extra = np.array([0.0, -0.0, 1e30, -1e30, np.inf, -np.inf, 24.0, -24.0, 23.99], np.float32)
    x = np.concatenate([x, ties, extra])
    for qb in (1, 6, 10, 14):
        got = CH.quantize_llr_device(torch.from_numpy(x).cuda(), q_b=qb).cpu().numpy()
        assert np.array_equal(got, P.quantize_llr(x, qb).values), qb


@pytest.mark.parametrize("name", [n[len("waterfall_"):-4] for n in _cases("waterfall", "csv")])
def test_waterfall_with_reference_frames_equals_reference_table(name):
    meta = json.loads((GOLDEN / "waterfall_cases.json").read_text())[name]
    mm = P.get_model_matrix(meta["std"], meta["n"], meta["rate"])
    cfg = P.DecoderConfig(max_iterations=meta["max_iterations"], arithmetic=P.Arithmetic(meta["arithmetic"]))
    table = CH.run_waterfall(mm, cfg, meta["snrs"], min_errors=meta["min_errors"], max_frames=meta["max_frames"],
                             seed=meta["seed"], min_frames=meta["min_frames"], frames="reference")
    assert table.to_csv() == (GOLDEN / f"waterfall_{name}.csv").read_text()


def test_waterfall_device_frames_calibrated_operating_points():
    """The reference's operating-point pins (test_acceptance.py:159-179):
    N=2304 R1/2, float32, 8 iterations; 2.0 dB: BER in [1.25e-3, 2.8e-3]
    and 6.36 +/- 0.5 iterations; 1.0 dB: 8.00 +/- 0.2 iterations."""
    mm = P.get_model_matrix("wimax", 2304, "1/2")
    cfg = P.DecoderConfig(max_iterations=8)
    table = CH.run_waterfall(mm, cfg, [1.0, 2.0], min_errors=10000, max_frames=20480, seed=7, min_frames=2048)
    p1, p2 = table.points
    assert 1.25e-3 <= p2.ber <= 2.8e-3, p2
    assert abs(p2.avg_iterations - 6.36) <= 0.5, p2
    assert abs(p1.avg_iterations - 8.00) <= 0.2, p1
    assert p1.bit_errors >= 10000 and p2.bit_errors >= 10000


def test_waterfall_device_frames_independent_of_chunking():
    mm = P.get_model_matrix("wimax", 576, "1/2")
    cfg = P.DecoderConfig(max_iterations=6, arithmetic=P.Arithmetic.Fixed16)
    a = CH.run_waterfall(mm, cfg, [2.0, 3.0], min_errors=500, max_frames=6000, seed=3, chunk_frames=256)
    b = CH.run_waterfall(mm, cfg, [2.0, 3.0], min_errors=500, max_frames=6000, seed=3, chunk_frames=1 << 16)
    assert a.to_csv() == b.to_csv()


def test_device_frames_are_counter_keyed_and_balanced():
    dev = torch.device("cuda", 0)
    a = CH.frames_info_device(9, 2, 0, 40, 1000, dev)
    b = CH.frames_info_device(9, 2, 13, 27, 1000, dev)
    assert torch.equal(a[13:], b)
    c = CH.frames_info_device(9, 3, 0, 40, 1000, dev)
    assert not torch.equal(a, c)
    big = CH.frames_info_device(1, 0, 0, 4096, 2304, dev).double()
    assert set(torch.unique(big).tolist()) <= {0.0, 1.0}
    assert abs(big.mean().item() - 0.5) < 0.002


def test_device_noise_is_standard_normal():
    n, w = 2304, 512
    bits = torch.zeros((w, n), dtype=torch.uint8, device="cuda")
    s2 = 0.5
    llr = CH.channel_llr_device(bits, s2, seed=4, point=1).double()
    g = (llr * s2 / 2.0 - 1.0) / math.sqrt(s2)                  # invert y = 1 + sqrt(s2) g, llr = 2y/s2
    m, v = g.mean().item(), g.var().item()
    assert abs(m) < 0.005 and abs(v - 1.0) < 0.01, (m, v)
    k4 = ((g - m) ** 4).mean().item() / v ** 2
    assert abs(k4 - 3.0) < 0.05


@pytest.mark.parametrize("name", sorted(json.loads((GOLDEN / "records_cases.json").read_text())))
def test_decode_llr_file_writes_reference_records(name, tmp_path):
    meta = json.loads((GOLDEN / "records_cases.json").read_text())[name]
    mm = P.get_model_matrix(meta["std"], meta["n"], meta["rate"])
    cfg = P.DecoderConfig(max_iterations=meta["max_iterations"], early_termination=meta["early_termination"])
    out = tmp_path / "rec.bin"
    llrio.decode_llr_file(mm, GOLDEN / f"llr0_{name}.llr", out, cfg)
    assert out.read_bytes() == (GOLDEN / f"records_{name}.bin").read_bytes()


def test_pack_records_clamps_iterations():
    hard = torch.arange(3 * 2, dtype=torch.uint8, device="cuda").reshape(3, 2)
    iters = torch.tensor([0, 255, 300], dtype=torch.int32, device="cuda")
    conv = torch.tensor([1, 0, 7], dtype=torch.uint8, device="cuda")
    rec = llrio.pack_records_device(hard, iters, conv, 16).cpu().numpy()
    assert rec.tolist() == [[0, 1, 0, 1], [2, 3, 255, 0], [4, 5, 255, 1]]


def test_throughput_bench_report():
    mm = P.get_model_matrix("wimax", 2304, "1/2")
    rep = CH.run_throughput_bench(mm, P.DecoderConfig(), frames=4096)
    assert rep.frames == 4096 and rep.info_bits == 4096 * mm.k and rep.mbps > 0
    assert rep.csv_line().startswith("float32,1,cuda,4096,")


def _crossing_db(points, target=1e-4):
    """Eb/N0 where a BER curve crosses `target`, log-linear between points."""
    pts = sorted(points)
    for (x0, b0), (x1, b1) in zip(pts, pts[1:]):
        if b0 >= target >= b1 > 0.0:
            return x0 if b0 == b1 else x0 + math.log(b0 / target) / math.log(b0 / b1) * (x1 - x0)
    raise AssertionError(f"target BER {target} not bracketed by {pts}")


def test_fixed_point_penalty_within_budget():
    """The reference's fixed-point pin (test_acceptance.py:182-205) on device
    frames: int16 decoding crosses BER 1e-4 at most 0.15 dB (Wi-Fi 1944 R1/2)
    / 0.05 dB (WiMAX 576 R5/6) right of float32, same noise for both."""
    cases = [(("wifi", 1944, "1/2"), [2.1, 2.25, 2.4], 400, 20000, 0.15),
             (("wimax", 576, "5/6"), [4.0, 4.25, 4.5], 350, 25000, 0.05)]
    for code, snrs, min_err, max_frames, budget in cases:
        mm = P.get_model_matrix(*code)
        cross = {}
        for arith in (P.Arithmetic.Float32, P.Arithmetic.Fixed16):
            table = CH.run_waterfall(mm, P.DecoderConfig(arithmetic=arith), snrs, min_errors=min_err,
                                     max_frames=max_frames, seed=1006)
            cross[arith] = _crossing_db([(p.ebn0_db, p.ber) for p in table.points])
        penalty = cross[P.Arithmetic.Fixed16] - cross[P.Arithmetic.Float32]
        assert penalty <= budget, (code, penalty)


def test_rate_curves_keep_order():
    """test_acceptance.py:208-241 on device frames: with >= 1e4 bit errors per
    point a lower rate never shows a higher BER at the same Eb/N0 and every
    curve is monotone (Wi-Fi 1944, four rates)."""
    plans = [("1/2", [2.3], 400_000), ("2/3", [2.3, 2.7], 60_000),
             ("3/4", [2.3, 2.7, 3.1], 60_000), ("5/6", [2.3, 2.7, 3.1], 60_000)]
    curves = {}
    for rate, snrs, max_frames in plans:
        mm = P.get_model_matrix("wifi", 1944, rate)
        table = CH.run_waterfall(mm, P.DecoderConfig(), snrs, min_errors=10000, max_frames=max_frames, seed=1007)
        for p in table.points:
            assert p.bit_errors >= 10000, (rate, p)
        curves[mm.rate.fraction] = {p.ebn0_db: p.ber for p in table.points}
    comparisons = 0
    for snr in (2.3, 2.7, 3.1):
        ladder = sorted((frac, bers[snr]) for frac, bers in curves.items() if snr in bers)
        for (_, b_lo), (_, b_hi) in zip(ladder, ladder[1:]):
            comparisons += 1
            assert b_lo <= b_hi, (snr, ladder)
    assert comparisons == 6
    for bers in curves.values():
        assert (np.diff([bers[s] for s in sorted(bers)]) <= 0).all(), bers
