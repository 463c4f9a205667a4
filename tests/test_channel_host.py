"""CPU checks of the channel / waterfall / wire-format host logic against
fixtures produced by the REFERENCE (tools/make_golden_channel.py): frame
generation, LLR arithmetic, the waterfall stop rule, LLR0 containers."""

import json
import math

import numpy as np
import pytest

import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import channel as CH, llrio
from tests._util import GOLDEN


def _channel_cases():
    return sorted(p.name for p in GOLDEN.glob("channel_*.npz"))


@pytest.mark.parametrize("name", _channel_cases())
def test_host_frames_and_llrs_match_reference(name):
    z = np.load(GOLDEN / name)
    mm = P.get_model_matrix(str(z["std"]), int(z["n"]), str(z["rate"]))
    info, noise = CH.gen_batch_host(mm, int(z["seed"]), int(z["point"]), int(z["start"]), z["info"].shape[0])
    assert np.array_equal(info, z["info"]) and np.array_equal(noise, z["noise"])
    cw = P.encode_array(P.make_plan(mm), info)
    assert np.array_equal(cw, z["cw"])
    s2 = CH.ebn0_to_sigma2(float(z["ebn0"]), mm.rate.fraction)
    assert s2 == float(z["sigma2"])
    samples = CH.bpsk_modulate(cw) + math.sqrt(s2) * noise           # chansim._llr_batch
    f32 = CH.llr_from_samples(samples, s2).values
    assert f32.dtype == np.float32 and np.array_equal(f32.view(np.uint32), z["llr_f32"].view(np.uint32))
    i16 = P.quantize_llr(f32, 10).values
    assert np.array_equal(i16, z["llr_i16"])


def _reference_loop(batches, max_frames, min_errors, min_frames):
    """The reference's per-point loop (chansim.py:163-176) over precomputed
    per-batch counters (bit_errors, frame_errors, iter_sum)."""
    frames = be = fe = it = 0
    i = 0
    while True:
        count = min(CH.BATCH_FRAMES, max_frames - frames)
        if count <= 0:
            break
        b = batches[i]
        i += 1
        be += b[0]; fe += b[1]; it += b[2]
        frames += count
        if be >= min_errors and frames >= min_frames:
            break
    return [frames, be, fe, it]


@pytest.mark.parametrize("seed", range(8))
def test_chunked_stop_rule_equals_reference_loop(seed):
    rng = np.random.default_rng(seed)
    max_frames = int(rng.integers(1, 6000))
    min_errors = int(rng.integers(1, 3000))
    min_frames = int(rng.integers(1, 3000))
    nb = (max_frames + 255) // 256
    batches = np.stack([rng.integers(0, 200, nb), rng.integers(0, 20, nb), rng.integers(0, 2000, nb)], 1)
    want = _reference_loop(batches, max_frames, min_errors, min_frames)
    for chunk in (256, 512, 2048, 65536):
        state, b0 = [0, 0, 0, 0], 0
        while True:
            count = min(chunk, max_frames - state[0])
            if count <= 0:
                break
            nbt = (count + 255) // 256
            counts = [min(256, count - j * 256) for j in range(nbt)]
            if CH._walk_batches(batches[b0:b0 + nbt], counts, state, min_errors, min_frames):
                break
            b0 += nbt
        assert state == want, (chunk, state, want)


def test_waterfall_csv_format_matches_reference_fixture():
    text = (GOLDEN / "waterfall_wimax576_r12_f32.csv").read_text()
    rows = [r.split(",") for r in text.strip().splitlines()[1:]]
    pts = [CH.WaterfallPoint(float(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), float(r[7])) for r in rows]
    # the fixture's own avg_iters column is rounded to 6 digits: round-trip the other columns
    out = CH.WaterfallTable(pts).to_csv().splitlines()
    for got, want in zip(out, text.splitlines()):
        assert got.split(",")[:7] == want.split(",")[:7]
    assert out[0] == CH.WaterfallTable.CSV_HEADER


def test_sigma_and_channel_validation():
    with pytest.raises(ValueError):
        CH.ebn0_to_sigma2(1.0, 0.0)
    with pytest.raises(P.DivByZeroSigma):
        CH.llr_from_samples(np.zeros(4), 0.0)
    with pytest.raises(ValueError):
        CH.awgn(np.zeros(4), -1.0, np.random.default_rng(0))
    assert np.array_equal(CH.awgn(np.ones(3), 0.0, np.random.default_rng(0)), np.ones(3))
    cfg = CH.ChannelConfig(2.0, 0.5)
    assert cfg.sigma2 == CH.ebn0_to_sigma2(2.0, 0.5)


@pytest.mark.parametrize("name", ["wimax576_r12_f32", "wimax576_r12_i16"])
def test_llr0_container_round_trip_matches_reference_bytes(name, tmp_path):
    src = GOLDEN / f"llr0_{name}.llr"
    block = llrio.read_llr_file(src)
    assert block.values.shape[1] == 576
    out = tmp_path / "x.llr"
    llrio.write_llr_file(out, block)
    assert out.read_bytes() == src.read_bytes()


def test_llr0_container_errors(tmp_path):
    good = (GOLDEN / "llr0_wimax576_r12_f32.llr").read_bytes()
    cases = {"trunc": good[:10], "magic": b"LLR1" + good[4:], "arith": good[:12] + b"\x07" + good[13:],
             "payload": good[:-3]}
    for k, data in cases.items():
        p = tmp_path / f"{k}.llr"
        p.write_bytes(data)
        with pytest.raises(P.CorruptFile):
            llrio.read_llr_file(p)


def test_records_fixture_layout():
    meta = json.loads((GOLDEN / "records_cases.json").read_text())
    for name in meta:
        block = llrio.read_llr_file(GOLDEN / f"llr0_{name}.llr")
        rec = (GOLDEN / f"records_{name}.bin").read_bytes()
        assert len(rec) == block.values.shape[0] * (576 // 8 + 2)
