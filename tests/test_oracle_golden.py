"""Pin the CPU oracle (oracle/qc_oracle.c) to the reference's own outputs.

Fixtures in tests/golden/ were produced by running the reference package
(`tools/make_golden.py`): `decode_block` (kernel outputs), `init_state` +
`tier_update` sweeps (posteriors), `encode_packed`, and the known answers of
`pkg/tests/test_decoder.py:74-91, 103-110, 274-289`.  The oracle must agree
bit for bit before it is trusted as the checker of the CUDA path.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2306_12063_b200 import codebook as CB
from tests._util import golden_cases, load_case


@pytest.mark.parametrize("name", golden_cases("decode") + golden_cases("special"))
def test_oracle_matches_reference_kernel(name):
    d = load_case(name)
    hard, iters, conv, post = O.decode_batch(d["h"], d["llr"], int(d["max_iters"]),
                                             bool(d["early_term"]), workers=4, want_post=True)
    assert np.array_equal(hard, d["hard"])
    assert np.array_equal(iters, d["iters"])
    assert np.array_equal(conv, d["conv"])
    if "post" in d:
        k = d["post"].shape[0]
        # bitwise: compare the raw bit patterns (float -0.0 vs +0.0 matters)
        assert np.array_equal(post[:k].view(np.uint8), d["post"].view(np.uint8))


def test_oracle_worker_invariance():
    d = load_case("decode_wimax576_r12_f32_et.npz")
    base = O.decode_batch(d["h"], d["llr"], 10, True, workers=1)
    for w in (2, 3, 7):
        got = O.decode_batch(d["h"], d["llr"], 10, True, workers=w)
        assert all(np.array_equal(a, b) for a, b in zip(base, got))


def test_oracle_known_answers(golden_dir):
    kat = np.load(golden_dir / "kat.npz")
    toy = CB.ModelMatrix(CB.Standard.Wimax, CB.Rate.R12, 1, 3, 2, np.array([[0, 0, 0]]))
    h = CB.expand(toy)
    # degree-3 row by hand (reference test_decoder.py:74-91): one tier sweep
    _, _, _, post = O.decode_batch(h, np.array([[3.0, -1.0, 2.0]], np.float32), 1, False,
                                   want_post=True)
    assert np.array_equal(post[0], kat["deg3_post_f32"]) and np.array_equal(post[0], [2.0, 1.0, 1.0])
    _, _, _, post = O.decode_batch(h, np.array([[3, -1, 2]], np.int16), 1, False, want_post=True)
    assert np.array_equal(post[0], kat["deg3_post_i16"])
    # int16 wrap: abs(-32768) stays -32768 and wins the min
    _, _, _, post = O.decode_batch(h, np.array([[-32768, 5, 7]], np.int16), 1, False, want_post=True)
    assert np.array_equal(post[0], kat["wrap_post"])
    # all-zero LLRs: all ones, never converges (test_decoder.py:103-110)
    hard, iters, conv = O.decode_batch(h, np.zeros((1, 3), np.float32), 3, True)
    assert np.array_equal(hard[0], kat["zero_hard"]) and iters[0] == 3 and conv[0] == 0


def test_oracle_encoder_matches_reference(golden_dir):
    z = np.load(golden_dir / "encode_packed.npz")
    checked = 0
    for key in z.files:
        if not key.startswith("cw_"):
            continue
        _, n, rate, wb = key.split("_")
        rate = rate[0] + "/" + rate[1:]
        mm = CB.get_model_matrix("wimax", int(n), rate)
        got = O.encode_packed(mm, z[f"info_{n}_{rate.replace('/', '')}"], int(wb))
        assert np.array_equal(got, z[key]), key
        checked += 1
    assert checked >= 20


@pytest.mark.parametrize("fixed", [True, False])
def test_oracle_matches_reference_acceptance_case(fixed):
    """test_acceptance.py:139-156 (decoder-oracle): 1000 noisy frames per
    arithmetic, hard bits / iterations / converged equal to the reference's."""
    from tests._util import acceptance_case
    h, llr, hard, iters, conv = acceptance_case(fixed)
    oh, oi, oc = O.decode_batch(h, llr, 10, True, workers=4)
    assert np.array_equal(oh, hard) and np.array_equal(oi, iters) and np.array_equal(oc, conv)
