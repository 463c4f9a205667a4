"""GPU parity at BASELINE sizes, the reference's acceptance case, and the host /
stream plumbing around the kernels.

* C1 (all 1,024 codewords vs the oracle), C4 (one decode_grouped over
  18 x 16,384, sampled), C5 (2^22 codewords = 19.3 GB of int16 LLRs, sampled
  uniformly and past the 2^31-element mark) -- each checked bit for bit against
  the CPU oracle (oracle/qc_oracle.c, pinned to the reference's outputs in
  tests/test_oracle_golden.py) plus size-independent properties.
* The decoder-oracle acceptance case of the reference
  (/root/reference/pkg/tests/test_acceptance.py:139-156) through decode_block.
* The drop-in host path (`_kernels.decode_batch_*`) with pageable and
  page-locked buffers; side streams and graph capture on the device path.
Inputs for the big configs come from the device channel keyed by global frame
index (workloads.shard_llrs), the same generator bench.py times.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2306_12063_b200 as P  # noqa: E402
from paper_2306_12063_b200 import _kernels, _lib  # noqa: E402
from paper_2306_12063_b200.workloads import WORKLOADS, shard_info, shard_llrs  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests._util import acceptance_case, noisy_llrs  # noqa: E402

pytestmark = pytest.mark.gpu


def _oracle_rows(mm, llr_t, outs, idx, iters, early=False):
    ti = torch.from_numpy(np.asarray(idx)).cuda()
    llr = llr_t[ti].cpu().numpy()
    oh, oi, oc = O.decode_batch(P.expand(mm), llr, iters, early, workers=8)
    hard, it, conv = (x[ti].cpu().numpy() for x in outs[:3])
    assert np.array_equal(hard, oh), "hard decisions differ from the oracle"
    assert np.array_equal(it, oi) and np.array_equal(conv, oc)


@pytest.mark.parametrize("fixed", [True, False])
def test_reference_acceptance_case_through_decode_block(fixed):
    """test_acceptance.py:139-156: 1000 noisy WiMAX 576 R1/2 frames at 1.8 dB,
    default config (10 iterations, early termination), both arithmetics."""
    h, llr, hard, iters, conv = acceptance_case(fixed)
    arith = P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32
    res = P.decode_block(h, P.LlrBlock(llr, arith), P.DecoderConfig(arithmetic=arith), workers=4, pool="mtx")
    assert np.array_equal(np.stack([r.hard_bits for r in res]), hard)
    assert [r.iterations for r in res] == iters.tolist()
    assert [r.converged for r in res] == conv.astype(bool).tolist()
    hb, ib, cb = P.decode_batch(h, llr, P.DecoderConfig(arithmetic=arith))
    assert np.array_equal(hb, hard) and np.array_equal(ib, iters) and np.array_equal(cb, conv)


def test_full_size_c1_every_codeword_vs_oracle():
    """C1: Wi-Fi 648 R1/2 float32, 10 iterations, 1024 codewords at 2.0 dB."""
    wl = WORKLOADS["C1"]
    mm = wl.model_matrices()[0]
    t = shard_llrs(wl, 0, 0, wl.w_per_code, "cuda")
    hard, it, conv, post = P.decode_batch(mm, t, wl.config(), posteriors=True)
    torch.cuda.synchronize()
    _oracle_rows(mm, t, (hard, it, conv), np.arange(wl.w_per_code), wl.iters)
    oh, oi, oc, op = O.decode_batch(P.expand(mm), t.cpu().numpy(), wl.iters, False, workers=8, want_post=True)
    assert np.array_equal(post.cpu().numpy(), op, equal_nan=True)


def test_full_size_c4_grouped_vs_oracle():
    """C4: all 18 codes x 16384 codewords in ONE decode_grouped call; 64 rows per
    code (half of them from the tail) vs the oracle; info-bit BER sane."""
    wl = WORKLOADS["C4"]
    mms = wl.model_matrices()
    llrs = [shard_llrs(wl, ci, 0, wl.w_per_code, "cuda") for ci in range(len(mms))]
    outs = P.decode_grouped(list(zip(mms, llrs)), wl.config())
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    for ci, (mm, t, o) in enumerate(zip(mms, llrs, outs)):
        idx = np.unique(np.concatenate([rng.integers(0, wl.w_per_code, 32),
                                        rng.integers(wl.w_per_code - 1024, wl.w_per_code, 32)]))
        _oracle_rows(mm, t, o, idx, wl.iters)
        assert (o[1] == wl.iters).all()
        info = shard_info(wl, ci, 0, wl.w_per_code, "cuda")
        ber = (o[0][:, :mm.k] != info).float().mean().item()
        assert ber < 0.05, (mm, ber)            # 3.0 dB: the decoder decodes


def test_full_size_c5_2pow22_sampled_past_2pow31():
    """C5: WiMAX 2304 R3/4A int16, 10 iterations, 2^22 codewords in one launch
    (19.3 GB of LLRs; element offsets up to 9.7e9).  Sampled rows vs the oracle
    (uniform + the last 4096), packed == packbits(unpacked) on the tail, a tail
    sub-batch decoded separately equals the same rows of the full launch, conv
    <=> zero syndrome, and the info-bit error rate near the raw channel's."""
    wl = WORKLOADS["C5"]
    mm = wl.model_matrices()[0]
    w = wl.w_per_code
    assert w == 1 << 22
    t = shard_llrs(wl, 0, 0, w, "cuda")
    assert t.shape[0] * mm.n > 2 ** 33
    hard, it, conv = P.decode_batch(mm, t, wl.config())
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([rng.integers(0, w, 512), rng.integers(w - 4096, w, 512), [w - 1]]))
    assert idx.max() * mm.n * 2 > 2 ** 31 * 8
    _oracle_rows(mm, t, (hard, it, conv), idx, wl.iters)
    tail = t[w - 5000:]
    hp, it2, cv2 = P.decode_batch(mm, tail, wl.config(), hard_packed=True)
    torch.cuda.synchronize()
    assert np.array_equal(hp.cpu().numpy(), np.packbits(hard[w - 5000:].cpu().numpy(), axis=-1))
    assert torch.equal(it2, it[w - 5000:]) and torch.equal(cv2, conv[w - 5000:])
    assert (it == wl.iters).all()
    par = P.row_parities(P.expand(mm), hard[w - 2048:].cpu().numpy())
    assert np.array_equal(conv[w - 2048:].cpu().numpy() == 1, ~par.any(axis=-1))
    # 2.0 dB is below this R3/4 code's threshold (raw channel BER ~6 %): the
    # decoded info bits sit near the raw BER -- a sanity bound, not a pin
    info = shard_info(wl, 0, w - 65536, w, "cuda")
    ber = (hard[w - 65536:, :mm.k] != info).float().mean().item()
    assert 0.0 < ber < 0.1, ber


@pytest.mark.parametrize("fixed", [True, False])
def test_host_dropin_pageable_and_pinned_agree(fixed):
    """`_kernels.decode_batch_*` (qc_decode_batch_*_host) on a block that spans
    several 32 MB chunks and a ragged tail: pageable numpy (pinned staging ring
    + copy pool) and page-locked buffers (direct DMA) both equal the device
    path, twice in a row (staging slots reused)."""
    mm = P.get_model_matrix("wimax", 2304, "3/4A" if fixed else "1/2")
    base, _, _ = noisy_llrs(mm, 4096, 2.0, seed=31, fixed=fixed)
    w = 4096 * 9 + 123                       # int16: 171 MB -> 6 chunks; float32: 11 chunks
    llr = np.ascontiguousarray(np.resize(base, (w, mm.n)))
    h = P.expand(mm)
    cfg = P.DecoderConfig(max_iterations=6, early_termination=False,
                          arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
    dh, di, dc = (x.cpu().numpy() for x in P.decode_batch(mm, torch.from_numpy(llr).cuda(), cfg))
    fn = _kernels.decode_batch_i16 if fixed else _kernels.decode_batch_f32
    for pinned in (False, True, False):
        if pinned:
            keep = (torch.from_numpy(llr).pin_memory(), torch.empty((w, mm.n), dtype=torch.uint8).pin_memory(),
                    torch.empty(w, dtype=torch.int32).pin_memory(), torch.empty(w, dtype=torch.uint8).pin_memory())
            src, hard, iters, conv = (x.numpy() for x in keep)
        else:
            src, hard, iters, conv = llr, np.empty((w, mm.n), np.uint8), np.empty(w, np.int32), np.empty(w, np.uint8)
        fn(h.row_ptr, h.row_cols, h.m // h.z, h.z, src, 6, 0, hard, iters, conv)
        assert np.array_equal(hard, dh) and np.array_equal(iters, di) and np.array_equal(conv, dc), pinned


def test_side_stream_and_graph_capture_of_a_generic_code():
    """decode_batch on a side stream (outputs / temporaries recorded on it) and
    inside a CUDA graph capture -- also for a generic-kernel code, whose tables
    qc_code_create uploads eagerly (no allocation on the first decode)."""
    rng = np.random.default_rng(3)
    ent = rng.integers(-1, 17, size=(4, 10))
    ent[:, 0] = rng.integers(0, 17, size=4)
    generic = P.ModelMatrix(P.Standard.Wimax, P.Rate.R12, 17, 10, 6, ent)
    for mm in (generic, P.get_model_matrix("wimax", 2304, "1/2")):
        h = P.expand(mm)
        llr = (rng.standard_normal((50, mm.n)) * 2).astype(np.float32)
        cfg = P.DecoderConfig(max_iterations=4, early_termination=False)
        oh, oi, oc = O.decode_batch(h, llr, 4, False)
        s = torch.cuda.Stream()
        t = torch.from_numpy(llr).cuda()
        s.wait_stream(torch.cuda.current_stream())
        hard, it, conv = P.decode_batch(mm, t, cfg, stream=s)
        s.synchronize()
        assert np.array_equal(hard.cpu().numpy(), oh) and np.array_equal(it.cpu().numpy(), oi)
        fresh = _lib.Code(mm.entries, mm.z)      # a new handle: its first decode is the captured one
        out = tuple(torch.zeros_like(x) for x in (hard, it, conv))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            P.decode_batch(fresh, t, cfg, out=out, stream=s)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out[0].cpu().numpy(), oh) and np.array_equal(out[2].cpu().numpy(), oc)
