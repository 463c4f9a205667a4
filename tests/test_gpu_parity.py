"""GPU parity: libqcb200's sm_100a decoder/encoder vs the reference's outputs.

Every test here runs the CUDA path through the C ABI (device entry points via
`decode_batch`, host entry points via the drop-in `_kernels` / `decode_block`)
and compares bit for bit -- hard decisions, iteration counts, convergence
flags and posterior LLR bit patterns -- with
  * golden fixtures produced by the reference itself (tests/golden, made by
    tools/make_golden.py), and
  * the CPU oracle (oracle/qc_oracle.c, pinned to those fixtures in
    tests/test_oracle_golden.py) on seeded inputs for all 126 codes.
Tolerance: none.  int16 is bit-exact by definition; float32 is bit-exact
too (identical IEEE operations in identical order), which is stricter than
the 1e-5 relative bound north_star allows.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2306_12063_b200 as P  # noqa: E402
from paper_2306_12063_b200 import _kernels  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests._util import golden_cases, load_case, noisy_llrs  # noqa: E402

pytestmark = pytest.mark.gpu


def _cfg(d):
    arith = P.Arithmetic.Float32 if str(d["arithmetic"]) == "float32" else P.Arithmetic.Fixed16
    return P.DecoderConfig(max_iterations=int(d["max_iters"]), arithmetic=arith,
                           early_termination=bool(d["early_term"]))


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint16)


def _post_equal(got, want):
    """int16: bitwise.  float32: bitwise except the sign of an exact zero and
    NaN payloads -- the specialised kernel canonicalises -0.0 inputs to +0.0
    (see ArithF32::canon in csrc/decode_layered.cuh), which can flip the sign
    of a zero posterior; values compare equal and every decision is identical.
    north_star allows 1e-5 relative for float posteriors."""
    got, want = np.asarray(got), np.asarray(want)
    if got.dtype == np.int16:
        return np.array_equal(got, want)
    return np.array_equal(got, want, equal_nan=True)


def _gpu(mm, llr, cfg, posteriors=True, hard_packed=False):
    out = P.decode_batch(mm, torch.from_numpy(llr).cuda(), cfg, posteriors=posteriors,
                         hard_packed=hard_packed)
    torch.cuda.synchronize()
    return [None if t is None else t.cpu().numpy() for t in out]


@pytest.mark.parametrize("name", golden_cases("decode") + golden_cases("special"))
def test_device_path_matches_reference_goldens(name):
    d = load_case(name)
    hard, iters, conv, post = _gpu(d["mm"], d["llr"], _cfg(d))
    assert np.array_equal(hard, d["hard"])
    assert np.array_equal(iters, d["iters"])
    assert np.array_equal(conv, d["conv"])
    if "post" in d:
        k = d["post"].shape[0]
        assert _post_equal(post[:k], d["post"])
    hp, _, _ = _gpu(d["mm"], d["llr"], _cfg(d), posteriors=False, hard_packed=True)
    assert np.array_equal(hp, d["hard_packed"])


@pytest.mark.parametrize("name", golden_cases("decode") + golden_cases("special"))
def test_dropin_kernel_boundary_matches_goldens(name):
    """The reference's own kernel signature (_kernels.py:17-19), host buffers."""
    d = load_case(name)
    h, llr = d["h"], d["llr"]
    w = llr.shape[0]
    hard = np.empty((w, h.n), np.uint8)
    iters = np.empty(w, np.int32)
    conv = np.empty(w, np.uint8)
    fn = _kernels.decode_batch_f32 if llr.dtype == np.float32 else _kernels.decode_batch_i16
    fn(h.row_ptr, h.row_cols, h.m // h.z, h.z, llr, int(d["max_iters"]), int(d["early_term"]),
       hard, iters, conv)
    assert np.array_equal(hard, d["hard"]) and np.array_equal(iters, d["iters"])
    assert np.array_equal(conv, d["conv"])


def test_decode_block_api_matches_goldens():
    d = load_case("decode_wimax576_r12_f32_et.npz")
    cfg = _cfg(d)
    res = P.decode_block(d["h"], P.LlrBlock(d["llr"]), cfg, workers=4, pool="mtx")
    for w, r in enumerate(res):
        assert np.array_equal(r.hard_bits, d["hard"][w])
        assert r.iterations == d["iters"][w] and r.converged == bool(d["conv"][w])
        assert np.array_equal(r.info_bits, d["hard"][w][:d["mm"].k])
    one = P.decode(d["h"], P.LlrBlock(d["llr"][3]), cfg)
    assert np.array_equal(one.hard_bits, d["hard"][3]) and one.iterations == d["iters"][3]


@pytest.mark.parametrize("fixed", [False, True])
@pytest.mark.parametrize("early", [False, True])
def test_all_126_codes_match_oracle(fixed, early):
    """Every supported code (12 Wi-Fi + 114 WiMAX), seeded noisy inputs, vs the C oracle."""
    rng_seed = 100 + 2 * fixed + early
    for idx, (std, n, rate) in enumerate(P.supported_codes()):
        mm = P.get_model_matrix(std, n, rate)
        h = P.expand(mm)
        ebn0 = 1.5 + 2.0 * mm.rate.fraction
        llr, _, _ = noisy_llrs(mm, 5, ebn0, seed=rng_seed * 1000 + idx, fixed=fixed)
        iters = 6 if early else 4
        cfg = P.DecoderConfig(max_iterations=iters,
                              arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32,
                              early_termination=early)
        hard, it, conv, post = _gpu(mm, llr, cfg)
        oh, oi, oc, op = O.decode_batch(h, llr, iters, early, workers=4, want_post=True)
        assert np.array_equal(hard, oh), (std, n, rate)
        assert np.array_equal(it, oi) and np.array_equal(conv, oc), (std, n, rate)
        assert _post_equal(post, op), (std, n, rate)


C4_CODES = [("wifi", n, r) for n in (648, 1296, 1944) for r in ("1/2", "2/3", "3/4", "5/6")] + \
    [("wimax", 2304, r) for r in ("1/2", "2/3A", "2/3B", "3/4A", "3/4B", "5/6")]


@pytest.mark.parametrize("fixed", [False, True])
@pytest.mark.parametrize("early", [False, True])
def test_grouped_mixed_code_batch_matches_oracle(fixed, early):
    """BASELINE config 4's shape: all 18 codes (plus an empty job and a
    generic-kernel code) in ONE decode_grouped call, the jobs running
    concurrently on side streams; every job bit-identical to the oracle and
    to the serial per-code path."""
    rng = np.random.default_rng(41 + 2 * fixed + early)
    arith = P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32
    cfg = P.DecoderConfig(max_iterations=5, arithmetic=arith, early_termination=early)
    mms = [P.get_model_matrix(*c) for c in C4_CODES]
    ent = rng.integers(-1, 17, size=(4, 10))
    ent[:, 0] = rng.integers(0, 17, size=4)
    mms.append(P.ModelMatrix(P.Standard.Wimax, P.Rate.R12, 17, 10, 6, ent))      # generic kernel
    jobs, llrs = [], []
    for i, mm in enumerate(mms):
        w = 0 if i == 3 else 23 + 3 * i                                         # job 3 is empty
        if i < len(C4_CODES):
            llr, _, _ = noisy_llrs(mm, max(w, 1), 1.5 + 2.0 * mm.rate.fraction, seed=900 + i, fixed=fixed)
            llr = llr[:w]
        elif fixed:
            llr = rng.integers(-600, 600, size=(w, mm.n)).astype(np.int16)
        else:
            llr = (rng.standard_normal((w, mm.n)) * 2).astype(np.float32)
        llrs.append(llr)
        jobs.append((mm, torch.from_numpy(np.ascontiguousarray(llr)).cuda()))
    outs = P.decode_grouped(jobs, cfg)
    torch.cuda.synchronize()
    for (mm, t), llr, (hard, it, conv) in zip(jobs, llrs, outs):
        assert hard.shape == (llr.shape[0], mm.n)
        if llr.shape[0] == 0:
            continue
        oh, oi, oc = O.decode_batch(P.expand(mm), llr, 5, early, workers=4)
        assert np.array_equal(hard.cpu().numpy(), oh), mm
        assert np.array_equal(it.cpu().numpy(), oi) and np.array_equal(conv.cpu().numpy(), oc), mm
        serial = P.decode_batch(mm, t, cfg)
        for a, b in zip(serial, (hard, it, conv)):
            assert torch.equal(a, b)


def test_grouped_batch_graph_capture_and_preallocated_outputs():
    """The grouped call is stream-ordered: captured into a CUDA graph (fork /
    join of the side streams inside the capture) it replays to the same
    outputs; packed hard decisions equal np.packbits of the unpacked ones."""
    cfg = P.DecoderConfig(max_iterations=4, early_termination=False)
    mms = [P.get_model_matrix(*c) for c in C4_CODES[::3]]
    jobs = []
    for i, mm in enumerate(mms):
        llr, _, _ = noisy_llrs(mm, 40 + i, 2.5, seed=70 + i)
        jobs.append((mm, torch.from_numpy(llr).cuda()))
    ref = P.decode_grouped(jobs, cfg)
    packed = P.decode_grouped(jobs, cfg, hard_packed=True)
    torch.cuda.synchronize()
    outs = [tuple(torch.zeros_like(x) for x in o) for o in ref]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        P.decode_grouped(jobs, cfg, out=outs, stream=s)
    g.replay()
    torch.cuda.synchronize()
    for (mm, _), a, b, pk in zip(jobs, ref, outs, packed):
        for x, y in zip(a, b):
            assert torch.equal(x, y)
        assert np.array_equal(pk[0].cpu().numpy(), np.packbits(a[0].cpu().numpy(), axis=1))
    with pytest.raises(P.SizeMismatch):
        P.decode_grouped(jobs, cfg, out=[(o[0][:, :-1], o[1], o[2]) for o in outs])


def test_generic_kernel_on_nonstandard_codes():
    """Codes outside the 18 standard structures take the generic kernel."""
    rng = np.random.default_rng(7)
    toy = P.ModelMatrix(P.Standard.Wimax, P.Rate.R12, 1, 3, 2, np.array([[0, 0, 0]]))
    assert not P.code_handle(toy).specialised
    cases = [(toy, 3)]
    for z, mb, nb in [(5, 3, 9), (17, 4, 10), (40, 6, 16), (7, 2, 30)]:
        ent = rng.integers(-1, z, size=(mb, nb))
        ent[rng.random((mb, nb)) < 0.4] = -1
        ent[:, 0] = rng.integers(0, z, size=mb)
        cases.append((P.ModelMatrix(P.Standard.Wimax, P.Rate.R12, z, nb, nb - mb, ent), 5))
    for mm, iters in cases:
        h = P.expand(mm)
        for dt, arith in ((np.float32, P.Arithmetic.Float32), (np.int16, P.Arithmetic.Fixed16)):
            if dt == np.float32:
                llr = rng.standard_normal((9, mm.n)).astype(np.float32) * 2
            else:
                llr = rng.integers(-600, 600, size=(9, mm.n)).astype(np.int16)
            for early in (False, True):
                cfg = P.DecoderConfig(max_iterations=iters, arithmetic=arith, early_termination=early)
                hard, it, conv, post = _gpu(mm, llr, cfg)
                oh, oi, oc, op = O.decode_batch(h, llr, iters, early, want_post=True)
                assert np.array_equal(hard, oh) and np.array_equal(it, oi) and np.array_equal(conv, oc)
                assert _post_equal(post, op)


def test_standard_structure_with_foreign_shifts():
    """A standard zero-block pattern at its native Z (or at a scaled WiMAX Z) but with
    other shift values must not take the compile-time-shift kernels (decoder and
    encoder): the runtime-Z kernels serve it."""
    rng = np.random.default_rng(17)
    for std, n, rate in (("wimax", 2304, "1/2"), ("wimax", 2304, "3/4A"), ("wifi", 1944, "5/6"),
                         ("wifi", 648, "1/2"), ("wimax", 960, "3/4A"), ("wimax", 576, "2/3A")):
        base = P.get_model_matrix(std, n, rate)
        ent = base.entries.copy()
        nz = ent >= 0
        ent[nz] = rng.integers(0, base.z, size=int(nz.sum()))
        ent[:, base.kb:] = base.entries[:, base.kb:]          # keep the dual-diagonal part
        mm = P.ModelMatrix(base.standard, base.rate, base.z, base.nb, base.kb, ent)
        assert P.code_handle(mm).specialised
        h = P.expand(mm)
        for fixed in (False, True):
            llr, _, _ = noisy_llrs(mm, 7, 3.0, seed=int(rng.integers(1 << 30)), fixed=fixed)
            cfg = P.DecoderConfig(max_iterations=5, early_termination=False,
                                  arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
            hard, it, conv, post = _gpu(mm, llr, cfg)
            oh, oi, oc, op = O.decode_batch(h, llr, 5, False, want_post=True)
            assert np.array_equal(hard, oh) and np.array_equal(conv, oc), (std, n, rate, fixed)
            assert _post_equal(post, op), (std, n, rate, fixed)
        if mm.z % 8 == 0:
            info = rng.integers(0, 256, size=(300, mm.k // 8), dtype=np.uint8)
            plan = P.make_plan(mm, P.EncoderVariant.Packed)
            dev = P.encode_packed(plan, torch.from_numpy(info).cuda()).cpu().numpy()
            assert np.array_equal(dev, O.encode_packed(mm, info)), (std, n, rate)
        else:                                      # bit-granular encoder: runtime-shift kernel
            bits = rng.integers(0, 2, size=(300, mm.k), dtype=np.uint8)
            got = P.encode_bits(mm, P.pack_bits(bits))
            assert np.array_equal(got, P.pack_bits(P.encode_array(P.make_plan(mm), bits))), (std, n, rate)


def test_known_answers(golden_dir):
    kat = np.load(golden_dir / "kat.npz")
    toy = P.ModelMatrix(P.Standard.Wimax, P.Rate.R12, 1, 3, 2, np.array([[0, 0, 0]]))
    cfg1 = P.DecoderConfig(max_iterations=1, early_termination=False)
    _, _, _, post = _gpu(toy, np.array([[3.0, -1.0, 2.0]], np.float32), cfg1)
    assert np.array_equal(post[0], [2.0, 1.0, 1.0])
    cfg16 = P.DecoderConfig(max_iterations=1, arithmetic=P.Arithmetic.Fixed16, early_termination=False)
    _, _, _, post = _gpu(toy, np.array([[-32768, 5, 7]], np.int16), cfg16)
    assert np.array_equal(post[0], kat["wrap_post"])
    r = P.decode(P.expand(toy), P.LlrBlock(np.zeros(3, np.float32)), P.DecoderConfig(max_iterations=3))
    assert np.array_equal(r.hard_bits, [1, 1, 1]) and r.iterations == 3 and not r.converged


def test_noiseless_converges_in_one_iteration():
    mm = P.get_model_matrix("wifi", 648, "1/2")
    rng = np.random.default_rng(3)
    info = rng.integers(0, 2, (4, mm.k), dtype=np.uint8)
    cw = P.encode_array(P.make_plan(mm), info)
    llr = ((1.0 - 2.0 * cw) * 8.0).astype(np.float32)
    hard, it, conv = _gpu(mm, llr, P.DecoderConfig(), posteriors=False)
    assert conv.all() and (it == 1).all() and np.array_equal(hard, cw)


@pytest.mark.parametrize("fixed", [False, True])
def test_sign_gauge_symmetry(fixed):
    """Flipping LLR signs on a codeword's support XORs the decision with it
    (reference test_decoder.py:149-163, same code / SNR / frame count: the
    symmetry is exact only while int16 never wraps, as in the reference)."""
    mm = P.get_model_matrix("wimax", 576, "1/2")
    llr, _, _ = noisy_llrs(mm, 6, 2.0, seed=4, fixed=fixed)
    cw = P.encode_array(P.make_plan(mm), np.random.default_rng(5).integers(0, 2, mm.k, dtype=np.uint8))
    flip = (llr * (1 - 2 * cw.astype(np.int32))).astype(llr.dtype)
    cfg = P.DecoderConfig(arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
    a = _gpu(mm, llr, cfg, posteriors=False)
    b = _gpu(mm, flip, cfg, posteriors=False)
    assert np.array_equal(a[0] ^ cw, b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    h = P.expand(mm)
    for x, got in ((llr, a), (flip, b)):
        want = O.decode_batch(h, x, 10, True)
        assert all(np.array_equal(u, v) for u, v in zip(got, want))


def test_float32_power_of_two_scale_invariance():
    """Scaling float32 LLRs by a power of two changes no decision or
    iteration count (reference test_decoder.py:166-176: WiMAX 576 R5/6,
    3.5 dB, scales 1/4 and 4), plus a larger batch on the device."""
    mm = P.get_model_matrix("wimax", 576, "5/6")
    cfg = P.DecoderConfig()
    for w in (6, 4096):
        llr, _, _ = noisy_llrs(mm, w, 3.5, seed=6, fixed=False)
        base = _gpu(mm, llr, cfg, posteriors=False)
        for scale in (0.25, 4.0):
            got = _gpu(mm, (llr * np.float32(scale)).astype(np.float32), cfg, posteriors=False)
            assert np.array_equal(base[0], got[0]) and np.array_equal(base[1], got[1])


def test_batch_partition_invariance():
    """Outputs do not depend on how the batch is cut (the worker-invariance
    contract, reference test_decoder.py:228-242): whole batch == slices ==
    a permutation of the batch."""
    mm = P.get_model_matrix("wifi", 1944, "5/6")
    llr, _, _ = noisy_llrs(mm, 301, 4.0, seed=11, fixed=True)
    cfg = P.DecoderConfig(max_iterations=8, arithmetic=P.Arithmetic.Fixed16, early_termination=True)
    full = _gpu(mm, llr, cfg)
    for cut in (1, 7, 150):
        parts = [_gpu(mm, llr[i:i + cut], cfg) for i in range(0, 301, cut)]
        for k in range(4):
            assert np.array_equal(np.concatenate([p[k] for p in parts]), full[k])
    perm = np.random.default_rng(1).permutation(301)
    sh = _gpu(mm, llr[perm], cfg)
    for k in range(4):
        assert np.array_equal(sh[k], full[k][perm])


def test_empty_and_tiny_batches():
    mm = P.get_model_matrix("wimax", 576, "1/2")
    h = P.expand(mm)
    cfg = P.DecoderConfig()
    assert P.decode_block(h, P.LlrBlock(np.empty((0, h.n), np.float32)), cfg) == []
    one = P.decode_block(h, P.LlrBlock(np.zeros((1, h.n), np.float32) + 5.0), cfg)
    assert len(one) == 1 and one[0].converged and one[0].iterations == 1
    out = P.decode_batch(mm, torch.zeros((0, h.n), device="cuda"), cfg)
    assert out[0].shape == (0, h.n)


@pytest.mark.parametrize("fixed", [False, True])
def test_misaligned_device_buffers_take_the_scalar_paths(fixed):
    """LLR / output tensors that are views at an element offset (not 16-byte
    aligned) must give the same results as aligned ones (vectorised prologue /
    epilogue fall back to element accesses)."""
    mm = P.get_model_matrix("wimax", 2304, "1/2")
    llr, _, _ = noisy_llrs(mm, 300, 1.8, seed=77, fixed=fixed)
    cfg = P.DecoderConfig(max_iterations=6, early_termination=False,
                          arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
    dt = torch.int16 if fixed else torch.float32
    aligned = torch.from_numpy(llr).cuda()
    flat = torch.empty(llr.size + 1, dtype=dt, device="cuda")
    flat[1:] = aligned.reshape(-1)
    shifted = flat[1:].view(llr.shape)
    assert shifted.data_ptr() % 16 != 0
    ref = P.decode_batch(mm, aligned, cfg, posteriors=True)
    hard_buf = torch.empty(300 * mm.n + 3, dtype=torch.uint8, device="cuda")
    post_buf = torch.empty(llr.size + 1, dtype=dt, device="cuda")
    out = (hard_buf[3:].view(300, mm.n), torch.empty(300, dtype=torch.int32, device="cuda"),
           torch.empty(300, dtype=torch.uint8, device="cuda"), post_buf[1:].view(llr.shape))
    got = P.decode_batch(mm, shifted, cfg, posteriors=True, out=out)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


@pytest.mark.parametrize("config", ["C2", "C3"])
def test_full_size_batch_properties(config):
    """BASELINE sizes: full batch on the GPU, a seeded sample checked against the
    oracle, and size-independent properties on all of it (packed == packbits of
    unpacked, conv <=> zero syndrome, posterior signs == hard bits)."""
    if config == "C2":
        mm, w, fixed, ebn0, iters = P.get_model_matrix("wimax", 2304, "1/2"), 65536, False, 1.5, 10
    else:
        mm, w, fixed, ebn0, iters = P.get_model_matrix("wifi", 1944, "5/6"), 262144, True, 4.0, 8
    h = P.expand(mm)
    base, _, _ = noisy_llrs(mm, 4096, ebn0, seed=2, fixed=fixed)
    llr = np.concatenate([base] * (w // 4096))
    cfg = P.DecoderConfig(max_iterations=iters, early_termination=False,
                          arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
    t = torch.from_numpy(llr).cuda()
    hard, it, conv, post = P.decode_batch(mm, t, cfg, posteriors=True)
    hp, _, _ = P.decode_batch(mm, t, cfg, hard_packed=True)
    torch.cuda.synchronize()
    hard, it, conv, post, hp = (x.cpu().numpy() for x in (hard, it, conv, post, hp))
    assert np.array_equal(np.packbits(hard, axis=-1), hp)
    assert (it == iters).all()
    assert np.array_equal(hard, (post <= 0).astype(np.uint8))
    # repeated blocks decode identically wherever they sit in the batch
    blocks = hard.reshape(-1, 4096, h.n)
    assert all(np.array_equal(blocks[0], b) for b in blocks[1:])
    sample = np.random.default_rng(0).choice(4096, 512, replace=False)
    oh, oi, oc, op = O.decode_batch(h, base[sample], iters, False, want_post=True)
    assert np.array_equal(hard[sample], oh) and np.array_equal(conv[sample], oc)
    assert _post_equal(post[sample], op)
    par = P.row_parities(h, hard[:2048])
    assert np.array_equal(conv[:2048] == 1, ~par.any(axis=-1))


# --- encoder ------------------------------------------------------------------

def test_packed_encoder_matches_reference_goldens(golden_dir):
    z = np.load(golden_dir / "encode_packed.npz")
    n_checked = 0
    for key in z.files:
        if not key.startswith("cw_"):
            continue
        _, n, rate, wb = key.split("_")
        mm = P.get_model_matrix("wimax", int(n), rate[0] + "/" + rate[1:])
        plan = P.make_plan(mm, P.EncoderVariant.Packed, word_bits=int(wb))
        info = z[f"info_{n}_{rate}"]
        assert np.array_equal(P.encode_packed(plan, info), z[key]), key
        dev = P.encode_packed(plan, torch.from_numpy(info).cuda()).cpu().numpy()
        assert np.array_equal(dev, z[key]), key
        n_checked += 1
    assert n_checked >= 20


def test_packed_encoder_all_octet_codes_vs_oracle_and_array():
    rng = np.random.default_rng(1003)
    codes = [(n, r) for s, n, r in P.supported_codes() if s is P.Standard.Wimax and (n // 24) % 8 == 0]
    assert len(codes) == 60
    for n, rate in codes:
        mm = P.get_model_matrix("wimax", n, rate)
        info = rng.integers(0, 2, size=(300, mm.k), dtype=np.uint8)
        ib = P.pack_bits(info)
        got = P.encode_packed(P.make_plan(mm, P.EncoderVariant.Packed), ib)
        assert np.array_equal(got, O.encode_packed(mm, ib)), (n, rate)
        assert np.array_equal(got, P.pack_bits(P.encode_array(P.make_plan(mm), info))), (n, rate)


@pytest.mark.parametrize("rate", ["1/2", "2/3A", "2/3B", "3/4A", "3/4B", "5/6"])
def test_packed_encoder_native_z96_tiles_tail_and_misaligned(rate):
    """Native Z=96 codes take the bulk-copy pipeline for whole 128-codeword
    tiles and the staged kernel for the ragged tail / misaligned buffers."""
    mm = P.get_model_matrix("wimax", 2304, rate)
    plan = P.make_plan(mm, P.EncoderVariant.Packed)
    rng = np.random.default_rng(hash(rate) % 1000)
    info = rng.integers(0, 256, size=(128 * 700 + 77, mm.k // 8), dtype=np.uint8)
    ref = O.encode_packed(mm, info)
    dev = torch.from_numpy(info).cuda()
    assert np.array_equal(P.encode_packed(plan, dev).cpu().numpy(), ref)
    sub = dev[1:257]                                    # 8-byte-misaligned view
    assert np.array_equal(P.encode_packed(plan, sub).cpu().numpy(), ref[1:257])
    assert np.array_equal(P.encode_packed(plan, dev[:128 * 3]).cpu().numpy(), ref[:128 * 3])


def test_encode_then_decode_round_trip_c5_scale():
    """2^20 seeded info words (BASELINE config 5 code) -> GPU encode -> noiseless
    LLRs -> GPU decode converges in one iteration and returns the info bits."""
    mm = P.get_model_matrix("wimax", 2304, "3/4A")
    plan = P.make_plan(mm, P.EncoderVariant.Packed)
    w = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(5)
    info = torch.randint(0, 256, (w, mm.k // 8), dtype=torch.uint8, device="cuda", generator=g)
    cw = P.encode_packed(plan, info)
    assert torch.equal(cw[:, :mm.k // 8], info)
    sample = torch.randint(0, w, (2048,), device="cuda", generator=g)
    ref = O.encode_packed(mm, info[sample].cpu().numpy())
    assert np.array_equal(cw[sample].cpu().numpy(), ref)
    bits = torch.from_numpy(np.unpackbits(cw[:65536].cpu().numpy(), axis=-1)).cuda()
    llr = ((1 - 2 * bits.to(torch.int16)) * 300).to(torch.int16)
    cfg = P.DecoderConfig(arithmetic=P.Arithmetic.Fixed16)
    hard, it, conv = P.decode_batch(mm, llr, cfg, hard_packed=True)
    assert bool(conv.all()) and bool((it == 1).all())
    assert torch.equal(hard, cw[:65536])


def test_bit_granular_encoder_all_codes_any_z():
    """np.packbits-layout encoding for every code, Z % 8 != 0
    included (Wi-Fi Z = 27/54/81, scaled WiMAX Z = 28, 36, ...), equal to
    pack_bits(encode_array) -- the reference's array encoder, encoder.py:133-163."""
    rng = np.random.default_rng(2024)
    n_unaligned = 0
    for std, n, rate in P.supported_codes():
        mm = P.get_model_matrix(std, n, rate)
        n_unaligned += mm.z % 8 != 0
        for w in (1, 129):
            info = rng.integers(0, 2, size=(w, mm.k), dtype=np.uint8)
            want = P.pack_bits(P.encode_array(P.make_plan(mm), info))
            got = P.encode_bits(mm, P.pack_bits(info))
            assert np.array_equal(got, want), (std, n, rate, w)
    assert n_unaligned == 12 + 54


def test_bit_granular_encoder_codewords_satisfy_h():
    """Independent of encode_array: every encoded word is in the null space
    of the expanded H (codebook.expand), for unaligned Z (structure kernels)
    and a non-standard table (generic kernel), from a misaligned view."""
    rng = np.random.default_rng(99)
    base = P.get_model_matrix("wifi", 648, "1/2")
    ent = base.entries.copy()
    ent[0, 0] = -1                                     # not a standard zero pattern: generic kernel
    generic = P.ModelMatrix(base.standard, base.rate, base.z, base.nb, base.kb, ent)
    mms = [P.get_model_matrix("wifi", 648, "5/6"), P.get_model_matrix("wifi", 1944, "1/2"),
           P.get_model_matrix("wimax", 672, "3/4A"), generic]
    for mm in mms:
        info = rng.integers(0, 2, size=(300, mm.k), dtype=np.uint8)
        dev = torch.from_numpy(P.pack_bits(info)).cuda()
        cw = P.unpack_bits(P.encode_bits(mm, dev[1:]).cpu().numpy(), mm.n)   # misaligned view
        assert np.array_equal(cw[:, :mm.k], info[1:])
        h = P.codebook.expand(mm)
        rows = np.repeat(np.arange(h.m), np.diff(h.row_ptr))
        syn = np.zeros((cw.shape[0], h.m), np.uint8)
        np.bitwise_xor.at(syn.T, rows, cw[:, h.row_cols].T)
        assert not syn.any(), (mm.n, mm.z)


@pytest.mark.parametrize("std,n,rate", [("wifi", 648, "1/2"), ("wifi", 1296, "2/3"), ("wifi", 1944, "5/6"),
                                        ("wimax", 576, "2/3A"), ("wimax", 1344, "3/4B"), ("wimax", 2208, "5/6")])
def test_bit_granular_encoder_pipeline_many_tiles(std, n, rate):
    """Native Wi-Fi codes and scaled WiMAX codes (compile-time scaled shifts)
    stream whole 128-codeword tiles through the bulk-copy pipeline (several
    tiles per CTA: both buffer parities), the ragged tail through the staged
    kernel."""
    mm = P.get_model_matrix(std, n, rate)
    rng = np.random.default_rng(n)
    bits = rng.integers(0, 2, size=(128 * 1200 + 77, mm.k), dtype=np.uint8)
    want = P.pack_bits(P.encode_array(P.make_plan(mm), bits))
    got = P.encode_bits(mm, torch.from_numpy(P.pack_bits(bits)).cuda()).cpu().numpy()
    assert np.array_equal(got, want)


def test_tmem_message_kernel_matches_oracle():
    """The TMEM-resident-message float32 kernel (csrc/decode_tmem.cuh), forced with
    QCB_TMEM=1 in a fresh process (the choice is read once per process), on the
    degree-20 codes and a low-degree one, fixed iterations and early termination."""
    import subprocess
    import sys
    script = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2306_12063_b200 as P
from oracle import oracle as O
from tests._util import noisy_llrs
for i, code in enumerate([("wifi", 1944, "5/6"), ("wimax", 2304, "5/6"), ("wimax", 1152, "5/6"), ("wimax", 2304, "1/2")]):
    mm = P.get_model_matrix(*code)
    llr, _, _ = noisy_llrs(mm, 37, 2.5 + mm.rate.fraction, seed=500 + i)
    for early in (False, True):
        cfg = P.DecoderConfig(max_iterations=6, early_termination=early)
        hard, it, conv, post = [t.cpu().numpy() for t in P.decode_batch(mm, torch.from_numpy(llr).cuda(), cfg, posteriors=True)]
        oh, oi, oc, op = O.decode_batch(P.expand(mm), llr, 6, early, workers=4, want_post=True)
        assert np.array_equal(hard, oh) and np.array_equal(it, oi) and np.array_equal(conv, oc), code
        assert np.array_equal(post, op, equal_nan=True), code
print("ok")
'''
    import os
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, QCB_TMEM="1")
    res = subprocess.run([sys.executable, "-c", script], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stdout + res.stderr


SCALED_Z = list(range(24, 93, 4))


@pytest.mark.parametrize("fixed", [False, True])
def test_scaled_codes_compile_time_kernels_at_plan_size_match_oracle(fixed):
    """The 108 scaled WiMAX codes run decoders compiled for their own Z
    (csrc/decode_scaled.cuh) with the measured codewords-per-CTA plan
    (csrc/scaled_plan_gen.h; int16 Wi-Fi 1944 R1/2 and R2/3 too, native_fill_cw),
    which only engages for batches of several waves:
    10,000 codewords per code here, device channel frames, every code, fixed
    iterations (and early termination on a Z subset), checked against the C
    oracle on sampled rows: the first and last CTAs' codewords (including a
    ragged final CTA) and random rows in between."""
    from paper_2306_12063_b200 import channel as CH
    from tests._util import sigma2
    dev = torch.device("cuda", 0)
    arith = P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32
    rng = np.random.default_rng(77 + fixed)
    w = 10_001
    codes = [(s.value, n, r.value) for s, n, r in P.supported_codes() if s.value == "wimax" and n != 2304]
    assert len(codes) == 108
    if fixed:       # native int16 codes with a multi-pair plan (native_fill_cw)
        codes += [("wifi", 1944, "1/2"), ("wifi", 1944, "2/3"), ("wifi", 1944, "3/4"), ("wifi", 1944, "5/6")]
    for ci, (std, n, rate) in enumerate(codes):
        mm = P.get_model_matrix(std, n, rate)
        h = P.expand(mm)
        info = CH.frames_info_device(31, ci, 0, w, mm.k, dev)
        llr = CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(1.5 + 2 * mm.rate.fraction,
                                                                             mm.rate.fraction), arith, seed=31, point=ci)
        rows = np.unique(np.concatenate([np.arange(40), np.arange(w - 40, w), rng.integers(0, w, 40)]))
        llr_rows = llr[torch.from_numpy(rows).to(dev)].cpu().numpy()
        for early in ((False, True) if mm.z in (24, 36, 48, 72, 84) else (False,)):
            cfg = P.DecoderConfig(max_iterations=5, arithmetic=arith, early_termination=early)
            hard, it, conv, post = P.decode_batch(mm, llr, cfg, posteriors=True)
            torch.cuda.synchronize()
            oh, oi, oc, op = O.decode_batch(h, llr_rows, 5, early, workers=4, want_post=True)
            sel = torch.from_numpy(rows).to(dev)
            assert np.array_equal(hard[sel].cpu().numpy(), oh), (n, rate, early)
            assert np.array_equal(it[sel].cpu().numpy(), oi) and np.array_equal(conv[sel].cpu().numpy(), oc), (n, rate)
            assert _post_equal(post[sel].cpu().numpy(), op), (n, rate, early)
        del llr, info


@pytest.mark.parametrize("rate", ["1/2", "2/3", "3/4", "5/6"])
def test_one_warp_cta_codes_small_and_multi_wave_batches_match_oracle(rate):
    """Wi-Fi 648 float32 (Z = 27, one-warp CTAs with __syncwarp tier barriers and
    shadow lanes; BASELINE C1's code): a small batch and one of several waves against
    the C oracle: fixed iterations and early termination, noisy frames plus hostile
    values (+-0.0, +-inf, NaN, huge, denormal), packed hard bits and posteriors."""
    mm = P.get_model_matrix("wifi", 648, rate)
    h = P.expand(mm)
    for w, seed in ((37, 900), (3001, 901)):
        llr, _, _ = noisy_llrs(mm, w, 1.0 + 2.0 * mm.rate.fraction, seed=seed + int(mm.rate.fraction * 100))
        rng = np.random.default_rng(seed)
        bad = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 3e38, -3e38, 1e-45], np.float32)
        for row in range(0, min(w, 12)):                      # rows 0..11: sprinkled to all-hostile
            k = (row + 1) * mm.n // 12
            idx = rng.choice(mm.n, size=k, replace=False)
            llr[row, idx] = bad[rng.integers(0, len(bad), size=k)]
        for early in (False, True):
            cfg = P.DecoderConfig(max_iterations=7, early_termination=early)
            hard, it, conv, post = _gpu(mm, llr, cfg)
            oh, oi, oc, op = O.decode_batch(h, llr, 7, early, workers=4, want_post=True)
            assert np.array_equal(hard, oh), (rate, w, early)
            assert np.array_equal(it, oi) and np.array_equal(conv, oc), (rate, w, early)
            assert _post_equal(post, op), (rate, w, early)
            hp, _, _ = _gpu(mm, llr, cfg, posteriors=False, hard_packed=True)
            assert np.array_equal(hp, np.packbits(oh, axis=-1)), (rate, w, early)
