"""Generate tests/golden/ fixtures for the device channel, the waterfall
loop and the LLR0 / decode-record formats by running the REFERENCE.

Runs only in the build container (imports /root/reference/pkg/src/qcldpc);
the GPU box only reads the committed fixtures.

channel_<case>.npz  frames [start, start+count) of (seed, point): info bits
                   and float64 noise from the reference's _gen_batch, the
                   encode_array codewords, and _llr_batch's float32 and
                   Fixed16 (q_b = 10) LLRs.
waterfall_<case>.csv  reference run_waterfall(...).to_csv() (arguments in
                   WATERFALL below).
llr0_<case>.llr / records_<case>.bin  a reference write_llr_file container
                   and the bytes the reference CLI `decode` writes for it
                   (cli.py:169-183: decode_block, packbits, iters, conv).

Usage:  python tools/make_golden_channel.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from qcldpc import chansim, codebook, decoder, encoder  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"

CHANNEL = [  # name, standard, n, rate, ebn0, seed, point, start, count
    ("wimax576_r12", "wimax", 576, "1/2", 2.0, 21, 1, 300, 40),
    ("wifi648_r23", "wifi", 648, "2/3", 3.0, 22, 0, 0, 24),
    ("wimax2304_r34a", "wimax", 2304, "3/4A", 2.5, 23, 2, 7, 16),
]

WATERFALL = [  # name, standard, n, rate, arithmetic, max_iters, snrs, min_errors, max_frames, seed, min_frames
    ("wimax576_r12_f32", "wimax", 576, "1/2", "float32", 8, [1.5, 2.5], 300, 4096, 11, 512),
    ("wimax576_r12_i16", "wimax", 576, "1/2", "fixed16", 8, [1.5, 2.5], 300, 4096, 11, 512),
    ("wifi648_r12_f32", "wifi", 648, "1/2", "float32", 10, [2.0], 200, 2048, 12, 1),
    ("wimax1152_r56_i16", "wimax", 1152, "5/6", "fixed16", 10, [3.5, 4.0], 100, 3072, 13, 256),
]

RECORDS = [  # name, standard, n, rate, arithmetic, count, ebn0, seed, max_iters, early
    ("wimax576_r12_f32", "wimax", 576, "1/2", "float32", 33, 1.8, 31, 10, True),
    ("wimax576_r12_i16", "wimax", 576, "1/2", "fixed16", 33, 1.8, 32, 6, False),
]


def _mm(std, n, rate):
    return codebook.get_model_matrix(std, n, rate)


def channel():
    for name, std, n, rate, ebn0, seed, point, start, count in CHANNEL:
        mm = _mm(std, n, rate)
        info, noise = chansim._gen_batch(mm, seed, point, start, count)
        cw = encoder.encode_array(encoder.make_plan(mm), info)
        sigma2 = chansim.ebn0_to_sigma2(ebn0, mm.rate.fraction)
        f32 = chansim._llr_batch(cw, noise, sigma2, decoder.DecoderConfig())
        i16 = chansim._llr_batch(cw, noise, sigma2, decoder.DecoderConfig(arithmetic=decoder.Arithmetic.Fixed16))
        np.savez_compressed(OUT / f"channel_{name}.npz", std=std, n=n, rate=rate, ebn0=ebn0, seed=seed,
                            point=point, start=start, sigma2=sigma2, info=info, noise=noise, cw=cw,
                            llr_f32=f32.values, llr_i16=i16.values)
        print("channel", name, info.shape)


def waterfall():
    meta = {}
    for name, std, n, rate, arith, iters, snrs, min_err, max_frames, seed, min_frames in WATERFALL:
        mm = _mm(std, n, rate)
        cfg = decoder.DecoderConfig(max_iterations=iters, arithmetic=decoder.Arithmetic(arith))
        table = chansim.run_waterfall(mm, cfg, snrs, min_errors=min_err, max_frames=max_frames, seed=seed,
                                      min_frames=min_frames)
        (OUT / f"waterfall_{name}.csv").write_text(table.to_csv())
        meta[name] = dict(std=std, n=n, rate=rate, arithmetic=arith, max_iterations=iters, snrs=snrs,
                          min_errors=min_err, max_frames=max_frames, seed=seed, min_frames=min_frames)
        print("waterfall", name)
        print(table.to_csv())
    (OUT / "waterfall_cases.json").write_text(json.dumps(meta, indent=1) + "\n")


def records():
    meta = {}
    for name, std, n, rate, arith, count, ebn0, seed, iters, early in RECORDS:
        mm = _mm(std, n, rate)
        h = codebook.expand(mm)
        info, noise = chansim._gen_batch(mm, seed, 0, 0, count)
        cw = encoder.encode_array(encoder.make_plan(mm), info)
        sigma2 = chansim.ebn0_to_sigma2(ebn0, mm.rate.fraction)
        a = decoder.Arithmetic(arith)
        block = chansim._llr_batch(cw, noise, sigma2, decoder.DecoderConfig(arithmetic=a))
        path = OUT / f"llr0_{name}.llr"
        decoder.write_llr_file(path, block)
        back = decoder.read_llr_file(path)
        cfg = decoder.DecoderConfig(max_iterations=iters, arithmetic=back.arithmetic, early_termination=early)
        results = decoder.decode_block(h, back, cfg)
        with open(OUT / f"records_{name}.bin", "wb") as f:           # cli.py:180-183
            for r in results:
                f.write(encoder.pack_bits(r.hard_bits).tobytes())
                f.write(bytes([min(r.iterations, 255), 1 if r.converged else 0]))
        meta[name] = dict(std=std, n=n, rate=rate, max_iterations=iters, early_termination=early)
        print("records", name)
    (OUT / "records_cases.json").write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    channel()
    records()
    waterfall()
