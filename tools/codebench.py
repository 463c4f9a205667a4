"""Per-code decode throughput (coded Gbit/s) on one GPU, any of the 126 codes.

    python tools/codebench.py [--codes all|native|scaled|wimax-576-r12,...]
                              [--arith f32,i16] [--w 65536] [--iters 10] [--json out.json]

Inputs: seeded device channel frames (Philox info bits -> encode_array ->
BPSK/AWGN at 3 dB -> LLRs), fixed iterations (early termination off), one
warm-up call then the median of 5 event-timed calls on the launching stream.
Next to each scaled WiMAX code the native Z = 96 code of the same rate is
reported, so "within 20 % of native" can be read off directly.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import paper_2306_12063_b200 as P
    from paper_2306_12063_b200 import channel as CH
    from paper_2306_12063_b200.workloads import sigma2

    ap = argparse.ArgumentParser()
    ap.add_argument("--codes", default="all")
    ap.add_argument("--arith", default="f32,i16")
    ap.add_argument("--w", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    allc = [(s.value, n, r.value) for s, n, r in list(P.supported_codes())]
    if args.codes == "all":
        codes = allc
    elif args.codes in ("native", "scaled"):
        native = {(s, n, r) for s, n, r in allc if (s == "wimax" and n == 2304) or s == "wifi"}
        codes = [c for c in allc if (c in native) == (args.codes == "native")]
    else:
        codes = []
        for tok in args.codes.split(","):
            s, n, r = tok.split("-")
            codes.append((s, int(n), r[1:].replace("23", "2/3").replace("34", "3/4").replace("12", "1/2")
                          .replace("56", "5/6")))
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    out = []
    for ar in args.arith.split(","):
        fixed = ar == "i16"
        arith = P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32
        cfg = P.DecoderConfig(max_iterations=args.iters, early_termination=False, arithmetic=arith)
        for ci, code in enumerate(codes):
            mm = P.get_model_matrix(*code)
            w = args.w
            info = CH.frames_info_device(7, ci, 0, w, mm.k, dev)
            llr = CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(3.0, mm.rate.fraction), arith,
                                        seed=7, point=ci)
            del info
            res = P.decode_batch(mm, llr, cfg)
            torch.cuda.synchronize()
            times = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                P.decode_batch(mm, llr, cfg, out=res)
                b.record()
                b.synchronize()
                times.append(a.elapsed_time(b))
            ms = statistics.median(times)
            gbs = w * mm.n / (ms * 1e-3) / 1e9
            rec = {"code": f"{code[0]}-{code[1]}-r{code[2].replace('/', '')}", "arith": ar, "z": mm.z,
                   "gbit_s": round(gbs, 2), "ms": round(ms, 3), "w": w,
                   "edge_upd_per_s": round(w * mm.edges * args.iters / (ms * 1e-3) / 1e12, 4)}
            out.append(rec)
            print(json.dumps(rec), flush=True)
            del llr, res
    if args.json:
        Path(args.json).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
