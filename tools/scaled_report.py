"""profiles/r02_scaled_decode.txt from a tools/codebench.py --codes all --json run.

    python tools/scaled_report.py gpurun_out/codebench_all.json profiles/r02_scaled_decode.txt

Every scaled WiMAX code (N = 24 Z, Z = 24..92) next to the native Z = 96 code of its rate;
the 'runtime-Z' column (the same codes on the round-1 runtime-Z kernels, QCB_SCALED=0) is
carried over from the existing report when there is one.
"""
import json, sys
from pathlib import Path

src, dst = Path(sys.argv[1]), Path(sys.argv[2])
rows = json.load(open(src))
old_rt = {}
if dst.exists():
    for l in dst.read_text().splitlines():
        t = l.split()
        if len(t) == 7 and not l.startswith("#"):
            old_rt[(t[0], t[1])] = t[6]
native = {(r["code"].split("-r")[1], r["arith"]): r["gbit_s"] for r in rows if r["code"].startswith("wimax-2304-")}
out, ratios = [], []
for r in rows:
    if not r["code"].startswith("wimax-") or r["code"].startswith("wimax-2304-"):
        continue
    nat = native[(r["code"].split("-r")[1], r["arith"])]
    ratio = r["gbit_s"] / nat
    ratios.append(ratio)
    out.append(f"{r['code']:<16} {r['arith']:>4} {r['z']:>3}  {r['gbit_s']:>6.1f}  {nat:>6.1f}   {ratio:.2f}  {old_rt.get((r['code'], r['arith']), '-'):>6}")
ratios.sort()
hdr = f"""# round 2 (final): per-code decode throughput on one B200 (tools/codebench.py --codes all --w {rows[0]['w']}, 10
# fixed iterations, 3 dB device frames; written by tools/scaled_report.py).  Scaled WiMAX codes run decoders
# compiled for their own Z (csrc/decode_scaled.cuh) with the measured codewords-per-CTA plan
# (csrc/scaled_plan_gen.h) and the chunked, bank-conflict-free row mapping where G | 32 and 32 / G | Z;
# 'runtime-Z' = the same codes on the runtime-Z kernels (QCB_SCALED=0, the round-1 path, measured earlier in round 2).
# code arith Z  Gbit/s  native(Z=96)  ratio  runtime-Z"""
n_ok = sum(1 for x in ratios if x >= 0.8)
tail = f"# {n_ok} of {len(ratios)} scaled (code, arith) within 20 % of their native structure; median ratio {ratios[len(ratios) // 2]:.2f}, min {ratios[0]:.2f}"
dst.write_text(hdr + "\n" + "\n".join(out) + "\n" + tail + "\n")
print(tail)
