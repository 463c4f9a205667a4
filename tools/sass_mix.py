"""Opcode mix of one kernel from an ncu source-page CSV (--page source --csv --print-source sass).

    python tools/sass_mix.py gpurun_out/c5_sass.csv <work units per launch>

Prints executed thread-instructions per work unit by opcode, with the share of
warp-stall samples on those instructions.
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
hdr = rows[1]
data = rows[2:]
ii = hdr.index("Thread Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = tots = 0
ops, samp = collections.Counter(), collections.Counter()
for r in data:
    n, s = int(r[ii] or 0), int(r[si] or 0)
    toks = r[1].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    key = op if op.startswith(("VIMNMX", "VIADD", "LDS", "STS", "LOP3", "BAR")) else op.split(".")[0]
    ops[key] += n
    samp[key] += s
    tot += n
    tots += s
print(f"thread instructions per unit: {tot / units:.2f}")
for k, v in ops.most_common(40):
    print(f"{k:22s} {v / units:7.3f}   stall samples {100 * samp[k] / max(tots, 1):5.1f}%")
