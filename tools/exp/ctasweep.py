"""Sweep codewords-per-CTA (QCB_CW_PER_CTA) for a few codes: subprocess per setting."""
import json, os, subprocess, sys
codes = [("wifi", 648, "1/2"), ("wifi", 1296, "1/2"), ("wifi", 1944, "1/2"), ("wifi", 1944, "5/6"), ("wimax", 2304, "1/2"), ("wimax", 2304, "3/4A")]
prog = r'''
import sys, json, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200.workloads import device_llrs
std, n, rate, fixed = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4] == "1"
mm = P.get_model_matrix(std, n, rate)
w = 65536 if fixed else 16384
llr, _ = device_llrs(mm, w, 3.0, 7, fixed, torch.device('cuda', 0))
cfg = P.DecoderConfig(max_iterations=10, early_termination=False, arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
out = P.decode_batch(mm, llr, cfg); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): P.decode_batch(mm, llr, cfg, out=out)
b.record(); torch.cuda.synchronize()
print(round(w * mm.n / (a.elapsed_time(b) / 5 * 1e-3) / 1e9, 1))
'''
for fixed in ("0", "1"):
    for code in codes:
        row = []
        for p in ["auto", 1, 2, 3, 4, 5, 7]:
            env = dict(os.environ)
            if p != "auto":
                env["QCB_CW_PER_CTA"] = str(p)
            r = subprocess.run([sys.executable, "-c", prog, code[0], str(code[1]), code[2], fixed], env=env,
                               capture_output=True, text=True)
            row.append((p, r.stdout.strip() or r.stderr.strip()[-80:]))
        print("i16" if fixed == "1" else "f32", code, row, flush=True)
