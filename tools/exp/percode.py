"""Per-code decode throughput on the GPU (BASELINE config 4's 18 codes, f32 and i16)."""
import json, sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200.workloads import ALL_18, device_llrs
dev = torch.device('cuda', 0)
res = []
for fixed in (False, True):
    for ci, code in enumerate(ALL_18):
        mm = P.get_model_matrix(*code)
        w = 16384 if not fixed else 65536
        llr, _ = device_llrs(mm, w, 3.0, 4000 + ci, fixed, dev)
        cfg = P.DecoderConfig(max_iterations=10, early_termination=False,
                              arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
        out = P.decode_batch(mm, llr, cfg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            P.decode_batch(mm, llr, cfg, out=out)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        gbs = w * mm.n / (ms * 1e-3) / 1e9
        frac = mm.edges * 10 * w * 12 / (ms * 1e-3) / 37.225e12
        res.append((code, "i16" if fixed else "f32", round(gbs, 1), round(frac, 3), mm.z, int((mm.entries >= 0).sum(1).max())))
        print(res[-1], flush=True)
