"""Decode throughput of scaled WiMAX codes (runtime-Z kernels) vs the native Z=96 ones."""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200.workloads import device_llrs
dev = torch.device('cuda', 0)
for fixed in (False, True):
    for n in (576, 960, 1152, 1536, 1920, 2304):
        for rate in ("1/2", "3/4A"):
            mm = P.get_model_matrix("wimax", n, rate)
            w = (1 << 22) * 2304 // n // (4 if not fixed else 1) // 8
            llr, _ = device_llrs(mm, w, 3.0, 11, fixed, dev)
            cfg = P.DecoderConfig(max_iterations=10, early_termination=False,
                                  arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
            out = P.decode_batch(mm, llr, cfg)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3): P.decode_batch(mm, llr, cfg, out=out)
            b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 3
            print("i16" if fixed else "f32", n, rate, "z", mm.z, "W", w, round(w * mm.n / (ms * 1e-3) / 1e9, 1), "Gb/s", flush=True)
            del llr, out
