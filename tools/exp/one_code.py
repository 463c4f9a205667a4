"""Decode one code repeatedly (profiling target): python tools/exp/one_code.py wifi 648 1/2 f32 65536"""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200.workloads import device_llrs
std, n, rate, ar, w = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
fixed = ar == "i16"
mm = P.get_model_matrix(std, n, rate)
llr, _ = device_llrs(mm, w, 3.0, 11, fixed, torch.device('cuda', 0))
cfg = P.DecoderConfig(max_iterations=10, early_termination=False, arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
out = P.decode_batch(mm, llr, cfg)
for _ in range(3):
    P.decode_batch(mm, llr, cfg, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); P.decode_batch(mm, llr, cfg, out=out); b.record(); torch.cuda.synchronize()
print(std, n, rate, ar, w, round(w * mm.n / (a.elapsed_time(b) * 1e-3) / 1e9, 1), "Gb/s")
