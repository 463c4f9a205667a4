"""One decode for profiling: code, arithmetic, Eb/N0, early termination (0/1) from argv."""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import channel as CH
from paper_2306_12063_b200.workloads import sigma2
std, n, rate, ar, snr, et = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], float(sys.argv[5]), int(sys.argv[6])
dev = torch.device('cuda', 0); torch.cuda.set_device(0)
mm = P.get_model_matrix(std, n, rate)
arith = P.Arithmetic.Fixed16 if ar == "i16" else P.Arithmetic.Float32
W = 65536
info = CH.frames_info_device(9, 3, 0, W, mm.k, dev)
llr = CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(snr, mm.rate.fraction), arith, seed=9, point=3)
cfg = P.DecoderConfig(max_iterations=10, early_termination=bool(et), arithmetic=arith)
out = P.decode_batch(mm, llr, cfg)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): P.decode_batch(mm, llr, cfg, out=out)
b.record(); torch.cuda.synchronize()
print(f"{std}-{n}-{rate} {ar} {snr} dB et={et}: {a.elapsed_time(b) / 5:.3f} ms, avg iterations {out[1].float().mean().item():.2f}")
