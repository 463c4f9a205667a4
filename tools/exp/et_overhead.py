"""Per-iteration cost of the early-termination machinery: frames at -3 dB (nothing converges, so
ET runs all max_iters sweeps plus one syndrome per sweep) against fixed iterations."""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import channel as CH
from paper_2306_12063_b200.workloads import sigma2
dev = torch.device('cuda', 0)
torch.cuda.set_device(0)
W = 65536
for ci, code in enumerate((("wifi", 648, "1/2"), ("wifi", 1296, "1/2"), ("wifi", 1944, "5/6"), ("wimax", 2304, "1/2"), ("wimax", 2304, "3/4A"))):
    mm = P.get_model_matrix(*code)
    for fixed in (False, True):
        arith = P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32
        info = CH.frames_info_device(9, ci, 0, W, mm.k, dev)
        llr = CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(-3.0, mm.rate.fraction), arith, seed=9, point=ci)
        res = []
        for et in (False, True):
            cfg = P.DecoderConfig(max_iterations=10, early_termination=et, arithmetic=arith)
            out = P.decode_batch(mm, llr, cfg)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5): P.decode_batch(mm, llr, cfg, out=out)
            b.record(); torch.cuda.synchronize()
            res.append((a.elapsed_time(b) / 5, out[1].float().mean().item()))
        print(f"{code[0]}-{code[1]}-r{code[2].replace('/', '')} {'i16' if fixed else 'f32'}: fixed {res[0][0]:.3f} ms, ET {res[1][0]:.3f} ms (avg iterations {res[1][1]:.2f}): +{(res[1][0] / res[0][0] - 1) * 100:.1f} %", flush=True)
