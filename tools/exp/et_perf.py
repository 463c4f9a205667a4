"""Early-termination throughput (the reference's default mode): 65536 codewords, max 10
iterations, device channel frames at several Eb/N0, both arithmetics, against fixed iterations."""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import channel as CH
from paper_2306_12063_b200.workloads import sigma2
dev = torch.device('cuda', 0)
torch.cuda.set_device(0)
W = 65536
for ci, code in enumerate((("wimax", 2304, "1/2"), ("wimax", 2304, "3/4A"), ("wifi", 1944, "5/6"), ("wifi", 648, "1/2"))):
    mm = P.get_model_matrix(*code)
    base = {"1/2": 1.5, "3/4A": 2.5, "5/6": 3.5}[code[2]]
    for fixed in (False, True):
        arith = P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32
        for snr in (base, base + 1.0, base + 2.0):
            info = CH.frames_info_device(9, ci, 0, W, mm.k, dev)
            llr = CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(snr, mm.rate.fraction), arith, seed=9, point=ci)
            res = []
            for et in (False, True):
                cfg = P.DecoderConfig(max_iterations=10, early_termination=et, arithmetic=arith)
                out = P.decode_batch(mm, llr, cfg)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(5): P.decode_batch(mm, llr, cfg, out=out)
                b.record(); torch.cuda.synchronize()
                ms = a.elapsed_time(b) / 5
                res.append((round(W * mm.n / (ms * 1e-3) / 1e9, 1), round(out[1].float().mean().item(), 2)))
            print(f"{code[0]}-{code[1]}-r{code[2].replace('/', '')} {'i16' if fixed else 'f32'} {snr:.1f} dB: fixed {res[0][0]} Gb/s, ET {res[1][0]} Gb/s (avg iterations {res[1][1]})", flush=True)
