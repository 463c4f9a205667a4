"""C1 kernel time against batch size (Wi-Fi 648 R1/2 float32, 10 fixed iterations):
is the 1024-codeword step bound by the per-warp dependency chain (time flat in W
up to one warp per sub-partition and beyond) or by issue slots (time ~ warps per
sub-partition)?  Events recorded inside a CUDA graph around one decode, L2 flushed."""
import statistics, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import channel as CH
from paper_2306_12063_b200.workloads import sigma2

code = sys.argv[1] if len(sys.argv) > 1 else "wifi-648-r12"
s, n, r = code.split("-")
rate = r[1:].replace("23", "2/3").replace("34", "3/4").replace("12", "1/2").replace("56", "5/6")
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
mm = P.get_model_matrix(s, int(n), rate)
cfg = P.DecoderConfig(max_iterations=10, early_termination=False, arithmetic=P.Arithmetic.Float32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.Stream(dev)
for w in (148, 296, 592, 888, 1024, 1184, 1776, 2048, 2368, 4096, 8192):
    info = CH.frames_info_device(7, 0, 0, w, mm.k, dev)
    llr = CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(2.0, mm.rate.fraction), P.Arithmetic.Float32, seed=7, point=0)
    res = P.decode_batch(mm, llr, cfg)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(3):
            P.decode_batch(mm, llr, cfg, out=res, stream=stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
    with torch.cuda.graph(g, stream=stream):
        ev[0].record(stream)
        P.decode_batch(mm, llr, cfg, out=res, stream=stream)
        ev[1].record(stream)
    torch.cuda.synchronize()
    ts = []
    with torch.cuda.stream(stream):
        for _ in range(30):
            flush.zero_()
            g.replay()
            stream.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
    us = statistics.median(ts) * 1e3
    print(json.dumps({"code": code, "w": w, "us": round(us, 2), "gbit_s": round(w * mm.n / us / 1e3, 2)}), flush=True)
