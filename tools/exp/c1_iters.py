"""C1 kernel time against the iteration count (Wi-Fi 648 R1/2 float32, W codewords):
slope = time per sweep (12 tiers), intercept = launch + prologue + syndrome + epilogue.
40 back-to-back launches on distinct batches inside one CUDA graph, events inside the graph."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import paper_2306_12063_b200 as P
from paper_2306_12063_b200 import channel as CH
from paper_2306_12063_b200.workloads import sigma2

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
mm = P.get_model_matrix("wifi", 648, "1/2")
K = 40
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.Stream(dev)
llrs = []
for s in range(K):
    info = CH.frames_info_device(7, 0, s * w, w, mm.k, dev)
    llrs.append(CH.channel_llr_device(CH.encode_array_device(mm, info), sigma2(2.0, mm.rate.fraction), P.Arithmetic.Float32, seed=7, point=0, frame0=s * w))
for iters in (0, 1, 2, 5, 10, 20, 40):
    cfg = P.DecoderConfig(max_iterations=max(iters, 1), early_termination=False, arithmetic=P.Arithmetic.Float32) if iters else None
    if cfg is None:
        continue
    outs = [P.decode_batch(mm, l, cfg) for l in llrs]
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
    with torch.cuda.graph(g, stream=stream):
        ev[0].record(stream)
        for l, o in zip(llrs, outs):
            P.decode_batch(mm, l, cfg, out=o, stream=stream)
        ev[1].record(stream)
    torch.cuda.synchronize()
    ts = []
    with torch.cuda.stream(stream):
        for _ in range(5):
            flush.zero_()
            g.replay()
            stream.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]) * 1e3 / K)
    print(json.dumps({"w": w, "iters": iters, "us_per_launch": round(min(ts), 3), "all": [round(t, 2) for t in ts]}), flush=True)
