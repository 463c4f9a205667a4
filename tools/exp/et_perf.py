"""Early-termination throughput: C2-size batches at several SNRs (W=65536, max 10 iterations)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200.workloads import device_llrs
dev = torch.device('cuda', 0)
for code, fixed in ((("wimax", 2304, "1/2"), False), (("wimax", 2304, "3/4A"), True)):
    mm = P.get_model_matrix(*code)
    for snr in (1.5, 2.5, 3.5):
        llr, _ = device_llrs(mm, 65536, snr, 9, fixed, dev)
        for et in (False, True):
            cfg = P.DecoderConfig(max_iterations=10, early_termination=et,
                                  arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
            out = P.decode_batch(mm, llr, cfg)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5): P.decode_batch(mm, llr, cfg, out=out)
            b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            print(code, "i16" if fixed else "f32", snr, "ET" if et else "fixed", round(65536 * mm.n / (ms * 1e-3) / 1e9, 1),
                  "Gb/s  avg iters", round(out[1].float().mean().item(), 2), flush=True)
