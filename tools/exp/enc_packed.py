"""Throughput of the packed encoders (qc_encode_bits = qc_encode_packed for Z % 8 == 0) on WiMAX codes at several Z."""
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
w = 1 << 22
for n in (576, 672, 1152, 1248, 1920, 2208, 2304):
    for rate in ("1/2", "5/6"):
        mm = P.get_model_matrix("wimax", n, rate)
        info = torch.randint(0, 256, (w, (mm.k + 7) // 8), dtype=torch.uint8, device="cuda")
        out = P.encode_bits(mm, info)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
        ev[0].record()
        for i in range(10):
            P.encode_bits(mm, info)
            ev[i + 1].record()
        torch.cuda.synchronize()
        per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(10))
        dt = per[5] * 1e-3
        gbs = w * (info.shape[1] + out.shape[1]) / dt / 1e9
        print(f"wimax {n} {rate} z={mm.z}: {w * mm.n / dt / 1e12:.2f} Tb/s coded, {gbs:.0f} GB/s HBM (median {dt * 1e6:.0f} us)")
        del info, out
