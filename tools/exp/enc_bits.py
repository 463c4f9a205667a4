"""Throughput of the bit-granular packed encoder per Wi-Fi code:
device time per launch from CUDA events around 20 back-to-back launches."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
w = 1 << 22
for n in (648, 1296, 1944):
    for rate in ("1/2", "2/3", "3/4", "5/6"):
        mm = P.get_model_matrix("wifi", n, rate)
        info = torch.randint(0, 256, (w, (mm.k + 7) // 8), dtype=torch.uint8, device="cuda")
        out = P.encode_bits(mm, info)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        t0 = time.perf_counter()
        ev[0].record()
        for i in range(20):
            P.encode_bits(mm, info)
            ev[i + 1].record()
        torch.cuda.synchronize()
        host = (time.perf_counter() - t0) / 20
        per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
        dt = per[len(per) // 2] * 1e-3
        gbs = w * (info.shape[1] + out.shape[1]) / dt / 1e9
        print(f"wifi {n} {rate} z={mm.z}: {w * mm.n / dt / 1e12:.2f} Tb/s coded, {gbs:.0f} GB/s HBM "
              f"(median launch {dt * 1e6:.0f} us, host {host * 1e6:.0f} us/call)")
        del info, out
