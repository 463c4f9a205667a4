# per-code int16 A/B: default lib vs the libs given as arguments
cat > /tmp/pc16.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
from paper_2306_12063_b200.workloads import ALL_18, device_llrs
dev = torch.device('cuda', 0)
for ci, code in enumerate(ALL_18):
    mm = P.get_model_matrix(*code)
    w = 65536
    llr, _ = device_llrs(mm, w, 3.0, 4000 + ci, True, dev)
    cfg = P.DecoderConfig(max_iterations=10, early_termination=False, arithmetic=P.Arithmetic.Fixed16)
    out = P.decode_batch(mm, llr, cfg); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): P.decode_batch(mm, llr, cfg, out=out)
    b.record(); torch.cuda.synchronize()
    print(code, round(w * mm.n / (a.elapsed_time(b) / 5 * 1e-3) / 1e9, 1), flush=True)
PY
for lib in libqcb200.so "$@"; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python /tmp/pc16.py > gpurun_out/pc16_$lib.txt 2>&1; done
paste -d' ' gpurun_out/pc16_libqcb200.so.txt $(for l in "$@"; do echo "<(awk '{print \$NF}' gpurun_out/pc16_$l.txt)"; done | tr '\n' ' ') 2>/dev/null || true
