timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_new.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/t_new.log)"
bash tools/exp/ab_lib.sh "C5 C3" libqcb200_m0.so libqcb200_m1.so libqcb200.so 2>&1 | grep -v tests | head -6
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
for lib in libqcb200_m0.so libqcb200_m1.so libqcb200.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python /tmp/pc16.py > gpurun_out/pc16_$lib.txt 2>&1; done
paste gpurun_out/pc16_libqcb200_m0.so.txt gpurun_out/pc16_libqcb200_m1.so.txt gpurun_out/pc16_libqcb200.so.txt | awk -F'\t' '{split($1,a,")"); split($2,b,")"); split($3,c,")"); print a[1]")", a[2], b[2], c[2]}'
