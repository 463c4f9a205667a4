# round 2 (session 4): float32 sign application by FFMA2 + FMUL2 (default) against LOP3 + IMAD (lib_fma0): parity, then C2 / C4 / C1 and the native codes
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c40_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c40_pytest.log
for rep in 1 2; do
for c in C2 C4 C1; do
for lib in libqcb200.so lib_fma0.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python bench.py --config $c --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
done
for lib in libqcb200.so lib_fma0.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/codebench.py --codes native --arith f32 --w 65536 > gpurun_out/c40_native_$lib.log 2>&1; echo "$lib native rc=$?"
done
paste <(python -c "
import json
for l in open('gpurun_out/c40_native_libqcb200.so.log'):
    d=json.loads(l); print(d['code'], d['gbit_s'])") <(python -c "
import json
for l in open('gpurun_out/c40_native_lib_fma0.so.log'):
    d=json.loads(l); print(d['gbit_s'])")
