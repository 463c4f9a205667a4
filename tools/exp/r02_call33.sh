# round 2 (session 4): PDL for single-wave float32 launches (C1), int16 sign-op pipe balance re-measured on the current C3 / C5 kernels
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c33_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c33_pytest.log
for p in 1 0; do
  QCB_PDL=$p timeout 300 python bench.py --config C1 --no-e2e --no-cpu > gpurun_out/c33_C1_pdl$p.log 2>&1; echo -n "C1 pdl=$p rc=$? "; tail -1 gpurun_out/c33_C1_pdl$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'], d['timing'][-40:])"
  QCB_PDL=$p timeout 300 python tools/exp/c1_iters.py 1024 > gpurun_out/c33_iters_pdl$p.log 2>&1; cat gpurun_out/c33_iters_pdl$p.log | cut -c1-70
done
for rep in 1 2; do
for c in C3 C5; do
for lib in libqcb200.so lib_as0.so lib_xs2.so lib_as0xs2.so; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
done
