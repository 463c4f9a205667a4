# round 2: ADDSIGN (default) vs XOR sign test (as0) vs TMEM-hybrid messages (t3, t4)
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for lib in lib_as0.so lib_t3.so lib_t4.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "126 or grouped or known or misaligned or full_size" > gpurun_out/t_$lib.log 2>&1; echo "$lib tests rc=$? $(tail -1 gpurun_out/t_$lib.log)"
done
for rep in 1 2; do
for c in C5 C3; do
for lib in libqcb200.so lib_as0.so lib_t3.so lib_t4.so; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode --no-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
done
done
