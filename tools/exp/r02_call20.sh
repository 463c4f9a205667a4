# round 2: A/B current vs 1b4b37e (before the chunked mapping / padded I/O) on C5 / C2 / C3, interleaved
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c20.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c20.log
for rep in 1 2; do
 for lib in libqcb200.so lib_old.so; do
  for c in C5 C2 C3; do
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-check > gpurun_out/ab_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$c.json'));print('$lib $c', d['value'], d['ms_per_step'])"
  done
 done
done
