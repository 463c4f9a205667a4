# round 2: parity with the measured scaled plans; per-code refresh; Z = 24 with CTA barriers;
# C3 address-table variants; C1 step timing with / without the CUDA graph
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_c4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c4.log
timeout 900 python tools/codebench.py --codes all --w 65536 --json gpurun_out/ct2_default.json > /dev/null 2>&1; echo "default rc=$?"
Z24=$(python -c "print(','.join(f'wimax-576-{r}' for r in ('r12','r23A','r23B','r34A','r34B','r56')))")
for g in 1 2 3 4; do
  QCB_LIB=$PWD/paper_2306_12063_b200/lib_z24.so QCB_CW_PER_CTA=$g timeout 600 python tools/codebench.py --codes $Z24 --w 65536 --json gpurun_out/z24_g$g.json > /dev/null 2>&1; echo "z24 G=$g rc=$?"
done
for lib in libqcb200.so lib_c3tab.so lib_c3tabsel.so lib_c3tabt0.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python tools/codebench.py --codes native --arith i16 --w 262144 --iters 8 --json gpurun_out/c3v_$lib.json > /dev/null 2>&1; echo "$lib rc=$?"
done
for i in 1 2; do
timeout 300 python bench.py --config C1 --no-cpu --no-e2e > gpurun_out/c1_graph_$i.json 2>/dev/null; echo "c1 graph rc=$?"
timeout 300 python bench.py --config C1 --no-cpu --no-e2e --no-graph > gpurun_out/c1_nograph_$i.json 2>/dev/null; echo "c1 nograph rc=$?"
done
