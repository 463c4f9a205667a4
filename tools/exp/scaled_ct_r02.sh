# round 2: compile-time scaled kernels -- parity, then per-code throughput (default plan,
# runtime-Z baseline, codewords-per-CTA sweep, TMEM for the degree-20 f32 codes)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_sc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_sc.log
timeout 900 python tools/codebench.py --codes all --w 65536 --json gpurun_out/ct_default.json > gpurun_out/ct_default.log 2>&1; echo "default rc=$?"
QCB_SCALED=0 timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/ct_runtime.json > /dev/null 2>&1; echo "runtime rc=$?"
for g in 1 2 3 4; do
  QCB_CW_PER_CTA=$g timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/ct_g$g.json > /dev/null 2>&1
  echo "G=$g rc=$?"
done
CODES=$(python -c "print(','.join(f'wimax-{24*z}-r56' for z in range(24,93,4)))")
QCB_TMEM=1 timeout 600 python tools/codebench.py --codes $CODES --arith f32 --w 65536 --json gpurun_out/ct_tmem_r56.json > /dev/null 2>&1; echo "tmem rc=$?"
