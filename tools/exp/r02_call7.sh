# round 2: parity (per-code caps + foreign-shift scaled Z); scaled refresh; int16 TMEM-tier /
# register-cap variants on the native codes and C5; then compute-sanitizer memcheck
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_c7.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c7.log
timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/ct4_scaled.json > /dev/null 2>&1; echo "scaled rc=$?"
for lib in libqcb200.so lib_t4c104.so lib_t4c96.so lib_t3c104.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python tools/codebench.py --codes native --arith i16 --w 262144 --json gpurun_out/tm_$lib.json > /dev/null 2>&1; echo "$lib rc=$?"
done
bash tools/sanitize_run.sh memcheck
