# round 2: product build (one TMEM store wait per sweep) parity + C5 / C3 benches; debug-check build
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_c8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c8.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c5_w0.json 2> gpurun_out/bench_c5_w0.err; echo "c5 rc=$?"; cut -c1-160 gpurun_out/bench_c5_w0.json
timeout 300 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/bench_c3_w0.json 2>/dev/null; echo "c3 rc=$?"; cut -c1-160 gpurun_out/bench_c3_w0.json
bash tools/debug_checks.sh run
