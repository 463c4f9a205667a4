# round 2 (session 4): final bench lines C1-C5 + reference arm with the final build; C1 on two ranks (gloo, one GPU)
cd $GRAFT_REPO_ROOT
for c in C2 C4 C3; do timeout 900 python bench.py --config $c > gpurun_out/c36_bench_$c.log 2>&1; echo "$c=$? $(tail -1 gpurun_out/c36_bench_$c.log | cut -c1-120)"; done
timeout 1200 python bench.py > gpurun_out/c36_bench_C5.log 2>&1; echo "C5=$? $(tail -1 gpurun_out/c36_bench_C5.log | cut -c1-120)"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/c36_bench_ref.log 2>&1; echo "ref=$? $(tail -1 gpurun_out/c36_bench_ref.log | cut -c1-200)"
QCB_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config C1 --no-e2e --no-cpu > gpurun_out/c36_bench_C1_2ranks.log 2>&1; echo "C1x2=$? $(tail -1 gpurun_out/c36_bench_C1_2ranks.log | cut -c1-200)"
timeout 300 python bench.py --config C1 --no-e2e --no-cpu --steps 100 --warmup 10 2>&1 | tail -1 | cut -c1-200
