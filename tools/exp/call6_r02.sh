cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python bench.py --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_c5_r02b.json; cat gpurun_out/bench_c5_r02b.json | cut -c1-300
bash tools/exp/scaled_sweep_r02.sh
python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 3 -c 1 -o gpurun_out/c3_r02 python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3=$?
python bench.py --config C1 --profile --steps 3 --warmup 2 --no-graph > gpurun_out/plain_c1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 3 -c 1 -o gpurun_out/c1_r02 python bench.py --config C1 --profile --steps 3 --warmup 2 --no-graph > gpurun_out/ncu_c1.log 2>&1; echo ncu_c1=$?
