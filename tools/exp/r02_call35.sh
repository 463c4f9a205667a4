# round 2 (session 4): final-build check: GPU suite, smoke, C1 bench + ncu capture (PDL kernel) + launch list
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c35_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c35_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/c35_smoke.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py --config C1 > gpurun_out/c35_bench_C1.log 2>&1; echo "C1=$?"; tail -1 gpurun_out/c35_bench_C1.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 6 -c 1 -o gpurun_out/prof_c1 -f python bench.py --config C1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c35_ncu_c1.log 2>&1; echo "ncu=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config C1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c35_launches.log 2>&1; echo "launches=$?"
