# round 2: C3 / C1 ncu captures + the codewords-per-CTA sweep of the scaled (runtime-Z) codes
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 300 python bench.py --config C1 --no-cpu --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?"
timeout 300 python bench.py --config C2 --no-cpu --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config C4 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
for g in 1 2 3 4; do
  QCB_CW_PER_CTA=$g timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/scaled_g$g.json > gpurun_out/scaled_g$g.log 2>&1
  echo "G=$g rc=$?"
done
timeout 300 python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/plain_c3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 3 -c 1 -o gpurun_out/prof_c3 python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 300 python bench.py --config C1 --profile --steps 3 --warmup 2 --no-graph > gpurun_out/plain_c1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 3 -c 1 -o gpurun_out/prof_c1 python bench.py --config C1 --profile --steps 3 --warmup 2 --no-graph > gpurun_out/ncu_c1.log 2>&1; echo ncu_c1=$?
timeout 300 python bench.py --config C2 --profile --steps 3 --warmup 2 > gpurun_out/plain_c2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --config C2 --profile --steps 3 --warmup 2 > gpurun_out/ncu_c2.log 2>&1; echo ncu_c2=$?
