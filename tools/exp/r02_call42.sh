# round 2 (session 4): final ncu refresh: C5, C3, C2 full captures of the final kernels (+ SASS source pages), C5 launch list
cd $GRAFT_REPO_ROOT
for c in C5 C3 C2; do
  k=decode_pair16; [ $c = C2 ] && k=decode_layered
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/p_plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_final_$c -f \
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/p_ncu_$c.log 2>&1; echo "ncu $c rc=$?"
  ncu -i gpurun_out/prof_final_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/final_${c}_sass.csv 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|encode" -c 100 --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_list_c5.log 2>&1; echo "launches rc=$?"
ls -la gpurun_out | tail -12
