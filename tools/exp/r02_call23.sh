# round 2: C4 traffic (DRAM bytes of the 18 kernels of one grouped step) + launch list for C4
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config C4 --profile --steps 1 --warmup 1 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:decode_ -s 18 -c 18 --csv --log-file gpurun_out/c4_metrics.csv python bench.py --config C4 --profile --steps 1 --warmup 1 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --profile --steps 2 --warmup 1 > gpurun_out/ncu_c4l.log 2>&1; echo ncu_c4l=$?
ls -la gpurun_out
