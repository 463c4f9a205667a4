# round 2: ncu evidence for the chunked row mapping (WiMAX 960 R3/4A f32, G = 4; 1152 R2/3B f32, G = 2)
cd $GRAFT_REPO_ROOT
for code in wimax-960-r34A wimax-1152-r23B; do
  timeout 300 python tools/codebench.py --codes $code --arith f32 --w 65536 > gpurun_out/p28_$code.log 2>&1 && \
  timeout 600 ncu --section MemoryWorkloadAnalysis_Tables --section SpeedOfLight --section LaunchStats --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:decode_layered -s 1 -c 1 --csv --page raw --log-file gpurun_out/ncu28_$code.csv python tools/codebench.py --codes $code --arith f32 --w 65536 > gpurun_out/ncu28_$code.log 2>&1; echo "$code ncu=$?"
  QCB_CHUNKED=0 true
done
