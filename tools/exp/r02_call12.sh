# round 2: TMEM-tier int16 kernels with several pairs per CTA (QCB_CW_PER_CTA) -- C3 / C5 structures
cd $GRAFT_REPO_ROOT
C="wifi-1944-r56,wifi-1944-r34A,wimax-2304-r34A,wimax-2304-r56"
for g in 1 2 3 4; do
  QCB_CW_PER_CTA=$g timeout 600 python tools/codebench.py --codes $C --arith i16 --w 262144 --iters 8 --json gpurun_out/tmg_g$g.json > gpurun_out/tmg_g$g.log 2>&1; echo "G=$g rc=$?"; tail -2 gpurun_out/tmg_g$g.log | cut -c1-200
done
