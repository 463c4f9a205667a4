# round 2: C3 with several codeword pairs per CTA (no TMEM tiers, 128-register cap) vs default
cd $GRAFT_REPO_ROOT
C="wifi-1944-r56,wifi-1944-r34A,wifi-1944-r23A,wifi-1944-r12,wifi-1296-r56,wifi-648-r56"
timeout 600 python tools/codebench.py --codes $C --arith i16 --w 262144 --iters 8 --json gpurun_out/c3g_default.json > /dev/null 2>&1; echo "default rc=$?"
for g in 1 2 3 4; do
  QCB_LIB=$PWD/paper_2306_12063_b200/lib_t0.so QCB_CW_PER_CTA=$g timeout 600 python tools/codebench.py --codes $C --arith i16 --w 262144 --iters 8 --json gpurun_out/c3g_t0_g$g.json > /dev/null 2>&1; echo "t0 G=$g rc=$?"
done
for g in 1 2 3; do
  QCB_CW_PER_CTA=$g timeout 600 python tools/codebench.py --codes wifi-1944-r56,wifi-1944-r12,wifi-1296-r12,wifi-648-r12 --arith f32 --w 65536 --json gpurun_out/c3g_f32_g$g.json > /dev/null 2>&1; echo "f32 G=$g rc=$?"
done
