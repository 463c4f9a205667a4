# round 2: codewords (pairs) per CTA for all 108 scaled WiMAX codes, f32 and int16
cd $GRAFT_REPO_ROOT
for g in 1 2 3 4; do
  QCB_CW_PER_CTA=$g timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/scaled_g$g.json > /dev/null 2>&1
  echo "G=$g rc=$?"
done
