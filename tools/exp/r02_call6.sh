# round 2: scaled codes with a 128-register cap (4 warps per SMSP) x codewords per CTA;
# C1 with in-graph events; then compute-sanitizer memcheck on tools/sanitize_cases.py
cd $GRAFT_REPO_ROOT
for g in 1 2 3 4; do
  QCB_LIB=$PWD/paper_2306_12063_b200/lib_cap128.so QCB_CW_PER_CTA=$g timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/cap_g$g.json > /dev/null 2>&1; echo "cap G=$g rc=$?"
done
timeout 300 python bench.py --config C1 --no-cpu --no-e2e > gpurun_out/c1_ingraph.json 2> gpurun_out/c1_ingraph.err; echo "c1 rc=$?"; cut -c1-400 gpurun_out/c1_ingraph.json; tail -3 gpurun_out/c1_ingraph.err
bash tools/sanitize_run.sh memcheck
