# round 2: chunked row mapping (conflict-free multi-codeword CTAs) -- parity, then the
# codewords-per-CTA sweep of the scaled codes at the default cap and at a 128-register cap
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_c16.log
for g in 1 2 3 4 8; do
  QCB_CW_PER_CTA=$g timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/ch_g$g.json > /dev/null 2>&1; echo "G=$g rc=$?"
done
for g in 2 3 4 8; do
  QCB_LIB=$PWD/paper_2306_12063_b200/lib_cap128.so QCB_CW_PER_CTA=$g timeout 900 python tools/codebench.py --codes scaled --w 65536 --json gpurun_out/chcap_g$g.json > /dev/null 2>&1; echo "cap G=$g rc=$?"
done
timeout 900 python tools/codebench.py --codes all --w 65536 --json gpurun_out/ch_default.json > /dev/null 2>&1; echo "default rc=$?"
