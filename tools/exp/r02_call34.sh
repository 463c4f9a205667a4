# PDL with launch_dependents before the epilogue (lib_pdl2) against no PDL
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for p in 1 0; do
  QCB_LIB=$PWD/paper_2306_12063_b200/lib_pdl2.so QCB_PDL=$p timeout 300 python bench.py --config C1 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$p', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
QCB_LIB=$PWD/paper_2306_12063_b200/lib_pdl2.so QCB_PDL=1 timeout 300 python tools/exp/c1_iters.py 1024 | cut -c1-70
