# C1: does an uncapped register budget (no occupancy to protect at 1.7 warps per sub-partition) shorten the one-warp chain?
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lib in libqcb200.so lib_slack100.so lib_slack160.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config C1 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C1', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
for lib in libqcb200.so lib_slack160.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib python tools/exp/c1_iters.py 1024 | cut -c1-60; done
