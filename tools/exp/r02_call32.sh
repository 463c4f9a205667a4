cd $GRAFT_REPO_ROOT
for w in 148 1024; do
QCB_SPLIT_MAX_W=0 python tools/exp/c1_iters.py $w > gpurun_out/c32_iters_one_$w.log 2>&1; echo one $w; cat gpurun_out/c32_iters_one_$w.log
QCB_SPLIT_MAX_W=100000 python tools/exp/c1_iters.py $w > gpurun_out/c32_iters_split_$w.log 2>&1; echo split $w; cat gpurun_out/c32_iters_split_$w.log
done
