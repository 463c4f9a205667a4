# round 2: int16 pair kernel per native structure: ADDSIGN x TMEM-hybrid tiers
cd $GRAFT_REPO_ROOT
for lib in libqcb200.so lib_as0.so lib_as1t2.so lib_as1t3.so lib_as1t4.so lib_as0t3.so lib_as0t2.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python tools/codebench.py --codes native --arith i16 --w 262144 \
     --json gpurun_out/p16_$lib.json > /dev/null 2>&1; echo "$lib rc=$?"
done
