# address table for every int16 structure (lib_tab) against the measured policy: does a smaller sweep body help the desynchronised ET CTAs at small Z?
cd $GRAFT_REPO_ROOT
for lib in libqcb200.so lib_tab.so; do
  for code in "wifi 648 1/2" "wifi 648 5/6" "wifi 1296 5/6"; do
    for et in 1 0; do echo -n "$lib: "; QCB_LIB=$PWD/paper_2306_12063_b200/$lib python tools/exp/fixed_one.py $code i16 2.5 $et; done
  done
done
