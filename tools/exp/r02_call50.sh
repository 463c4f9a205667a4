# int16 early termination at small Z: desynchronised one-warp CTAs starve on instruction fetch (no_instruction 2.0 per issue).
# Fewer, larger CTAs (several pairs per CTA, CTA barriers: lib_ws0 = QCB_WARP_SYNC=0) share their instruction stream.
cd $GRAFT_REPO_ROOT
for g in 0 1 2 4 8; do
  for code in "wifi 648 1/2" "wimax 768 3/4A"; do
    for et in 1 0; do
      if [ $g = 0 ]; then echo -n "default lib: "; python tools/exp/fixed_one.py $code i16 2.5 $et;
      else echo -n "ws0 G=$g: "; QCB_LIB=$PWD/paper_2306_12063_b200/lib_ws0.so QCB_CW_PER_CTA=$g python tools/exp/fixed_one.py $code i16 2.5 $et; fi
    done
  done
done
for g in 0 2 3; do
  for et in 1 0; do
  if [ $g = 0 ]; then echo -n "default lib: "; python tools/exp/fixed_one.py wifi 1296 1/2 i16 2.5 $et;
  else echo -n "G=$g: "; QCB_CW_PER_CTA=$g python tools/exp/fixed_one.py wifi 1296 1/2 i16 2.5 $et; fi
  done
done
