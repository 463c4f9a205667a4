timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1
bash tools/exp/ab_lib.sh "C1 C4" libqcb200_ws0.so libqcb200.so 2>&1 | grep -v tests | head -4
for lib in libqcb200_ws0.so libqcb200.so; do echo "== $lib"; for ar in f32 i16; do for r in 1/2 5/6; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib python tools/exp/one_code.py wifi 648 $r $ar 65536; done; done; done
