# ET syndrome grouping A/B (first group size), parity on the variants, then et_perf per lib
for lib in libqcb200_e1.so libqcb200_e2.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_$lib.log 2>&1; echo "$lib tests rc=$? $(tail -1 gpurun_out/t_$lib.log)"
done
for lib in libqcb200.so libqcb200_e1.so libqcb200_e2.so; do echo "== $lib"; QCB_LIB=$PWD/paper_2306_12063_b200/$lib python tools/exp/et_perf.py 2>&1 | grep " ET "; done
