timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_new.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/t_new.log)"
bash tools/exp/ab_lib.sh "C2 C5 C3 C1 C4" libqcb200_r0.so libqcb200.so 2>&1 | grep -v tests | head -10
for lib in libqcb200_r0.so libqcb200.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/exp/percode.py > gpurun_out/percode_$lib.txt 2>&1; done
paste -d' ' <(cut -c1-60 gpurun_out/percode_libqcb200_r0.so.txt) <(cut -d, -f4-6 gpurun_out/percode_libqcb200.so.txt)
