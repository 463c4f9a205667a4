timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_new.log 2>&1; echo "tests rc=$? $(tail -n 1 gpurun_out/t_new.log)"
bash tools/exp/ab_lib.sh "C2 C1 C4" libqcb200_fm0.so libqcb200.so 2>&1 | grep -v tests | head -6
for lib in libqcb200_fm0.so libqcb200.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/exp/percode.py 2>&1 | grep "'f32'" > gpurun_out/pcf_$lib.txt; done
paste -d' ' <(cut -c1-48 gpurun_out/pcf_libqcb200_fm0.so.txt) <(cut -d, -f5 gpurun_out/pcf_libqcb200.so.txt)
