for lib in libqcb200.so libqcb200_el0.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/exp/percode.py 2>&1 | grep "'f32'" > gpurun_out/pce_$lib.txt; done
paste -d' ' <(cut -c1-48 gpurun_out/pce_libqcb200.so.txt) <(cut -d, -f5 gpurun_out/pce_libqcb200_el0.so.txt)
