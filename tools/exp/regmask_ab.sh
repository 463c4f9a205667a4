# per-code A/B of register-cap masks: none raised / all raised / current default
for lib in libqcb200_none.so libqcb200_all.so libqcb200.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/exp/percode.py > gpurun_out/pcm_$lib.txt 2>&1; done
paste -d' ' <(cut -c1-48 gpurun_out/pcm_libqcb200_none.so.txt) <(cut -d, -f5 gpurun_out/pcm_libqcb200_all.so.txt) <(cut -d, -f5 gpurun_out/pcm_libqcb200.so.txt)
