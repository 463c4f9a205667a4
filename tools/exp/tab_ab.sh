# address-table policy A/B per code: default / all tables / no tables
for lib in libqcb200.so libqcb200_ton.so libqcb200_toff.so; do QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/exp/percode.py > gpurun_out/pct_$lib.txt 2>&1; done
paste -d' ' <(cut -c1-48 gpurun_out/pct_libqcb200.so.txt) <(cut -d, -f5 gpurun_out/pct_libqcb200_ton.so.txt) <(cut -d, -f5 gpurun_out/pct_libqcb200_toff.so.txt)
