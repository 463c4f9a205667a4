bash tools/exp/pc16_ab.sh libqcb200_xs.so > /dev/null 2>&1
paste gpurun_out/pc16_libqcb200.so.txt gpurun_out/pc16_libqcb200_xs.so.txt | awk -F'\t' '{n=split($2,b," "); print $1, b[n]}'
