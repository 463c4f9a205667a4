# float32 degree-20 codes: TMEM kernel (default) vs register kernel at default / 128 / raised caps
for code in "wifi 1944 5/6" "wimax 2304 5/6"; do
  echo "$code TMEM: $(python tools/exp/one_code.py $code f32 65536 | awk '{print $(NF-1)}')"
  for lib in libqcb200.so libqcb200_a.so libqcb200_b.so; do
    echo "$code reg $lib: $(QCB_TMEM=0 QCB_LIB=$PWD/paper_2306_12063_b200/$lib python tools/exp/one_code.py $code f32 65536 | awk '{print $(NF-1)}')"
  done
done
