timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1
for code in "wimax 576 5/6" "wimax 1152 5/6" "wimax 1728 5/6" "wifi 1944 5/6" "wimax 2304 5/6"; do
  echo "$code default: $(python tools/exp/one_code.py $code f32 65536 | awk '{print $(NF-1)}')  register: $(QCB_LIB=$PWD/paper_2306_12063_b200/libqcb200_ts0.so python tools/exp/one_code.py $code f32 65536 | awk '{print $(NF-1)}')  tmem: $(QCB_TMEM=1 python tools/exp/one_code.py $code f32 65536 | awk '{print $(NF-1)}')"
done
