for rep in 1 2; do for c in C2 C1 C4; do for lib in libqcb200.so libqcb200_l1s0.so libqcb200_l0s1.so; do
 echo -n "$lib $c: "; QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
done; done; done
