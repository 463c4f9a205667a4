# C5: finer sweep of the TMEM register cap / tier count (all keep 4 warps per sub-partition)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lib in libqcb200.so lib_cap112.so lib_cap108.so lib_cap104.so lib_tmt2.so lib_t2c112.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C5', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
for lib in libqcb200.so lib_cap112.so lib_t2c112.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python tools/codebench.py --codes wimax-2304-r56,wifi-1944-r34A --arith i16 --w 262144 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$lib', d['code'], d['gbit_s'])
    except Exception: pass"
done
