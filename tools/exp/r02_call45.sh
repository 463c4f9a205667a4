# round 2 (session 4): split tier barrier (bar.arrive / bar.sync per warp, two barrier sets) for the three-warp int16 WiMAX CTAs: lib_split vs default
cd $GRAFT_REPO_ROOT
QCB_LIB=$PWD/paper_2306_12063_b200/lib_split.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu -k "not scaled" > gpurun_out/c45_pytest.log 2>&1; echo "pytest(split)=$?"; tail -2 gpurun_out/c45_pytest.log
for rep in 1 2; do
for lib in libqcb200.so lib_split.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python bench.py --config C5 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C5', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
for lib in libqcb200.so lib_split.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python tools/codebench.py --codes wimax-2304-r12,wimax-2304-r23A,wimax-2304-r23B,wimax-2304-r34A,wimax-2304-r34B,wimax-2304-r56 --arith i16 --w 262144 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print('$lib', d['code'], d['gbit_s'])
    except Exception: pass"
done
