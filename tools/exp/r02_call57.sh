# float32 register-cap policy re-measured after the FFMA2 sign application: default vs all <= 128 (fa), none clamped (fb), all raised to the band top (fc), none raised (fd)
cd $GRAFT_REPO_ROOT
for lib in libqcb200.so lib_fa.so lib_fb.so lib_fc.so lib_fd.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/codebench.py --codes native --arith f32 --w 65536 > gpurun_out/c57_$lib.log 2>&1; echo "$lib rc=$?"
done
python - <<'PY'
import json
libs=["libqcb200.so","lib_fa.so","lib_fb.so","lib_fc.so","lib_fd.so"]
tab={}
for l in libs:
    for line in open(f"gpurun_out/c57_{l}.log"):
        try: d=json.loads(line)
        except Exception: continue
        tab.setdefault(d["code"],{})[l]=d["gbit_s"]
for c,v in tab.items(): print(c, [v.get(l) for l in libs])
PY
