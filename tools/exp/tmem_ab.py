"""A/B the float32 TMEM-message kernel (QCB_TMEM=1) against the register kernel (QCB_TMEM=0)
on the high-degree codes where spec_plan may choose it."""
import os, subprocess, sys
codes = [("wifi", 648, "5/6"), ("wifi", 1296, "5/6"), ("wifi", 1944, "5/6"), ("wimax", 2304, "5/6"), ("wimax", 1152, "5/6")]
prog = open("tools/exp/ctasweep.py").read().split("prog = r'''")[1].split("'''")[0]
for code in codes:
    row = []
    for v in ["default", "0", "1"]:
        env = dict(os.environ)
        if v != "default":
            env["QCB_TMEM"] = v
        r = subprocess.run([sys.executable, "-c", prog, code[0], str(code[1]), code[2], "0"], env=env,
                           capture_output=True, text=True)
        row.append((v, r.stdout.strip() or r.stderr.strip()[-80:]))
    print("f32", code, row, flush=True)
