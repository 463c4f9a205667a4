#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/eb.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2306_12063_b200 as P
mm = P.get_model_matrix("wifi", int(sys.argv[1]) if len(sys.argv) > 1 else 1944, sys.argv[2] if len(sys.argv) > 2 else "1/2")
info = torch.randint(0, 256, (1 << 22, (mm.k + 7) // 8), dtype=torch.uint8, device="cuda")
for _ in range(3): P.encode_bits(mm, info)
torch.cuda.synchronize()
PY
python /tmp/eb.py $1 $2 || exit 1
ncu --set full --clock-control none -k regex:encode -s 1 -c 1 -o gpurun_out/prof_eb -f python /tmp/eb.py $1 $2 > gpurun_out/p_eb.log 2>&1
ncu -i gpurun_out/prof_eb.ncu-rep --page details --csv > gpurun_out/eb_details.csv 2>&1
rm -f gpurun_out/prof_eb.ncu-rep
