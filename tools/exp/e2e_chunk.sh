#!/bin/bash
# A/B of the host path's chunk size (QCB_HOST_CHUNK_MB) on the e2e number
mkdir -p gpurun_out
for cfg in C2 C5; do
  for mb in 8 16 32 64 128; do
    v=$(QCB_HOST_CHUNK_MB=$mb python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 10 --cpu-seconds 0.5 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['e2e']['value'], l['e2e']['ms_per_step'])")
    echo "$cfg chunk=${mb}MB e2e=$v"
  done
done
