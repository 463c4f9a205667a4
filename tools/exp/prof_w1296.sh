#!/bin/bash
# Wi-Fi 1296 (Z=54) f32 + int16: shared-memory wavefronts per access; torchrun single-rank smoke of bench
mkdir -p gpurun_out
python tools/exp/one_code.py wifi 1296 1/2 f32 65536 || exit 1
python tools/exp/one_code.py wifi 1296 1/2 i16 131072 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 2 -c 1 -o /tmp/prof_w1296 -f python tools/exp/one_code.py wifi 1296 1/2 f32 65536 > /dev/null 2>&1
ncu -i /tmp/prof_w1296.ncu-rep --page source --csv --print-source sass > gpurun_out/w1296_sass.csv 2>&1
python tools/profile_summary.py /tmp/prof_w1296.ncu-rep W1296 gpurun_out/w1296.json > /dev/null
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/tr1.log 2>&1; echo "torchrun rc=$?"; tail -1 gpurun_out/tr1.log | cut -c1-300
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/tr1r.log 2>&1; echo "torchrun ref rc=$?"; tail -1 gpurun_out/tr1r.log | cut -c1-300
