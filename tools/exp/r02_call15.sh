# round 2: ncu on lane-bound scaled codes (bank conflicts of multi-codeword CTAs?)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/codebench.py --codes wimax-864-r34A --arith f32 --w 65536 > gpurun_out/p15_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 1 -c 1 -o gpurun_out/prof_z36 python tools/codebench.py --codes wimax-864-r34A --arith f32 --w 65536 > gpurun_out/ncu_z36.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o gpurun_out/prof_z68 python tools/codebench.py --codes wimax-1632-r34A --arith i16 --w 65536 > gpurun_out/ncu_z68.log 2>&1; echo ncu2=$?
