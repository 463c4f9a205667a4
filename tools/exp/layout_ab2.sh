timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_new.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/t_new.log)"
bash tools/exp/ab_lib.sh "C5 C3" libqcb200_old.so libqcb200.so 2>&1 | grep -v tests
