#!/bin/bash
# usage: tools/exp/build_variant.sh NAME "-DQCB_X=1 -DQCB_Y=2"
# builds paper_2306_12063_b200/lib_NAME.so from its own object directory
# (load it with QCB_LIB=$PWD/paper_2306_12063_b200/lib_NAME.so)
set -e
NAME=$1; FLAGS=$2
QCB_BUILD_DIR=build_$NAME QCB_LIB=$PWD/paper_2306_12063_b200/lib_$NAME.so QCB_NVCC_EXTRA="$FLAGS" \
  python -c "from paper_2306_12063_b200 import _build; _build.build()"
rm -rf paper_2306_12063_b200/build_$NAME   # object files do not travel (keeps the gpurun snapshot small)
echo "built lib_$NAME.so ($FLAGS)"
