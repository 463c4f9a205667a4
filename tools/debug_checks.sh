#!/bin/bash
# Device-side invariant checks in place of compute-sanitizer (closed on this GPU pool):
# builds paper_2306_12063_b200/lib_debug.so with QCB_DEBUG_CHECKS=1 (csrc/debug_checks.cuh:
# shared-memory bounds + alignment on every cell / table / I/O access, poisoned dynamic
# shared memory, CTA chunk inside the batch) -- here, on the CPU box:
#     bash tools/debug_checks.sh build
# and runs the GPU parity suite and tools/sanitize_cases.py against it -- under gpurun:
#     bash tools/debug_checks.sh run
set -e
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
if [ "$1" = "build" ]; then
  bash tools/exp/build_variant.sh debug "-DQCB_DEBUG_CHECKS=1"
  exit 0
fi
export QCB_LIB=$PWD/paper_2306_12063_b200/lib_debug.so
set +e
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/debug_pytest.log 2>&1
echo "debug pytest rc=$?"; tail -3 gpurun_out/debug_pytest.log
timeout 900 python tools/sanitize_cases.py > gpurun_out/debug_sanitize_cases.log 2>&1
echo "debug sanitize_cases rc=$?"; tail -2 gpurun_out/debug_sanitize_cases.log
QCB_CW_PER_CTA=3 timeout 900 python tools/sanitize_cases.py > gpurun_out/debug_sanitize_cases_g3.log 2>&1
echo "debug sanitize_cases (3 codewords / pairs per CTA) rc=$?"; tail -2 gpurun_out/debug_sanitize_cases_g3.log
QCB_CW_PER_CTA=4 timeout 900 python tools/sanitize_cases.py > gpurun_out/debug_sanitize_cases_g4.log 2>&1
echo "debug sanitize_cases (4 codewords / pairs per CTA: chunked row mapping where 8 | Z) rc=$?"; tail -2 gpurun_out/debug_sanitize_cases_g4.log
