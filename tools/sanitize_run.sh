# usage (under gpurun): bash tools/sanitize_run.sh <memcheck|racecheck|synccheck|initcheck> [--quick]
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md), after a plain run of the
# same command has exited 0.  Summary -> gpurun_out/sanitize_<tool>.log
cd $GRAFT_REPO_ROOT
TOOL=$1; shift
timeout 600 python tools/sanitize_cases.py "$@" > gpurun_out/sanitize_plain_$TOOL.log 2>&1 || { echo "plain run failed"; exit 1; }
EXTRA=""
[ "$TOOL" = "racecheck" ] && EXTRA="--racecheck-report all"
[ "$TOOL" = "memcheck" ] && EXTRA="--leak-check no"
timeout 2400 compute-sanitizer --tool $TOOL $EXTRA --print-limit 200 --log-file gpurun_out/sanitize_$TOOL.log \
  python tools/sanitize_cases.py "$@" > gpurun_out/sanitize_${TOOL}_stdout.log 2>&1
echo "sanitizer rc=$?"
tail -5 gpurun_out/sanitize_$TOOL.log
