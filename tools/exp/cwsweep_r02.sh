# round 2: codewords (pairs) per CTA for the runtime-Z (scaled WiMAX) kernels
cd $GRAFT_REPO_ROOT
CODES=wimax-576-r12,wimax-864-r34A,wimax-960-r34A,wimax-1056-r23B,wimax-1152-r12,wimax-1632-r12,wimax-1920-r56,wimax-2304-r12,wimax-2304-r34A
for g in 1 2 3 4; do
  echo "== G=$g"
  QCB_CW_PER_CTA=$g timeout 600 python tools/codebench.py --codes $CODES --w 65536 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['code'], d['arith'], d['z'], d['gbit_s'])"
done
