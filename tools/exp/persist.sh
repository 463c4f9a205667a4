#!/bin/bash
for v in "1 1" "0 1" "1 0" "0 0"; do
  set -- $v
  echo -n "bulk=$1 persist=$2: "
  QCB_BULK=$1 QCB_PERSIST=$2 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])"
done
