#!/bin/bash
# A/B of run-time environment variants on one box: bench (no CPU baseline, no
# fp32 record) alternated twice per variant.  usage: tools/ab_env.sh "A=1" "A=0" ...
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  for v in "$@"; do
    r=$(env $v timeout 300 python bench.py --no-cpu-baseline --no-fp32 --e2e-steps 300 --steps 5000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f us/step' % (d['ms_per_step']*1e3))")
    echo "$v: $r"
  done
done
