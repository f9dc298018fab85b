#!/bin/bash
# Same-box A/B of the working tree against another checkout of the repo
# (default .ab_old, a git worktree of an earlier commit with its libpn.so
# built): alternates bench.py runs, ms/step each.  usage: tools/ab_tree.sh [dir] [rounds]
cd "$(dirname "$0")/.."
other=${1:-.ab_old}
for r in $(seq ${2:-3}); do
  for d in . "$other"; do
    (cd "$d" && python bench.py --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 > /tmp/ab_tree.json)
    python -c "import json; d=json.load(open('/tmp/ab_tree.json')); print('$d', round(d['ms_per_step']*1e3,2))"
  done
done
