# A/B benchmark: tools/ab.sh "ENV=1" "ENV2=1" ...  (variant "-" = no extra env); 2 rounds, ms/step each
for r in 1 2; do
  for v in "$@"; do
    if [ "$v" = "-" ]; then e=""; else e="$v"; fi
    env $e python bench.py --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 > /tmp/ab.json
    python -c "import json; d=json.load(open('/tmp/ab.json')); print('$v', round(d['ms_per_step']*1e3,2))"
  done
done
