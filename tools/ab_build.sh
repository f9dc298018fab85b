# A/B of compile-time variants: tools/ab_build.sh "-DX=1" "-DX=2" ... (each: rebuild, bench twice)
for v in "$@"; do
  if [ "$v" = "-" ]; then export PN_NVCC_FLAGS=""; else export PN_NVCC_FLAGS="$v"; fi
  python -c "from paper_2005_13076_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for r in 1 2; do
    python bench.py --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 > /tmp/ab.json
    python -c "import json; d=json.load(open('/tmp/ab.json')); print('$v', round(d['ms_per_step']*1e3,2))"
  done
done
