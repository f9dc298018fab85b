# e2e A/B of compile-time variants: tools/ab_e2e.sh "-DX" ...
for v in "$@"; do
  if [ "$v" = "-" ]; then export PN_NVCC_FLAGS=""; else export PN_NVCC_FLAGS="$v"; fi
  python -c "from paper_2005_13076_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for r in 1 2; do python bench.py --no-cpu-baseline --steps 2000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['ms_per_step']*1e3,2), round(d['e2e']['value']/1e6,3))"; done
done
