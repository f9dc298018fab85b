# A/B of compile-time variants on a bench workload: tools/ab_build_wl.sh <workload> <stage-substring> "-DX" ...
WL=$1; SUB=$2; shift 2
for v in "$@"; do
  if [ "$v" = "-" ]; then export PN_NVCC_FLAGS=""; else export PN_NVCC_FLAGS="$v"; fi
  python -c "from paper_2005_13076_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  python bench.py --workload $WL --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 > /tmp/ab.json
  python -c "import json; d=json.load(open('/tmp/ab.json')); print('$v', round(d['ms_per_step']*1e3,2), {k: round(x*1e3,1) for k,x in d['stages_ms'].items() if '$SUB' in k})"
done
