#!/bin/bash
# One GPU round trip: build, the -m gpu suite with the parity report, smoke,
# and (optionally) compute-sanitizer over smoke and a short bench.
# usage: tools/gpu_round.sh [tests] [sanitize] [bench]
cd "$(dirname "$0")/.."
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
for step in "$@"; do
  case $step in
    tests)
      rm -f $out/parity.jsonl
      PN_PARITY_LOG=$out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -x -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > $out/pytest_gpu.log 2>&1
      echo "pytest rc=$?"; tail -5 $out/pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $out/smoke.log ;;
    sanitize)
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
          python -c "import __graft_entry__ as g; g.smoke()" > $out/sanitizer_$tool.log 2>&1
        echo "sanitizer $tool rc=$?"; tail -4 $out/sanitizer_$tool.log
        timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
          python tools/sanitize_extra.py > $out/sanitizer_extra_$tool.log 2>&1
        echo "sanitizer (extra plans) $tool rc=$?"; tail -4 $out/sanitizer_extra_$tool.log
      done ;;
    bench)
      timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; tail -c 3000 $out/bench.json ;;
  esac
done
