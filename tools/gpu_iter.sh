#!/bin/bash
# quick GPU iteration: build, the selected GPU tests (PYTEST_FILES, default the
# LeNet parity + loopback DP tests), smoke, a default bench line without the CPU
# baseline, then the in-graph step timeline from a -DPN_STEPTRACE rebuild (last:
# it replaces libpn.so on the box)
cd "$(dirname "$0")/.."
out=gpurun_out; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -30 $out/build.log; exit 1; }
F=${PYTEST_FILES:-tests/test_gpu_parity.py tests/test_gpu_dp_loopback.py tests/test_gpu_smoke.py}
timeout 1200 python -m pytest $F -x -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > $out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -4 $out/pytest_iter.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > $out/bench_iter.json 2> $out/bench_iter.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1])
print("value %.0f  us/step %.2f  e2e %.0f  inf %.0f" % (d["value"], d["ms_per_step"] * 1e3, d["e2e"]["value"], d.get("inference", {}).get("value", 0)))
if "fp32" in d: print("fp32 us/step %.1f" % (d["fp32"]["ms_per_step"] * 1e3))
print({k: round(v * 1e3, 2) for k, v in d["stages_ms"].items()})
PY
PN_NVCC_FLAGS=-DPN_STEPTRACE timeout 300 python tools/step_trace.py tf32 2>&1 | grep -v Warn > $out/step_trace.log; cat $out/step_trace.log
