# quick GPU iteration: LeNet parity tests, in-graph timeline, default bench line
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; tail -15 gpurun_out/pytest_parity.log
timeout 300 python tools/step_probe.py > gpurun_out/step_probe.log 2>&1; grep -v Warn gpurun_out/step_probe.log | tail -22
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_last.json; python -c "import json; d=json.load(open('gpurun_out/bench_last.json')); print('value', d['value'], 'us/step', d['ms_per_step']*1e3, d['roofline'])"
