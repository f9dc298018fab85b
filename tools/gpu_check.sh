# tests + launch list (ncu, per-kernel device time) + short bench
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; grep -E "^E  |passed|failed" gpurun_out/pytest_gpu.log | head -5
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv --log-file gpurun_out/launches_tf32.csv python bench.py --steps 40 --warmup 3 --e2e-steps 3 --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_last.json
python -c "import json; d=json.load(open('gpurun_out/bench_last.json')); print('value', d['value'], 'us/step', d['ms_per_step']*1e3)"
