# byte-input (NEXT #4) GPU checks + bench lines with the pipelined e2e
timeout 600 python -m pytest tests/test_data_ingest.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_ingest.log 2>&1; tail -3 gpurun_out/pytest_ingest.log
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_last.json; python -c "import json; d=json.load(open('gpurun_out/bench_last.json')); print('value', d['value'], 'us/step', d['ms_per_step']*1e3, 'e2e', d['e2e'])"
timeout 300 python bench.py --workload cifar10_quick --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_cifar.json; python -c "import json; d=json.load(open('gpurun_out/bench_cifar.json')); print('value', d['value'], 'us/step', d['ms_per_step']*1e3, 'e2e', d['e2e'])"
