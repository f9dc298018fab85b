# conv-engine tests + bench lines of the three workloads
timeout 900 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_parity.py -m gpu -q 2>&1 | grep -E "^E  .*(Error|error)|passed|failed" > gpurun_out/pytest_conv.log
cat gpurun_out/pytest_conv.log
timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_lenet.json
timeout 300 python bench.py --workload cifar10_quick --e2e-steps 200 --profile-steps 10 2>&1 | tail -3 > gpurun_out/bench_cifar.json
timeout 600 python bench.py --workload alexnet_conv --e2e-steps 10 --profile-steps 3 2>&1 | tail -3 > gpurun_out/bench_alex.json
timeout 600 python bench.py --workload alexnet_grouped --e2e-steps 10 --profile-steps 3 2>&1 | tail -3 > gpurun_out/bench_alexg.json
for f in lenet cifar alex alexg; do python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], 'us/step', d['ms_per_step']*1e3, d['roofline']['kernel'], d['roofline']['frac'])
except Exception as e: print('$f', 'ERR', open('gpurun_out/bench_$f.json').read()[-2000:])
"; done
