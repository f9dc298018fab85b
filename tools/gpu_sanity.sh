timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/step_probe.py > gpurun_out/step_probe.log 2>&1; tail -40 gpurun_out/step_probe.log
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench_last.json; cat gpurun_out/bench_last.json | head -c 600
