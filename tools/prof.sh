set -x
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 100 --csv --log-file gpurun_out/launches_tf32.csv python bench.py --steps 40 --warmup 3 --e2e-steps 3 --profile-steps 2 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 40 -c 6 -o gpurun_out/prof_tc python bench.py --steps 10 --warmup 3 --e2e-steps 3 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
