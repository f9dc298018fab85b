# one ncu --set full capture of the kernels matching $1 (regex), $2 launches
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$1 -s ${3:-20} -c ${2:-1} -o gpurun_out/prof_$1 python bench.py --steps 10 --warmup 3 --e2e-steps 3 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu_$1.log 2>&1
tail -2 gpurun_out/ncu_$1.log
