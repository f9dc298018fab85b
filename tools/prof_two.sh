for K in IpDgradUnpool conv2_dgrad_persistent; do
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 8 -c 1 \
   -o gpurun_out/full_$K python bench.py --steps 10 --warmup 3 --e2e-steps 3 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu_$K.log 2>&1
tail -2 gpurun_out/ncu_$K.log
done
