# Round profile: launch list (every kernel, device time) of a short bench run,
# one `ncu --set full` capture per tensor-core / SIMT hot kernel.  Writes into gpurun_out/.
PREC=${1:-tf32}
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 80 --csv \
    --log-file gpurun_out/launches_${PREC}.csv python bench.py --precision $PREC --steps 40 --warmup 3 \
    --e2e-steps 3 --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
for K in conv2_dgrad_persistent conv2_fwd_persistent conv2_wgrad_persistent IpFwd IpWgrad IpDgradUnpool \
         lenet_conv1_wgrad conv1_pool1_tc lenet_ip2_loss lenet_ip2_bwd lenet_solver \
         reduce_partials_multi; do
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 8 -c 1 \
      -o gpurun_out/full_$K python bench.py --precision $PREC --steps 10 --warmup 3 --e2e-steps 3 \
      --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out
