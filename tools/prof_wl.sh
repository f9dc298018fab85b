# ncu --set full captures of the layerwise-plan kernels of one workload (arg 1)
# plus its launch list (per-kernel device time, cold cache, serialised).
W=${1:-cifar10_quick}
run() {  # $1 = kernel regex, $2 = launches to skip, $3 = tag
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
     -o gpurun_out/full_${W}_$3 python bench.py --workload $W --steps 1 --warmup 1 --e2e-steps 1 --profile-steps 1 \
     --no-cpu-baseline > /dev/null 2>&1
}
run conv_tap_tma 1 tap_fwd          # second tap-GEMM launch of the step (conv2 fwd on both workloads)
run conv_gemm_tma 1 gemm            # wgrad / fwd GEMM over materialised operands
run im2col_t 1 im2col_t
run pool_bwd_plane 0 pool_bwd
run to_nhwc 1 nhwc
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}.csv \
    python bench.py --workload $W --steps 2 --warmup 1 --e2e-steps 1 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
