# ncu --set full captures of a layerwise workload's hot kernels (arg 1) plus
# its launch list (per-kernel device time, cold cache, serialised).  The skip
# counts select a launch of the first warm-up step (order: DESIGN.md §5).
W=${1:-cifar10_quick}
run() {  # $1 = kernel regex, $2 = launches to skip, $3 = tag
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
     -o gpurun_out/full_${W}_$3 python bench.py --workload $W --steps 1 --warmup 1 --e2e-steps 1 --profile-steps 1 \
     --no-cpu-baseline > /dev/null 2>&1
}
if [ "$W" = alexnet_conv ]; then
  run tc_persistent 12 conv2_dgrad
  run tc_persistent 1 conv2_fwd
  run tc_persistent 11 conv2_wgrad
  run im2col_t 4 conv1_wgrad_im2col
  run pool_bwd_plane 2 pool1_bwd
else  # cifar10_quick (round 2 engines: plane tap GEMM, tap weight gradient)
  run conv_plane_taps 0 conv1_fwd
  run conv_plane_taps 1 conv2_fwd
  run conv_plane_taps 2 conv2_dgrad
  run conv_wgrad_taps 0 conv2_wgrad
  run stem_wgrad 0 conv1_wgrad
  run pool_fwd_generic 0 pool1_fwd
  run plane_pack 1 conv2_planes
  run tc_persistent 0 conv3_fwd
fi
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}.csv \
    python bench.py --workload $W --steps 2 --warmup 1 --e2e-steps 1 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
