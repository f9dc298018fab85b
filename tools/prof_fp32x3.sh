# ncu captures of the fp32-class plan with PN_3XTF32 (bench --precision fp32x3): the 3xTF32 ip1
# kernels, the operand split, the SIMT conv2 gradients, and the launch list (writes gpurun_out/)
W=lenet_fp32x3
run() {
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$1 -s $2 -c 1 \
     -o gpurun_out/full_${W}_$3 python bench.py --precision fp32x3 --steps 5 --warmup 3 --e2e-steps 2 --profile-steps 1 \
     --no-cpu-baseline --no-fp32 > /dev/null 2>&1
}
run Ip3Fwd 2 ip1_fwd_3x
run "Ip3Grad" 4 ip1_grad_3x
run "split3" 4 split3
run lenet_conv2_dgrad_simt 2 conv2_dgrad
run lenet_conv2_wgrad_simt 2 conv2_wgrad
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}.csv \
    python bench.py --precision fp32x3 --steps 2 --warmup 3 --e2e-steps 1 --profile-steps 1 --no-cpu-baseline --no-fp32 > /dev/null 2>&1
ls gpurun_out
