# ncu --set full of the general conv kernels on the AlexNet trunk (conv2 wgrad, conv2 fwd)
W=${1:-alexnet_conv}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_wgrad -s 3 -c 1 \
   -o gpurun_out/full_${W}_wgrad python bench.py --workload $W --steps 1 --warmup 1 --e2e-steps 1 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_fwd -s 1 -c 1 \
   -o gpurun_out/full_${W}_fwd python bench.py --workload $W --steps 1 --warmup 1 --e2e-steps 1 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
