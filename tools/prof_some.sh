# ncu --set full of the kernels named on the command line (demangled regex), one launch each
for K in "$@"; do
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 8 -c 1 \
      -o gpurun_out/full_$K python bench.py --steps 10 --warmup 3 --e2e-steps 3 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out
