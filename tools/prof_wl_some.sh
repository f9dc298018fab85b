# ncu --set full of kernels (demangled regex) in a given bench workload: prof_wl_some.sh <workload> <k1> [k2...]
WL=$1; shift
for K in "$@"; do
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 4 -c 1 \
      -o gpurun_out/full_${WL}_$K python bench.py --workload $WL --steps 6 --warmup 3 --e2e-steps 3 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out
