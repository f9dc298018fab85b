# AlexNet-trunk conv sweep (BASELINE config 5): tensor-pipe utilisation and
# device time of every kernel of one training step, from ncu (serialised,
# cold cache), for profiles/<round>_alexnet_conv_sweep.md
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/sweep_alexnet.csv \
    python bench.py --workload alexnet_conv --steps 1 --warmup 3 --e2e-steps 1 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/sweep_alexnet.csv
