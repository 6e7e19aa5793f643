# C4 (float32 Cox, fused one-stream pass): plain bench first, then ncu passes (B200_PROFILING.md).
set -x
python bench.py --workload cox_c4 --steps 10 --warmup 3 > gpurun_out/c4_plain.json 2> gpurun_out/c4_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c4_launches.csv \
    python bench.py --workload cox_c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4_ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none \
    -k regex:cox_fused2_kernel -c 3 --csv --log-file gpurun_out/c4_traffic.csv \
    python bench.py --workload cox_c4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4_traffic.log 2>&1
