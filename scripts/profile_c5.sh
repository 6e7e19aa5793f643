# C5 (2-bit packed genotypes) profiling: plain bench first, then ncu passes (B200_PROFILING.md).
set -x
python bench.py --workload cox_c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/c5_plain.json 2> gpurun_out/c5_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c5_launches.csv \
    python bench.py --workload cox_c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/c5_ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:u2_ring -c 4 --csv \
    --log-file gpurun_out/c5_traffic.csv python bench.py --workload cox_c5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/c5_traffic.log 2>&1
python scripts/u2_one.py 100000 u2 > /dev/null &&
ncu --set full --clock-control none --import-source on -k regex:u2_ring -c 2 -o gpurun_out/prof_u2_r01 python scripts/u2_one.py 100000 u2 > gpurun_out/c5_ncu_full.log 2>&1
