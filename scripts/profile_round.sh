# Profiling recipe (B200_PROFILING.md): plain run first, then ncu passes.
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 4 --csv \
    --log-file gpurun_out/gemm_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_traffic.log 2>&1
python scripts/tc_one.py wstep > /dev/null &&
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/prof_wstep_r01 python scripts/tc_one.py wstep > gpurun_out/ncu_full.log 2>&1
