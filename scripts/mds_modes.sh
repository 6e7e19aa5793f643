# MDS tcgen05 pass bound analysis: full, no pair math (1), no MMAs (2), neither (3) at C3.
for m in 0 1 2 3; do
  echo "mode $m: $(BS_MDS_TC_MODE=$m timeout 300 python bench.py --workload mds_c3 --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["achieved"])')"
done
