# C2 NMF-APG bound analysis: accumulator group G, and BS_TC_MODE (1 = no A split, 2 = no MMAs).
run() { env "$@" timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 |
  python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["avg_launch_ms"], d["clocks"]["sm_mhz"])'; }
for g in 4 8 16; do echo "G=$g $(run BS_TC_GROUP=$g)"; done
for m in 1 2 3; do echo "mode=$m $(run BS_TC_MODE=$m)"; done
