"""Key throughput / stall numbers of one-kernel ncu reports: python scripts/ncu_summary.py rep [rep...]."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum",
        "smsp__sass_inst_executed_op_local_st.sum", "sm__cycles_active.avg"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, v = r[0], r[2]
    d = dict(zip(h, v))
    print(rep)
    for k in KEYS:
        print(f"  {k:70s} {d.get(k, '?')}")
    st = [(float(x), k) for k, x in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x]
    tot = sum(a for a, _ in st) or 1
    for a, k in sorted(st, reverse=True)[:8]:
        print(f"  {100 * a / tot:5.1f}% {k[len('smsp__pcsamp_warps_issue_stalled_'):]}")
