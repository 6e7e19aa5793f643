"""Top stall-sampled SASS lines of an ncu report: python scripts/ncu_hot.py rep [N]."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()[1:]))
h = r[0]
si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source"); ad = h.index("Address")
rows = []
for row in r[1:]:
    try:
        v = float(row[si])
    except (ValueError, IndexError):
        continue
    rows.append((v, row[ad][-5:], row[src].strip()))
tot = sum(v for v, _, _ in rows) or 1
for v, a, s in sorted(rows, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}% {a} {s[:120]}")
