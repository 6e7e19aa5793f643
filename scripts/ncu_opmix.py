"""Executed-instruction mix by opcode (and hottest lines) of an ncu report: python scripts/ncu_opmix.py rep."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()[1:]))
h = r[0]
ie = h.index("Instructions Executed"); src = h.index("Source")
mix = collections.Counter()
tot = 0
for row in r[1:]:
    try:
        n = float(row[ie])
    except (ValueError, IndexError):
        continue
    s = row[src].strip()
    toks = s.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    mix[op.split(".")[0]] += n
    tot += n
print(f"total warp-instructions {tot:.4g}")
for op, n in mix.most_common(40):
    print(f"{100 * n / tot:5.1f}% {n:12.4g} {op}")
