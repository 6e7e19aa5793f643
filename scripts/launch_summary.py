"""Per-kernel time summary of an ncu launch list (gpu__time_duration.sum CSV): last N launches."""
import collections, csv, sys
path = sys.argv[1]
tail = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mv = h.index("Kernel Name"), h.index("Metric Value")
data = [(r[ki], float(r[mv].replace(",", ""))) for r in rows[1:] if r[mv].replace(",", "").replace(".", "").isdigit()]
if tail:
    data = data[-tail:]
tot = sum(v for _, v in data)
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in data:
    name = k.split("(")[0].replace("void ", "")[:70]
    agg[name][0] += 1
    agg[name][1] += v
print(f"{len(data)} launches, {tot / 1e3:.1f} us total")
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{100 * t / tot:5.1f}%  {n:4d}x  {t / n / 1e3:9.1f} us  {name}")
