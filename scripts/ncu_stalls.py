"""Summarise an ncu report of a warp-specialised tcgen05 kernel: per-launch time and DRAM
bytes, plus the stall samples on every mbarrier wait (by barrier slot) and the hottest SASS.

    python scripts/ncu_stalls.py REPORT.ncu-rep KERNEL_REGEX BAR_BASE_HEX [names...]

BAR_BASE_HEX is the shared-memory offset of the barrier array; names label the slots in
order (name*count expands, e.g. raw_full*8)."""
import csv
import io
import re
import subprocess
import sys


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep, kre, base = sys.argv[1], sys.argv[2], int(sys.argv[3], 16)
    names = []
    for a in sys.argv[4:]:
        n, _, c = a.partition("*")
        names += [f"{n}{i}" for i in range(int(c or 1))]
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr = raw[0]
    for r in raw[2:]:
        g = lambda k: r[hdr.index(k)] if k in hdr else "?"
        print("launch:", g("gpu__time_duration.sum"), "ms; dram read", g("dram__bytes_read.sum"), "GB; issue active",
              g("smsp__issue_active.avg.pct_of_peak_sustained_active"), "%")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                                           f"regex:{kre}", "--launch-count", "1"))))
    hdr = rows[1]
    seen, d = set(), []
    for r in rows[2:]:
        if len(r) == len(hdr) and r[0].startswith("0x") and r[0] not in seen:
            seen.add(r[0])
            d.append(r)
    f = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
    tot = sum(f(r[2]) for r in d)
    print(f"samples {tot:.0f}")
    for k, r in enumerate(d):
        m = re.search(r"SYNCS.PHASECHK.TRANS64.TRYWAIT P\d, \[R\d+\+URZ\+0x([0-9a-f]+)\]", r[1])
        if m:
            slot = (int(m.group(1), 16) - base) // 8
            s = sum(f(x[2]) for x in d[k:k + 3])
            if s / tot > 0.002:
                print(f"  wait {names[slot] if 0 <= slot < len(names) else slot:>12} {s / tot * 100:5.1f}%")
    print("hottest:")
    for r in sorted(d, key=lambda r: -f(r[2]))[:12]:
        print(f"  {r[0][-5:]} {f(r[2]) / tot * 100:5.1f}% {r[1][:80]}")


if __name__ == "__main__":
    main()
