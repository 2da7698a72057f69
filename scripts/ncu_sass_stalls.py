"""Per-SASS-instruction stall summary of one kernel from an ncu report:
python scripts/ncu_sass_stalls.py <rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]


def f(r, c):
    try:
        return float(r[h.index(c)] or 0)
    except ValueError:
        return 0.0


reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"{len(data)} instructions, {tot:.0f} samples")
agg = {c: sum(f(r, c) for r in data) for c in reasons}
print("by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    rs = sorted(((f(r, c), c[6:]) for c in reasons), reverse=True)[:3]
    print(f"{r[h.index('Address')]:>6} {f(r, 'Warp Stall Sampling (All Samples)') / tot:6.2%} "
          f"{r[h.index('Source')][:64]:64} " + " ".join(f"{n}:{v:.0f}" for v, n in rs if v))
