"""Per-source-line hot spots from an ncu report (--page source, cuda+sass)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
lines = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        lines.append(r)
idx = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try:
        return float(r[idx[k]])
    except (ValueError, KeyError):
        return 0.0
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in lines)
keys = ["stall_barrier", "stall_long_sb", "stall_wait", "stall_short_sb", "stall_math", "stall_mio", "stall_lg"]
print(f"total samples {tot:.0f}")
for r in sorted(lines, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
    s = num(r, "Warp Stall Sampling (All Samples)")
    st = " ".join(f"{k[6:]}={num(r, k):.0f}" for k in keys if num(r, k) > 0.05 * s)
    print(f"{r[0]:>5s} {s / tot:6.1%} shx={num(r, 'L1 Wavefronts Shared Excessive'):9.0f} "
          f"gtag={num(r, 'L1 Tag Requests Global'):9.0f} {st} | {r[1].strip()[:60]}")
