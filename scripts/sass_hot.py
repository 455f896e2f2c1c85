"""Top SASS instructions of one kernel in an ncu report (stall samples, executed).
usage: python scripts/sass_hot.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si, ii, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
def num(x):
    try:
        return float(x or 0)
    except ValueError:
        return None
d = [r for r in rows[1:] if len(r) > ei and num(r[ii]) is not None]
tot_s = sum(float(r[ii] or 0) for r in d)
tot_e = sum(float(r[ei] or 0) for r in d)
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_e:.3e}, sass lines {len(d)}")
for idx, r in enumerate(d):
    r.append(idx)
top = sorted(d, key=lambda r: -float(r[ii] or 0))[:N]
for r in sorted(top, key=lambda r: r[-1]):
    print(f"{r[-1]:5d} {float(r[ii] or 0)/tot_s*100:5.1f}% ex={float(r[ei] or 0):.2e}  {r[si].strip()[:90]}")
