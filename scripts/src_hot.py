"""Per-CUDA-line hot spots of one kernel in an ncu report (needs -lineinfo).
usage: python scripts/src_hot.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
cur_file = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    try:
        s, e = float(r[si] or 0), float(r[ei] or 0)
    except ValueError:
        continue
    k = (cur_file, ln)
    a = agg.setdefault(k, [0.0, 0.0, r[1]])
    a[0] += s
    a[1] += e
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts:.0f}, warp instructions {te:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:N]:
    print(f"{k[0]}:{k[1]:<5d} inst {v[1]/te*100:5.1f}%  stall {v[0]/ts*100:5.1f}%  {v[2].strip()[:80]}")
