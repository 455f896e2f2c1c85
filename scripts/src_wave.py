"""Per-CUDA-line shared-memory wavefronts (total / excessive) of one kernel in an ncu report.
usage: python scripts/src_wave.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, cur, hdr = {}, None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        ln = int(r[0])
        w = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
        x = float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
        i = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault((cur, ln), [0.0, 0.0, 0.0, r[1]])
    a[0] += w; a[1] += x; a[2] += i
tw = sum(v[0] for v in agg.values()) or 1
print(f"total shared wavefronts {tw:.3e}, excessive {sum(v[1] for v in agg.values()):.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{k[0]}:{k[1]:<5d} wave {v[0]/tw*100:5.1f}%  ideal {v[2]:.2e} excess {v[1]:.2e}  {v[3].strip()[:70]}")
