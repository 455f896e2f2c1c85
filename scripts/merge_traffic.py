"""profiles/merge_level_traffic.json from the ncu DRAM-bytes CSV of the merge
launches (gpu_evidence.sh 'bytes' pass).  The command runs 3 sorts (stats,
warm-up, timed): the timed sort is the last third of the launches.
usage: python scripts/merge_traffic.py CSV ALGORITHMIC_BYTES_PER_STEP > profiles/merge_level_traffic.json"""
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
alg = float(sys.argv[2])
h = None
launches = {}
for r in rows:
    if "ID" in r and "Metric Name" in r:
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    i = int(r[h.index("ID")])
    m = r[h.index("Metric Name")]
    u = r[h.index("Metric Unit")]
    v = float(r[h.index("Metric Value")].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)
    launches.setdefault(i, {})[m] = v * scale
ids = sorted(launches)
timed = ids[2 * len(ids) // 3:]
per = []
for i in timed:
    d = launches[i]
    rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
    per.append({"bytes": rd + wr, "read": rd, "write": wr, "time_s": d.get("gpu__time_duration.sum", 0.0)})
tot = sum(p["bytes"] for p in per)
print(json.dumps({
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k "
              "regex:'k4_merge_level|k_merge_level' (bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "
              "--bounded-reps 0, n=2^30 cfg5, default two-level schedule; the timed sort = last third of the launches)",
    "launches": len(per), "bytes_per_step": tot, "bytes_per_launch": tot / max(len(per), 1),
    "algorithmic_bytes_per_step": alg, "traffic_over_algorithmic": tot / alg,
    "kernel_ms_per_step_ncu": sum(p["time_s"] for p in per) * 1e3, "per_launch": per}, indent=1))
