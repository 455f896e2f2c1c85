"""LSU data-pipe and shared-memory wavefront metrics of one ncu report.
usage: python scripts/lsu_pipe.py REP"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
keys = ["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "derived__memory_l1_wavefronts_shared_excessive",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"  {k:78s} {r[i]} {u[i]}")
