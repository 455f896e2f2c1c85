"""Per-launch summary of an ncu report: time, DRAM bytes, instructions, issue, stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
names = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
         'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
         'sm__warps_active.avg.pct_of_peak_sustained_active',
         'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'smsp__sass_inst_executed_op_shared_ld.sum',
         'smsp__sass_inst_executed_op_shared_st.sum', 'smsp__sass_inst_executed_op_local_ld.sum',
         'smsp__sass_inst_executed_op_local_st.sum', 'launch__grid_size', 'launch__registers_per_thread']
st = [n for n in h if 'smsp__pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued')]
for r in rows[2:]:
    print('---')
    for nm in names:
        if nm in h:
            i = h.index(nm)
            print(f"  {nm:60s} {r[i][:70]} {u[i]}")
    f = lambda n: float(r[h.index(n)].replace(',', '') or 0)
    tot = sum(f(n) for n in st) or 1
    top = sorted(st, key=lambda n: -f(n))[:7]
    print('  stalls:', ', '.join(f"{n.split('stalled_')[1]} {f(n) / tot * 100:.0f}%" for n in top))
