cd $GRAFT_REPO_ROOT
R=gpurun_out
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_runs_tables|k_runs_emit|k_powers_seg" -c 3 -o $R/p10_front $B1 > $R/p10_ncu.log 2>&1; echo "ncu=$?" > $R/p10_status.txt
