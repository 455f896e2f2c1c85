cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0 --log2n ${LOG2N:-30} ${EXTRA:-}"
timeout 600 $B > $R/ll_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|k4_" --csv --log-file $R/ll_launches.csv $B > $R/ll_ncu.log 2>&1; echo "ll=$?" > $R/ll_status.txt
