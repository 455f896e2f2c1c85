cd $GRAFT_REPO_ROOT
R=gpurun_out
LOG2N5=24 timeout 600 python scripts/bench_bounded.py > $R/bp_plain.log 2>&1
LOG2N5=24 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bd_" --csv --log-file $R/bp_launches.csv python scripts/bench_bounded.py > $R/bp_ncu.log 2>&1; echo "ll=$?" > $R/bp_status.txt
