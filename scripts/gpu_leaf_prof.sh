# launch list of the cfg5 bench command + --set full (with source) of both k_leaf_sort classes
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/lp_plain.log 2>&1; echo "plain=$?" > $R/lp_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/lp_launches.csv $B > $R/lp_ncu1.log 2>&1; echo "launch=$?" >> $R/lp_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_leaf_sort -s 0 -c 2 -o $R/leaf_full $B > $R/lp_ncu2.log 2>&1; echo "full=$?" >> $R/lp_status.txt
