cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_runs_tables|k_runs_emit|k_powers_seg|k_long_leaves" -c 6 -o $R/ev_other_full $B > $R/ev_ncu4.log 2>&1; echo "full2=$?" > $R/ev2_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k4_desc" -s 12 -c 2 -o $R/ev_desc_full $B > $R/ev_ncu5.log 2>&1; echo "full3=$?" >> $R/ev2_status.txt
