# ncu evidence for profiles/ (default schedule): launch list of the bench
# command, DRAM bytes of every merge launch (3 sorts: stats, warm-up, timed),
# --set full on two large merge launches and on the other top kernels.
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/ev_plain.log 2>&1; echo "plain=$?" > $R/ev_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/ev_launches.csv $B > $R/ev_ncu1.log 2>&1; echo "launch=$?" >> $R/ev_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k4_merge_level|k_merge_level" --csv --log-file $R/ev_merge_bytes.csv $B > $R/ev_ncu2.log 2>&1; echo "bytes=$?" >> $R/ev_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 2 -o $R/ev_merge_full $B > $R/ev_ncu3.log 2>&1; echo "full=$?" >> $R/ev_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_runs_tables|k_runs_emit|k_powers_seg|k_long_leaves" -c 6 -o $R/ev_other_full $B > $R/ev_ncu4.log 2>&1; echo "full2=$?" >> $R/ev_status.txt
