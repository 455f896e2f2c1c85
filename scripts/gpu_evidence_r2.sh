# round-2 ncu evidence for profiles/ (default schedule, cfg5 2^30): plain run,
# launch list, DRAM bytes of every merge launch, --set full of one large
# merge launch and of the other top kernels.  Each ncu pass only after the
# plain command exited 0.
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/ev2_plain.log 2>&1; echo "plain=$?" > $R/ev2_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/ev2_launches.csv $B > $R/ev2_ncu1.log 2>&1; echo "launch=$?" >> $R/ev2_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k4_merge_level" --csv --log-file $R/ev2_merge_bytes.csv $B > $R/ev2_ncu2.log 2>&1; echo "bytes=$?" >> $R/ev2_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/ev2_merge_full $B > $R/ev2_ncu3.log 2>&1; echo "full=$?" >> $R/ev2_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k4_desc" -s 8 -c 1 -o $R/ev2_desc_full $B > $R/ev2_ncu4.log 2>&1; echo "desc=$?" >> $R/ev2_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_runs_tables|k_runs_emit|k_long_leaves" -c 5 -o $R/ev2_other_full $B > $R/ev2_ncu5.log 2>&1; echo "other=$?" >> $R/ev2_status.txt
