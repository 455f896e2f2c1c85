# round-2 (fourth session) evidence refresh of HEAD: the plain command first, then
# merge DRAM bytes, --set full of one large k4_merge_level launch, of the leaf /
# run-detection / long-leaf kernels and of one large k4_desc launch.
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/e6_plain.log 2>&1; echo "plain=$?" > $R/e6_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k4_merge_level" --csv --log-file $R/e6_merge_bytes.csv $B > $R/e6_ncu2.log 2>&1; echo "bytes=$?" >> $R/e6_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/e6_merge_full $B > $R/e6_ncu3.log 2>&1; echo "full=$?" >> $R/e6_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_runs_tables|k_runs_emit|k_long_leaves|k_powers_seg" -c 6 -o $R/e6_other_full $B > $R/e6_ncu5.log 2>&1; echo "other=$?" >> $R/e6_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"^k4_desc$" -s 8 -c 1 -o $R/e6_desc_full $B > $R/e6_ncu4.log 2>&1; echo "desc=$?" >> $R/e6_status.txt
