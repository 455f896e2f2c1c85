# ncu evidence for profiles/: launch list of the bench command, DRAM bytes of
# every level-merge launch of one timed step at 2^30, full set on 2 launches.
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $B > $R/ev_plain.log 2>&1; echo "plain=$?" > $R/ev_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/ev_launches.csv $B > $R/ev_ncu1.log 2>&1; echo "launch=$?" >> $R/ev_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_merge_level -s 21 -c 21 --csv --log-file $R/ev_merge_bytes.csv $B > $R/ev_ncu2.log 2>&1; echo "bytes=$?" >> $R/ev_status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_merge_level -s 36 -c 2 -o $R/ev_merge_full $B > $R/ev_ncu3.log 2>&1; echo "full=$?" >> $R/ev_status.txt
