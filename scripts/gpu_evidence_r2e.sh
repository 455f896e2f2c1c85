# round-2 (fifth session) evidence refresh of HEAD (evict-first bulk loads in the
# level merge): the plain command first, then merge DRAM bytes and --set full of
# one large k4_merge_level launch.
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/e7_plain.log 2>&1; echo "plain=$?" > $R/e7_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k4_merge_level" --csv --log-file $R/e7_merge_bytes.csv $B > $R/e7_ncu2.log 2>&1; echo "bytes=$?" >> $R/e7_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/e7_merge_full $B > $R/e7_ncu3.log 2>&1; echo "full=$?" >> $R/e7_status.txt
