# two-level mode phases at 2^30; ncu --set full of the front-half and leaf kernels at 2^30
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B --two-level > $R/p2_two.log 2>&1; echo "two=$?" > $R/p2_status.txt
timeout 600 $B > $R/p2_one.log 2>&1; echo "one=$?" >> $R/p2_status.txt
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_runs_tables|k_runs_emit|k_leaf_sort|k_powers_seg|k_long_leaves" -c 5 -o $R/p2_front $B1 > $R/p2_ncu1.log 2>&1; echo "ncu1=$?" >> $R/p2_status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile_desc" -s 10 -c 2 -o $R/p2_desc $B1 > $R/p2_ncu2.log 2>&1; echo "ncu2=$?" >> $R/p2_status.txt
