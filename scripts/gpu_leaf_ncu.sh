# --set full of the leaf sort (both size classes) at cfg5 2^30, source-level
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort" -s 2 -c 2 -o $R/leaf_full $B > $R/leaf_ncu.log 2>&1; echo "leaf=$?" > $R/leaf_status.txt
