cd $GRAFT_REPO_ROOT
R=gpurun_out
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf_sort" -c 1 -o $R/p9_leaf $B1 > $R/p9_ncu.log 2>&1; echo "ncu=$?" > $R/p9_status.txt
