cd $GRAFT_REPO_ROOT
R=gpurun_out
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf_radix" -c 1 -o $R/p3_radix $B1 > $R/p3_ncu.log 2>&1; echo "ncu=$?" > $R/p3_status.txt
