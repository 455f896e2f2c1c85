cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B --leaf-merge --fuse-z 1024 > $R/ab_mz1024.log 2>&1; echo "mz1024=$?" > $R/p4_status.txt
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0 --leaf-merge"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_level" -s 8 -c 2 -o $R/p4_merge $B1 > $R/p4_ncu.log 2>&1; echo "ncu=$?" >> $R/p4_status.txt
