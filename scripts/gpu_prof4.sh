cd $GRAFT_REPO_ROOT
R=gpurun_out
B1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0 --two-level"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4_merge_level" -s 4 -c 1 -o $R/p8_k4 $B1 > $R/p8_ncu.log 2>&1; echo "ncu=$?" > $R/p8_status.txt
