cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/m4new $B > $R/m4new.log 2>&1; echo "full=$?" > $R/m4_status.txt
