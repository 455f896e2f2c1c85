# --set full of one large k4_merge_level launch (cfg5 2^30 bench, same launch index as profiles/r02_merge4_full.txt)
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/m4_plain.log 2>&1; echo "plain=$?" > $R/m4_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/m4_full $B > $R/m4_ncu.log 2>&1; echo "full=$?" >> $R/m4_status.txt
