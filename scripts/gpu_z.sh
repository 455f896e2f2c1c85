cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --bounded-reps 0"
for z in 512 1024; do timeout 300 $B --fuse-z $z > $R/z_$z.log 2>&1; done
