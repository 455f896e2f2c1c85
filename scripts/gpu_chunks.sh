cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --bounded-reps 0 --two-level"
timeout 300 $B > $R/ch_2.log 2>&1
for c in 1 4 8; do VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_c$c.so timeout 300 $B > $R/ch_$c.log 2>&1; done
