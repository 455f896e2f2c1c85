cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B > $R/sk_with.log 2>&1
VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_noskip.so timeout 300 $B > $R/sk_without.log 2>&1
timeout 300 python scripts/skip_demo.py > $R/sk_demo_with.log 2>&1
VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_noskip.so timeout 300 python scripts/skip_demo.py > $R/sk_demo_without.log 2>&1
