cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
: > $R/var_status.txt
for v in $VARIANTS; do
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 300 $B > $R/var_$v.log 2>&1; echo "$v=$?" >> $R/var_status.txt
done
