# ncu --set full of one large k4_merge_level launch (cfg5 2^30, launch 8 of
# the bench command) for each library in $AB_LIBS ("cur" = in-tree), reports
# gpurun_out/ncu_<tag>.ncu-rep; $NCU_K overrides the kernel regex, $NCU_S the skip
cd $GRAFT_REPO_ROOT
R=gpurun_out
K=${NCU_K:-k4_merge_level}
S=${NCU_S:-8}
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
for L in $AB_LIBS; do
  if [ "$L" = cur ]; then unset VMPS_LIB; tag=cur; else export VMPS_LIB=$GRAFT_REPO_ROOT/$L; tag=$(basename $L .so); fi
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o $R/ncu_$tag $B > $R/ncu_$tag.log 2>&1
  echo "$tag rc=$?" >> $R/ncu_status.txt
done
