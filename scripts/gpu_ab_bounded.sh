cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 600 python -m pytest tests/test_gpu_bounded.py -q -x > $R/bdv_tests.log 2>&1; echo "tests=$?" >> $R/bdv_tests.log
: > $R/bdv.log
for it in 1 2; do for v in $VARIANTS; do
  echo -n "$v " >> $R/bdv.log
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 300 python scripts/bd_probe.py ${LG:-30} 2 >> $R/bdv.log 2>&1
done; done
