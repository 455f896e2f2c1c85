cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiny_tiles or reduced" > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B --leaf-radix > $R/lr_4.log 2>&1
VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_r5.so timeout 300 $B --leaf-radix > $R/lr_5.log 2>&1
timeout 300 $B > $R/lr_m.log 2>&1
