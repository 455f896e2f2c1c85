cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist_plan.py -q -x > $R/d_plan.log 2>&1; echo "dplan=$?" > $R/d_status.txt
timeout 1500 python -m pytest tests -m gpu -q > $R/d_tests.log 2>&1; echo "tests=$?" >> $R/d_status.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B > $R/d_two.log 2>&1; echo "two=$?" >> $R/d_status.txt
