cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > $R/k_tests.log 2>&1; echo "tests=$?" > $R/k_status.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B > $R/k_two.log 2>&1; echo "two=$?" >> $R/k_status.txt
