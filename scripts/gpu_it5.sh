cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B > $R/q_two.log 2>&1; echo "two=$?" >> $R/q_status.txt
timeout 300 $B --one-level > $R/q_one.log 2>&1; echo "one=$?" >> $R/q_status.txt
