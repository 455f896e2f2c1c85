cd $GRAFT_REPO_ROOT
R=gpurun_out
free -g > $R/q_free.log; nproc >> $R/q_free.log
timeout 1200 python -m pytest tests -m gpu -x -q > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
timeout 900 python bench.py --bounded-reps 0 --no-cpu-baseline > $R/q_bench.log 2>&1; echo "bench=$?" >> $R/q_status.txt
