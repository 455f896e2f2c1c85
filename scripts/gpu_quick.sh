# quick iteration: all GPU tests, then the default bench line (no e2e / bounded / cpu legs)
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0 > $R/q_bench.log 2>&1; echo "bench=$?" >> $R/q_status.txt
