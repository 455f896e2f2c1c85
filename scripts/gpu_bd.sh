cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bounded.py -m gpu -x -q > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 2 > $R/q_bd.log 2>&1; echo "bench=$?" >> $R/q_status.txt
timeout 600 python scripts/bench_bounded.py > $R/q_bd2.log 2>&1; echo "bb=$?" >> $R/q_status.txt
