cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiny_tiles or reduced" > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B --two-level > $R/q_two.log 2>&1; echo "two=$?" >> $R/q_status.txt
