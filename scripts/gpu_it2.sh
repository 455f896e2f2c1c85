cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0 > $R/q_bench.log 2>&1; echo "bench=$?" >> $R/q_status.txt
timeout 300 python scripts/pcie_bw.py > $R/q_pcie.log 2>&1; echo "pcie=$?" >> $R/q_status.txt
