# round 2: GPU test suite + a short bench (no ncu)
cd $GRAFT_REPO_ROOT
R=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $R/c_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $R/c_tests.log 2>&1; echo "tests=$?" > $R/c_status.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0 > $R/c_bench.log 2>&1; echo "bench=$?" >> $R/c_status.txt
