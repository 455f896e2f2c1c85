# GPU parity tests of the in-tree library, then an A/B of library variants on the cfg5 bench
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $R/abt_tests.log 2>&1; echo "tests=$?" > $R/abt_status.txt
bash scripts/gpu_ab.sh
