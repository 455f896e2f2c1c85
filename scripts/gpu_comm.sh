cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 600 python -m pytest tests/test_gpu_comm.py -q -x > $R/c_tests.log 2>&1; echo "comm=$?" > $R/c_status.txt
timeout 1200 python -m pytest tests -m gpu -q > $R/c_all.log 2>&1; echo "all=$?" >> $R/c_status.txt
