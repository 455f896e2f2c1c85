cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --maxfail=5 ${PYTEST_K:+-k "$PYTEST_K"} > $R/t_all.log 2>&1; echo "tests=$?" > $R/t_status.txt
