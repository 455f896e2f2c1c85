cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 600 python -m pytest tests/test_gpu_records.py -q -x > $R/rec_tests.log 2>&1; echo "rec=$?" > $R/rec_status.txt
timeout 900 python scripts/paper_sweep.py $R/paper_sweep.jsonl > $R/sweep.log 2>&1; echo "sweep=$?" >> $R/rec_status.txt
