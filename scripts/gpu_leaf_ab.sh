# leaf kernel change: GPU parity tests, then an A/B of library variants on the cfg5 bench (phases)
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "parity or patterns or maxsize or paper or bounded" > $R/lab_tests.log 2>&1; echo "tests=$?" > $R/lab_status.txt
AB_LIBS="${AB_LIBS}" bash scripts/gpu_ab.sh
echo "ab=$?" >> $R/lab_status.txt
