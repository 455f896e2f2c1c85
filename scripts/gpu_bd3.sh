cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 600 python -m pytest tests/test_gpu_bounded.py -q -x > $R/bd3_tests.log 2>&1; echo "tests=$?" > $R/bd3_status.txt
timeout 300 python scripts/bd_probe.py 24 2 > $R/bd3_24.log 2>&1
timeout 300 python scripts/bd_probe.py 30 2 > $R/bd3_30.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bd_merge" -s 20000 -c 100 --csv --log-file $R/bd3_launch30.csv python scripts/bd_probe.py 30 1 > $R/bd3_ncu30.log 2>&1
echo done >> $R/bd3_status.txt
