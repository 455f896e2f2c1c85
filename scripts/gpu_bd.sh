cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 300 python scripts/bd_probe.py 24 2 > $R/bd_24.log 2>&1
timeout 300 python scripts/bd_probe.py 26 2 > $R/bd_26.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bd_" -s 300 -c 300 --csv --log-file $R/bd_launch.csv python scripts/bd_probe.py 24 1 > $R/bd_ncu.log 2>&1
echo done > $R/bd_status.txt
