cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 300 python scripts/bd_probe.py 30 1 > $R/bd_30.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bd_merge|k_bd_alloc" -s 20000 -c 200 --csv --log-file $R/bd_launch30.csv python scripts/bd_probe.py 30 1 > $R/bd_ncu30.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bd_merge" -s 10000 -c 1 -o $R/bd_merge30 python scripts/bd_probe.py 30 1 > $R/bd_ncu30f.log 2>&1
echo done > $R/bd_status.txt
