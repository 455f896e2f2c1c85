# round-2 (second session) evidence: default bench line, cfg5 launch list, bounded
# trace / cell sweep / one k_bd_level capture.  Each ncu pass only after its plain
# command exited 0.
cd $GRAFT_REPO_ROOT
R=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $R/e3_smi.txt 2>&1
timeout 900 python bench.py > $R/e3_bench.log 2>&1; echo "bench=$?" > $R/e3_status.txt
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/e3_plain.log 2>&1; echo "plain=$?" >> $R/e3_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/e3_launches.csv $B > $R/e3_ncu1.log 2>&1; echo "launch=$?" >> $R/e3_status.txt
VMPS_BD_TRACE=1 timeout 600 python scripts/bd_probe.py 30 1 > $R/e3_bdtrace.log 2>&1; echo "bdtrace=$?" >> $R/e3_status.txt
CHUNKS=22,23,24,31 timeout 900 python scripts/bd_cells_probe.py > $R/e3_cells.log 2>&1; echo "cells=$?" >> $R/e3_status.txt
export LOG2N=28 VMPS_BD_CELL=1073741824
timeout 300 python scripts/bd_one.py > $R/e3_bdone.log 2>&1; echo "bdone=$?" >> $R/e3_status.txt
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"^k_bd_level$" -s 8 -c 1 -o $R/e3_bdlevel_full python scripts/bd_one.py > $R/e3_ncu2.log 2>&1; echo "bdfull=$?" >> $R/e3_status.txt
