cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k4_desc" --csv --log-file $R/dl_8.csv $B > /dev/null 2>&1
for c in 4 16; do VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_c$c.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k4_desc" --csv --log-file $R/dl_$c.csv $B > /dev/null 2>&1; done
echo done > $R/dl_status.txt
