# round-2 (third session) evidence: GPU tests, smoke, default bench line, cfg5 launch
# list, merge DRAM bytes, --set full of one large k4_merge_level launch and of the
# leaf / run-detection / long-leaf kernels.  Each ncu pass only after its plain
# command exited 0.
cd $GRAFT_REPO_ROOT
R=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $R/e4_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $R/e4_tests.log 2>&1; echo "tests=$?" > $R/e4_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/e4_smoke.log 2>&1; echo "smoke=$?" >> $R/e4_status.txt
timeout 900 python bench.py > $R/e4_bench.log 2>&1; echo "bench=$?" >> $R/e4_status.txt
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/e4_plain.log 2>&1; echo "plain=$?" >> $R/e4_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/e4_launches.csv $B > $R/e4_ncu1.log 2>&1; echo "launch=$?" >> $R/e4_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k4_merge_level" --csv --log-file $R/e4_merge_bytes.csv $B > $R/e4_ncu2.log 2>&1; echo "bytes=$?" >> $R/e4_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/e4_merge_full $B > $R/e4_ncu3.log 2>&1; echo "full=$?" >> $R/e4_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_runs_tables|k_runs_emit|k_long_leaves|k_powers_seg" -c 6 -o $R/e4_other_full $B > $R/e4_ncu5.log 2>&1; echo "other=$?" >> $R/e4_status.txt
