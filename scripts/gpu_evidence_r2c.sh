# round-2 (third session, final) evidence: GPU tests, smoke, default bench line, cfg5 launch
# list, merge DRAM bytes, --set full of one large k4_merge_level launch and of the
# leaf / run-detection / long-leaf kernels.  Each ncu pass only after its plain
# command exited 0.
cd $GRAFT_REPO_ROOT
R=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $R/e5_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $R/e5_tests.log 2>&1; echo "tests=$?" > $R/e5_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/e5_smoke.log 2>&1; echo "smoke=$?" >> $R/e5_status.txt
timeout 900 python bench.py > $R/e5_bench.log 2>&1; echo "bench=$?" >> $R/e5_status.txt
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 600 $B > $R/e5_plain.log 2>&1; echo "plain=$?" >> $R/e5_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/e5_launches.csv $B > $R/e5_ncu1.log 2>&1; echo "launch=$?" >> $R/e5_status.txt
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k4_merge_level" --csv --log-file $R/e5_merge_bytes.csv $B > $R/e5_ncu2.log 2>&1; echo "bytes=$?" >> $R/e5_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k4_merge_level -s 8 -c 1 -o $R/e5_merge_full $B > $R/e5_ncu3.log 2>&1; echo "full=$?" >> $R/e5_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_runs_tables|k_runs_emit|k_long_leaves|k_powers_seg" -c 6 -o $R/e5_other_full $B > $R/e5_ncu5.log 2>&1; echo "other=$?" >> $R/e5_status.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"^k4_desc$" -s 8 -c 1 -o $R/e5_desc_full $B > $R/e5_ncu4.log 2>&1; echo "desc=$?" >> $R/e5_status.txt
timeout 900 python bench.py --impl reference > $R/e5_ref.log 2>&1; echo "ref=$?" >> $R/e5_status.txt
