# end-of-session check: GPU tests, smoke, default bench line, reference arm, launch list
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $R/f_tests.log 2>&1; echo "tests=$?" > $R/f_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/f_smoke.log 2>&1; echo "smoke=$?" >> $R/f_status.txt
timeout 900 python bench.py > $R/f_bench.log 2>&1; echo "bench=$?" >> $R/f_status.txt
timeout 900 python bench.py --impl reference > $R/f_ref.log 2>&1; echo "ref=$?" >> $R/f_status.txt
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/f_launches.csv $B > $R/f_ncu1.log 2>&1; echo "launch=$?" >> $R/f_status.txt
timeout 600 python scripts/cfg_times.py > $R/f_cfgs.log 2>&1; echo "cfgs=$?" >> $R/f_status.txt
