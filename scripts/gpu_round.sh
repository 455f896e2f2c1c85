# Full round check: GPU tests, smoke, default bench, reference arm.
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $R/r_tests.log 2>&1; echo "tests=$?" > $R/r_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/r_smoke.log 2>&1; echo "smoke=$?" >> $R/r_status.txt
timeout 900 python bench.py > $R/r_bench.log 2>&1; echo "bench=$?" >> $R/r_status.txt
timeout 600 python bench.py --impl reference > $R/r_ref.log 2>&1; echo "ref=$?" >> $R/r_status.txt
