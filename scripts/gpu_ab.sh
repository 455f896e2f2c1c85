# tests + A/B bench lines (radix leaf vs merge leaf, Z variants)
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $R/q_tests.log 2>&1; echo "tests=$?" > $R/q_status.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
timeout 300 $B > $R/ab_radix.log 2>&1; echo "radix=$?" >> $R/q_status.txt
timeout 300 $B --leaf-merge > $R/ab_merge.log 2>&1; echo "merge=$?" >> $R/q_status.txt
timeout 300 $B --fuse-z 1024 > $R/ab_z1024.log 2>&1; echo "z1024=$?" >> $R/q_status.txt
