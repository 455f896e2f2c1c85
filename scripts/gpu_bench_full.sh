cd $GRAFT_REPO_ROOT
R=gpurun_out
S=$(date +%s); timeout 900 python bench.py > $R/bf_bench.log 2> $R/bf_err.log; echo "bench=$? secs=$(( $(date +%s) - S ))" > $R/bf_status.txt
