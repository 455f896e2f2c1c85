cd $GRAFT_REPO_ROOT
R=gpurun_out
VMPS_DEBUG_SYNC=1 timeout 300 python scripts/repro_tiny.py > $R/d_rep.log 2>&1; echo "rep=$?" > $R/d_status.txt
