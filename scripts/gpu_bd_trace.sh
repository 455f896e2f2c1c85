# bounded cfg5 2^30: phase trace of the dyadic-cell mode (host wall per phase) + one-piece
cd $GRAFT_REPO_ROOT
R=gpurun_out
VMPS_BD_TRACE=1 timeout 600 python scripts/bd_probe.py ${LG:-30} 1 > $R/bdt.log 2>&1; echo "rc=$?" >> $R/bdt.log
