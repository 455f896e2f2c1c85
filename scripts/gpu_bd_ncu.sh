# bounded one-piece cfg5 2^28: launch list + a full capture of a large k_bd_level launch
cd $GRAFT_REPO_ROOT
R=gpurun_out
export LOG2N=28 VMPS_BD_CELL=1073741824


timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"^k_bd_level$" -s 8 -c 1 -o $R/bdn_level_full python scripts/bd_one.py > $R/bdn_ncu2.log 2>&1; echo "full=$?" >> $R/bdn_status.txt
