# usage: KREGEX=... SKIP=... COUNT=... LOG2N=... bash scripts/gpu_prof_one.sh
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 1 --warmup 1 --log2n ${LOG2N:-26} --no-e2e --no-cpu-baseline"
timeout 300 $B > $R/po_plain.log 2>&1 && \
 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${SKIP:-1} -c ${COUNT:-1} -o $R/${OUT:-prof_one} $B > $R/po_ncu.log 2>&1; echo "ncu=$?" > $R/po_status.txt
