# A/B of libvmps builds on the cfg5 bench: $AB_LIBS = space-separated .so paths
# (relative to the repo; "cur" = the in-tree library), two alternating passes
cd $GRAFT_REPO_ROOT
R=gpurun_out
: > $R/ab_summary.txt
for pass in 1 2; do
  for L in $AB_LIBS; do
    if [ "$L" = cur ]; then unset VMPS_LIB; else export VMPS_LIB=$GRAFT_REPO_ROOT/$L; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0 $AB_ARGS > $R/ab_tmp.log 2>&1
    python - "$L" "$pass" >> $R/ab_summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab_tmp.log").read().strip().splitlines()[-1])
    ph = d["phases_ms"]
    print(sys.argv[1], "pass", sys.argv[2], "ms %.2f" % d["ms_per_step"], " ".join("%s %.2f" % (k, v) for k, v in ph.items()), "ok" if d["verified"] else "NOT VERIFIED")
except Exception as e:
    print(sys.argv[1], "pass", sys.argv[2], "failed", e, open("gpurun_out/ab_tmp.log").read()[-400:])
PY
  done
done
