# A/B of library variants (VARIANTS="A B", libvmps_<V>.so) on configs 1-4, the paper's 10^7 workload and the cfg5 bench
cd $GRAFT_REPO_ROOT
R=gpurun_out
: > $R/abc.log
for v in $VARIANTS; do
  echo -n "$v " >> $R/abc.log
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 600 python scripts/cfg_times.py 2>/dev/null | tail -1 >> $R/abc.log
  echo -n "$v " >> $R/abc.log
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg5_ms': round(d['ms_per_step'],2), 'plan': round(d['phases_ms']['plan_ms'],3), 'leaf': round(d['phases_ms']['leaf_ms'],2), 'ok': d['verified']}))" >> $R/abc.log
done
