# GPU tests of the in-tree build, variants ($VARIANTS) on cfg1-4 + paper + cfg5 (phases) and the cfg5 bounded leg
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $R/abt_tests.log 2>&1; echo "tests=$?" > $R/abt_status.txt
bash scripts/gpu_ab_cfgs.sh
NO_NCU=1 bash scripts/gpu_m4_ab_ncu.sh
: > $R/bdab.log
for v in $VARIANTS; do
  echo -n "$v " >> $R/bdab.log
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 2 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); b=d['bounded']; print(json.dumps({'ms': round(d['ms_per_step'],2), 'bd_ms': round(b['ms_per_step'],1), 'x': round(b['slowdown_vs_unbounded'],3)}))" >> $R/bdab.log
done
