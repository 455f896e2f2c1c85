# library variants on the cfg5 bench ($VARIANTS, libvmps_<V>.so), then --set full of one large k4_merge_level launch of the in-tree build
cd $GRAFT_REPO_ROOT
R=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bounded-reps 0"
: > $R/m4v.log
for it in 1 2; do for v in $VARIANTS; do
  echo -n "$v " >> $R/m4v.log
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 300 $B 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'ms': round(d['ms_per_step'],2), **{k: round(v,2) for k,v in d['phases_ms'].items()}, 'ok': d['verified']}))" >> $R/m4v.log
done; done
[ -n "$NO_NCU" ] || bash scripts/gpu_merge_ncu.sh
