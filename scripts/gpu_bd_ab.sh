# bounded-mode leg of the cfg5 bench for library variants ($VARIANTS): ms, slowdown, peak extra bytes
cd $GRAFT_REPO_ROOT
R=gpurun_out
: > $R/bdab.log
for it in 1 2; do for v in $VARIANTS; do
  echo -n "$v " >> $R/bdab.log
  VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_$v.so timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --bounded-reps 2 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); b=d['bounded']; print(json.dumps({'ms': round(d['ms_per_step'],2), 'bd_ms': round(b['ms_per_step'],1), 'x': round(b['slowdown_vs_unbounded'],3), 'peakMB': b['peak_extra_device_bytes']/1e6, 'metaMB': b['metadata_bytes']/1e6}))" >> $R/bdab.log
done; done
