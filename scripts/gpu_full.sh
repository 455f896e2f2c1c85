cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k full_size > gpurun_out/gpu_full.log 2>&1; echo "full=$?" > gpurun_out/status2.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench30.log 2>&1; echo "bench30=$?" >> gpurun_out/status2.txt
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain30.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches30.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1=$?" >> gpurun_out/status2.txt
timeout 300 python bench.py --steps 1 --warmup 1 --log2n 26 --no-e2e --no-cpu-baseline > gpurun_out/plain26.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_level|k_leaf_sort|k_runs_tables|k_runs_emit" -s 40 -c 6 -o gpurun_out/prof26 python bench.py --steps 1 --warmup 1 --log2n 26 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu2=$?" >> gpurun_out/status2.txt
