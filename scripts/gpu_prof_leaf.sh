cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --maxfail=3 -k "not full_size" > $R/it_tests.log 2>&1; echo "tests=$?" > $R/it_status.txt
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $R/it_bench30.log 2>&1; echo "bench30=$?" >> $R/it_status.txt
B26="python bench.py --steps 1 --warmup 1 --log2n 26 --no-e2e --no-cpu-baseline"
timeout 300 $B26 > $R/it_plain26.log 2>&1 && \
 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_tile_desc" -s 20 -c 12 -o $R/prof_leaf $B26 > $R/it_ncu_leaf.log 2>&1; echo "ncu=$?" >> $R/it_status.txt
