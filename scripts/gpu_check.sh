cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?" > gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --maxfail=5 -k "not full_size" > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?" >> gpurun_out/status.txt
timeout 300 python bench.py --steps 3 --warmup 2 --log2n 26 --no-cpu-baseline --no-e2e > gpurun_out/bench26.log 2>&1; echo "bench26=$?" >> gpurun_out/status.txt
