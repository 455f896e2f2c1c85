# GPU parity tests of the in-tree library, then variants (libvmps_<V>.so, $VARIANTS) on cfg1-4, the paper's workload and cfg5
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $R/abt_tests.log 2>&1; echo "tests=$?" > $R/abt_status.txt
bash scripts/gpu_ab_cfgs.sh
