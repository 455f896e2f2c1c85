# A/B on configs + the paper workloads, then the GPU parity suites on variant B
cd $GRAFT_REPO_ROOT
VARIANTS="${VARIANTS:-A B B A}" bash scripts/gpu_ab_phases.sh
VMPS_LIB=$PWD/paper_2605_27147_b200/libvmps_B.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/abt.log 2>&1; echo "tests=$?" >> gpurun_out/abt.log
