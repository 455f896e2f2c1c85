# bounded mode: GPU parity tests + cfg5 2^30 timings (cells, one piece) with the phase trace
cd $GRAFT_REPO_ROOT
R=gpurun_out
timeout 900 python -m pytest tests/test_gpu_bounded.py tests/test_gpu_comm.py -q -x > $R/bdc_tests.log 2>&1; echo "tests=$?" > $R/bdc_status.txt
VMPS_BD_TRACE=1 timeout 600 python scripts/bd_probe.py 30 1 > $R/bdc_trace.log 2>&1; echo "trace=$?" >> $R/bdc_status.txt
CHUNKS=${CHUNKS:-23,31} timeout 900 python scripts/bd_cells_probe.py > $R/bdc_cells.log 2>&1; echo "cells=$?" >> $R/bdc_status.txt
