# End-of-round refresh: round check, ncu evidence, per-config phases, paper sweep.
cd $GRAFT_REPO_ROOT
bash scripts/gpu_round.sh
bash scripts/gpu_evidence.sh
python scripts/cfg_phases.py > gpurun_out/cfg_phases.log 2>&1
python scripts/cfg_times.py > gpurun_out/cfg_times.log 2>&1
timeout 900 python scripts/paper_sweep.py gpurun_out/paper_sweep.jsonl > gpurun_out/sweep.log 2>&1
