cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 600 python -m pytest tests/test_nccl_tp.py -q -x > gpurun_out/${T}_nccl.log 2>&1; echo rc=$? >> gpurun_out/${T}_nccl.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
