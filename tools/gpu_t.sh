cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 600 python -m pytest tests/test_nccl_tp.py tests/test_capture_contract.py -q -x > gpurun_out/${T}_nccl.log 2>&1; echo rc=$? >> gpurun_out/${T}_nccl.log
