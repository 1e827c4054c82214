cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 300 python tools/ttft_probe.py 10 > gpurun_out/${T}_ttft10.txt 2>&1
timeout 300 python tools/ttft_probe.py 500 > gpurun_out/${T}_ttft500.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
