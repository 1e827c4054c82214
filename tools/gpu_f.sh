cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_depth_parity.py -q -x -k "prefill or batched" > gpurun_out/${T}_fa_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_fa_tests.log
timeout 300 python tools/ttft_probe.py 500 > gpurun_out/${T}_ttft500.txt 2>&1
timeout 300 python tools/ttft_probe.py 300 > gpurun_out/${T}_ttft300.txt 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill|gemv" --csv --log-file gpurun_out/${T}_pf500.csv python tools/prefill_prof.py 500 4 1 > gpurun_out/${T}_pf500.log 2>&1
