cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_checkpoint.py tests/test_gpu_parity.py -m gpu -x -q -k "checkpoint or dump or strict or f16 or device_loop or ipc or all_modes" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$? secs=$(( $(date +%s) - s )) >> gpurun_out/bench3.err
