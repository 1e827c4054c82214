cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_paged_kv.py -m gpu -x -q -k "attention or long_context or paged or llama or device_loop or modes" > gpurun_out/t21.log 2>&1; echo rc=$? >> gpurun_out/t21.log
timeout 900 bash tools/multi_ab.sh 3 "GRT_ATTN_PREFETCH=0" "GRT_ATTN_PREFETCH=1" > gpurun_out/ab21.txt 2>&1
