cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_paged_kv.py tests/test_gpu_parity.py -m gpu -x -q -k "paged or fused or llama or attention or device_loop or batched or tp_" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
timeout 600 bash tools/multi_ab.sh 2 "GRT_X=0" > gpurun_out/ab6.txt 2>&1
