cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checkpoint.py -m gpu -x -q > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log
timeout 900 bash tools/multi_ab.sh 3 "GRT_PAIR_ATTN=0" "GRT_PAIR_ATTN=1" > gpurun_out/ab4.txt 2>&1
