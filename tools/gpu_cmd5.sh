cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "device_loop or llama or persistent or batched_prefill_matches" > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
timeout 900 bash tools/multi_ab.sh 2 "GRT_PAIR_ATTN=0" "GRT_PAIR_ATTN=1" "GRT_PAIR_ATTN=1 GRT_PAIR_ATTN_NS=1" "GRT_PAIR_ATTN=1 GRT_PAIR_ATTN_NS=2" > gpurun_out/ab5.txt 2>&1
