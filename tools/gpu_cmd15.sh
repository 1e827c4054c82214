cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_paged_kv.py -m gpu -x -q -k "attention or llama or device_loop or paged or long_context or tiny or modes" > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
timeout 900 bash tools/multi_ab.sh 3 "GRT_ATTN_PREFETCH=0" "GRT_ATTN_PREFETCH=1" > gpurun_out/ab15.txt 2>&1
for f in 0 1; do GRT_ATTN_PREFETCH=$f timeout 300 python tools/per_token.py hybrid > gpurun_out/per_token15_$f.txt 2>&1; done
