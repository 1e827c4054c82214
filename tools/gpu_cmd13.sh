cd $GRAFT_REPO_ROOT
for w in 2 3 4; do GRT_PG_WIDE_KSPLIT=$w timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-profile --sweep 300,400,500 --mixed 0 --ipc 0 > gpurun_out/sweep13_w$w.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/sweep13_w$w.json')); print($w, {k: v['ttft_ms'] for k, v in d['ttft_sweep'].items()})" >> gpurun_out/sweep13.txt; done
timeout 600 python -m pytest tests/test_prefill_fusion.py tests/test_gpu_parity.py -m gpu -x -q -k "fusion or batched or tp_batched" > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
