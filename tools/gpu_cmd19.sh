cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_paged_kv.py -m gpu -x -q -k "attention or long_context or paged or llama" > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
for c in 0 1 0 1; do GRT_ATTN_WAVE_CAP=$c timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-profile --sweep 10,200,500 --mixed 0 --ipc 0 > gpurun_out/sweep19_c$c.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/sweep19_c$c.json')); print($c, d['ttft_sweep'])" >> gpurun_out/sweep19.txt; done
