cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_prefill_fusion.py tests/test_gpu_parity.py -m gpu -x -q -k "fusion or batched or llama or tp_batched" > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
for r in 1 2; do GRT_ATTN_ROUNDS=$r timeout 300 python tools/per_token.py hybrid > gpurun_out/per_token_r$r.txt 2>&1; done
timeout 600 bash tools/multi_ab.sh 2 "GRT_ATTN_ROUNDS=2" "GRT_ATTN_ROUNDS=1" > gpurun_out/ab10.txt 2>&1
for f in 0 1; do GRT_PREFILL_FUSE_NORM=$f timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-profile --sweep 10,50,100,200,500 --mixed 0 --ipc 0 > gpurun_out/sweep_fuse$f.json 2>/dev/null; done
