cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_depth_parity.py -q -x -k "gemv or llama or full_depth or device_loop or tp_ or all_modes" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
B="python bench.py --steps 64 --warmup 5 --no-cpu-baseline --sweep= --mixed 0 --ipc 0 --modes="
for i in 1 2; do timeout 300 $B > gpurun_out/${T}_b_$i.json 2>> gpurun_out/${T}_b.err; done
timeout 300 $B --prompt-len 500 > gpurun_out/${T}_b500.json 2>> gpurun_out/${T}_b.err
