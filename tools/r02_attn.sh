cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "attention or long_context or llama_7b or device_loop" > gpurun_out/r02at_tests.log 2>&1; echo rc=$? >> gpurun_out/r02at_tests.log
B="python bench.py --steps 64 --warmup 5 --no-cpu-baseline --sweep= --mixed 0 --ipc 0 --modes= --no-profile"
for i in 1 2 3; do timeout 300 $B > gpurun_out/r02at_b_$i.json 2>> gpurun_out/r02at.err; done
timeout 300 $B --prompt-len 500 > gpurun_out/r02at_b500.json 2>> gpurun_out/r02at.err
timeout 300 $B --prompt-len 200 > gpurun_out/r02at_b200.json 2>> gpurun_out/r02at.err
