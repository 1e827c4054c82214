cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r02c1_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r02c1_host.txt; free -g >> gpurun_out/r02c1_host.txt
timeout 900 python -m pytest tests/test_capture_contract.py tests/test_gpu_parity.py -q -x -k "capture or c9 or c10 or replay or attention or foreign or dynamic or empty or open" > gpurun_out/r02c1_tests.log 2>&1; echo rc=$? >> gpurun_out/r02c1_tests.log
timeout 1200 python -m pytest tests/test_full_depth_parity.py -q -x --durations=0 > gpurun_out/r02c1_full.log 2>&1; echo rc=$? >> gpurun_out/r02c1_full.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c1_bench.json 2> gpurun_out/r02c1_bench.err; echo rc=$? >> gpurun_out/r02c1_bench.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r02c1_ref.json 2> gpurun_out/r02c1_ref.err
