cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_tests.log
timeout 700 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo rc=$? >> gpurun_out/r02_bench.err
