cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/check_tests.log 2>&1; echo rc=$? >> gpurun_out/check_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.log 2>&1; echo rc=$? >> gpurun_out/check_smoke.log
timeout 300 python bench.py --steps 128 --warmup 8 --no-cpu-baseline --sweep "" --mixed 0 --ipc 0 > gpurun_out/check_bench.json 2>/dev/null
