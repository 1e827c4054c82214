cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/last_tests.log 2>&1; echo rc=$? >> gpurun_out/last_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo rc=$? >> gpurun_out/last_smoke.log
timeout 600 python bench.py > gpurun_out/last_bench2.json 2> gpurun_out/last_bench2.err
