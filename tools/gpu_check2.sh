cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/check2_tests.log 2>&1; echo rc=$? >> gpurun_out/check2_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check2_smoke.log 2>&1; echo rc=$? >> gpurun_out/check2_smoke.log
timeout 900 bash tools/ab_builds.sh 2 ab_prev . > gpurun_out/check2_ab.txt 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file gpurun_out/check2_samp.csv python tools/topp_prof.py greedy > /dev/null 2>&1
