cd $GRAFT_REPO_ROOT
bash tools/ab_builds.sh 3 ab_old . > gpurun_out/ab7.txt 2>&1
timeout 300 python -m pytest tests/test_paged_kv.py tests/test_gpu_parity.py -m gpu -x -q -k "paged or fused or attention" > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
