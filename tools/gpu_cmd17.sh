cd $GRAFT_REPO_ROOT
timeout 1200 bash tools/multi_ab.sh 2 "GRT_GEMV_L2PRE=0" "GRT_GEMV_L2PRE=1" "GRT_GEMV_L2PRE=2" "GRT_GEMV_L2PRE=4" > gpurun_out/ab17.txt 2>&1
timeout 600 python -m pytest tests/test_paged_kv.py -m gpu -x -q > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
