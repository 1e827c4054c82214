cd $GRAFT_REPO_ROOT
timeout 1200 bash tools/multi_ab.sh 2 "GRT_PAIR_L2PRE=0" "GRT_PAIR_L2PRE=1" "GRT_PAIR_L2PRE=2" > gpurun_out/ab18.txt 2>&1
