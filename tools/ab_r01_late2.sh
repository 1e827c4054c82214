cd $GRAFT_REPO_ROOT
timeout 1500 bash tools/multi_ab.sh 2 "GRT_X=0" "GRT_QKV_CHMAX=1024" "GRT_QKV_CHMAX=4096" "GRT_WOUP_CHMAX=1024" "GRT_WOUP_CHMAX=4096" > gpurun_out/ab_late2.txt 2>&1
