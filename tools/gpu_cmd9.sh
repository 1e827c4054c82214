cd $GRAFT_REPO_ROOT
timeout 1200 bash tools/multi_ab.sh 2 "GRT_DOWN_CHMAX=3072" "GRT_DOWN_CHMAX=1408" "GRT_DOWN_CHMAX=1856" "GRT_DOWN_CHMAX=1024" > gpurun_out/ab9.txt 2>&1
timeout 300 python tools/per_token.py hybrid > gpurun_out/per_token.txt 2>&1
