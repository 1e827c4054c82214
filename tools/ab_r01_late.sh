cd $GRAFT_REPO_ROOT
timeout 1500 bash tools/multi_ab.sh 2 "GRT_ATTN_TRIGGER=0" "GRT_ATTN_TRIGGER=1" "GRT_ATTN_TRIGGER=2" "GRT_ATTN_PREFETCH=1 GRT_ATTN_ROUNDS=2" > gpurun_out/ab_late.txt 2>&1
