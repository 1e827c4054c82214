cd $GRAFT_REPO_ROOT
timeout 900 bash tools/multi_ab.sh 2 "GRT_ATTN_ROUNDS=1" "GRT_ATTN_ROUNDS=2" > gpurun_out/ab20.txt 2>&1
for r in 1 2; do GRT_ATTN_ROUNDS=$r timeout 300 python tools/per_token.py hybrid > gpurun_out/per_token20_$r.txt 2>&1; done
