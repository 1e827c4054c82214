cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_depth_parity.py tests/test_prefill_fusion.py -q -x -k "prefill or batched or fused" > gpurun_out/${T}_pf_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_pf_tests.log
for P in 10 100 500; do timeout 300 python tools/ttft_probe.py $P > gpurun_out/${T}_ttft$P.txt 2>&1; done
