cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "prefill_gemm_tcgen05" > gpurun_out/${T}_gemm.log 2>&1; echo rc=$? >> gpurun_out/${T}_gemm.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_depth_parity.py tests/test_prefill_fusion.py tests/test_paged_kv.py -q -x -k "prefill or batched or fused or paged or tp_" > gpurun_out/${T}_pf_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_pf_tests.log
for P in 200 300 500; do timeout 300 python tools/ttft_probe.py $P > gpurun_out/${T}_ttft$P.txt 2>&1; done
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill|gemv" --csv --log-file gpurun_out/${T}_pf500.csv python tools/prefill_prof.py 500 4 1 > gpurun_out/${T}_pf500.log 2>&1
