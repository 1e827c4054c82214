cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sampler" --durations=5 > gpurun_out/${T}_samp_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_samp_tests.log
NCU=/usr/local/cuda/bin/ncu
for k in topp topk greedy; do
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file gpurun_out/${T}_samp_$k.csv python tools/topp_prof.py $k > gpurun_out/${T}_samp_$k.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
