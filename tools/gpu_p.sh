cd "$GRAFT_REPO_ROOT"
T=${1:-run}
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sampler or topp or temperature" > gpurun_out/${T}_samp_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_samp_tests.log
for k in topp topk greedy; do
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file gpurun_out/${T}_samp_$k.csv python tools/topp_prof.py $k > gpurun_out/${T}_samp_$k.log 2>&1
done

