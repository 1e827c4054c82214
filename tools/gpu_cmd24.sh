cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sampler or temperature or ipc or device_loop or modes" > gpurun_out/t25.log 2>&1; echo rc=$? >> gpurun_out/t25.log
for k in greedy topp topk; do timeout 120 python tools/topp_prof.py $k >> gpurun_out/samp_times25.txt 2>&1; done
NCU=/usr/local/cuda/bin/ncu
for k in greedy topp; do timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file gpurun_out/samp25_$k.csv python tools/topp_prof.py $k > /dev/null 2>&1; done
