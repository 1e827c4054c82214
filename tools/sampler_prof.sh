cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sampler or device_loop_temperature" > gpurun_out/t28.log 2>&1; echo rc=$? >> gpurun_out/t28.log
for k in greedy topp topk; do timeout 120 python tools/topp_prof.py $k >> gpurun_out/samp_times28.txt 2>&1; done
NCU=/usr/local/cuda/bin/ncu
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file gpurun_out/samp28_topp.csv python tools/topp_prof.py topp > /dev/null 2>&1
