cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
for k in greedy topp topk; do timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file gpurun_out/samp_$k.csv python tools/topp_prof.py $k > gpurun_out/samp_$k.log 2>&1; done
for k in greedy topp topk; do timeout 120 python tools/topp_prof.py $k >> gpurun_out/samp_times.txt 2>&1; done
