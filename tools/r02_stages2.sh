cd $GRAFT_REPO_ROOT
B="python bench.py --steps 64 --warmup 5 --no-cpu-baseline --sweep= --mixed 0 --ipc 0 --modes= --no-profile"
timeout 300 $B --pass-impl 1 > gpurun_out/r02st2_p1.json 2>> gpurun_out/r02st2.err
GRT_STREAM_CHMAX=4096 timeout 300 $B --pass-impl 2 > gpurun_out/r02st2_p2_c4096.json 2>> gpurun_out/r02st2.err
GRT_STREAM_CHMAX=4096 timeout 300 python tools/stream_trace.py > gpurun_out/r02st2_trace_c4096.json 2>> gpurun_out/r02st2.err
GRT_QKV_CHMAX=4096 timeout 300 $B --pass-impl 1 > gpurun_out/r02st2_p1_q4096.json 2>> gpurun_out/r02st2.err
GRT_WOUP_CHMAX=4096 timeout 300 $B --pass-impl 1 > gpurun_out/r02st2_p1_w4096.json 2>> gpurun_out/r02st2.err
