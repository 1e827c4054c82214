cd $GRAFT_REPO_ROOT
B="python bench.py --steps 64 --warmup 5 --no-cpu-baseline --sweep= --mixed 0 --ipc 0 --modes= --no-profile"
timeout 300 $B --pass-impl 1 > gpurun_out/r02st_p1.json 2>> gpurun_out/r02st.err
GRT_GEMV_STAGES=2 timeout 300 $B --pass-impl 1 > gpurun_out/r02st_p1_g2.json 2>> gpurun_out/r02st.err
GRT_GEMV_STAGES=2 GRT_PAIR_STAGES=2 timeout 300 $B --pass-impl 1 > gpurun_out/r02st_p1_g2p2.json 2>> gpurun_out/r02st.err
GRT_PAIR_STAGES=2 timeout 300 $B --pass-impl 1 > gpurun_out/r02st_p1_p2.json 2>> gpurun_out/r02st.err
GRT_STREAM_STAGES=2 timeout 300 $B --pass-impl 2 > gpurun_out/r02st_p2_s2.json 2>> gpurun_out/r02st.err
GRT_STREAM_STAGES=2 timeout 300 python tools/stream_trace.py > gpurun_out/r02st_trace_s2.json 2>> gpurun_out/r02st.err
GRT_STREAM_STAGES=2 GRT_STREAM_CHMAX=1024 timeout 300 $B --pass-impl 2 > gpurun_out/r02st_p2_s2c1024.json 2>> gpurun_out/r02st.err
GRT_STREAM_STAGES=4 GRT_STREAM_CHMAX=1024 timeout 300 $B --pass-impl 2 > gpurun_out/r02st_p2_s4c1024.json 2>> gpurun_out/r02st.err
timeout 300 $B --pass-impl 2 > gpurun_out/r02st_p2_s3.json 2>> gpurun_out/r02st.err
