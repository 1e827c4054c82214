cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/r02p
# gemv_kernel launches of decode_prof (4 layers): 0 prefill head, then per step q0 d0 q1 d1 q2 d2 q3 d3 head
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_kernel --launch-skip 3 -c 2 -o ${O}_gemv_qkv_down -f python tools/decode_prof.py 10 4 2 > ${O}_gemv_qkv_down.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_kernel --launch-skip 9 -c 1 -o ${O}_gemv_head -f python tools/decode_prof.py 10 4 2 > ${O}_gemv_head.log 2>&1
