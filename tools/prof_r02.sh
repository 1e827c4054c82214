# Round-2 profile set (one GPU, run via gpurun): launch lists and one full ncu
# capture per decode / prefill kernel of the current build, into gpurun_out/.
cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/r02p
# one full capture of each decode kernel (eager step API, 4 layers; skip layer 0)
for k in "gemv_pair_kernel:2" "gemv_kernel<__nv_bfloat16, 2, 3>:2" "gemv_kernel<__nv_bfloat16, 0, 1>:2" "attn_decode_kernel:2" "gemv_kernel<__nv_bfloat16, 2, 0>:2"; do
  name=${k%%:*}; skip=${k##*:}; tag=$(echo "$name" | tr -cd 'a-z0-9_')
  timeout 600 $NCU --set full --clock-control none --import-source on -k "regex:${name//</\\<}" --launch-skip $skip -c 1 -o ${O}_${tag} -f python tools/decode_prof.py 10 4 2 > ${O}_${tag}.log 2>&1
done
timeout 600 $NCU --set full --clock-control none -k regex:attn_decode --launch-skip 2 -c 1 -o ${O}_attn500 -f python tools/decode_prof.py 500 4 2 > ${O}_attn500.log 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:grt_sample --launch-skip 4 -c 1 -o ${O}_sampler_topp -f python tools/topp_prof.py topp > ${O}_sampler_topp_full.log 2>&1
