# Round-2 profile set (one GPU; run via gpurun, outputs in gpurun_out/r02p_*):
# launch lists of a decode token / a batched prefill / the sampler, and one
# full ncu capture per decode and prefill kernel.  Summaries: tools/launch_summary.py,
# tools/ncu_summary.py -> profiles/r02_*.txt.
cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/r02p
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-profile --sweep= --mixed 0 --ipc 0 --modes="
# launch lists (gpu__time_duration only): decode at P=10 / P=500, prefill at P=10 / P=500, sampler
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_decode10_launches.csv $B > ${O}_l10.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_decode500_launches.csv python tools/decode_prof.py 500 32 2 > ${O}_l500.log 2>&1  # eager steps: bench.py at P=500 outruns the timeout under ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_prefill500_launches.csv python tools/prefill_prof.py 500 32 1 > ${O}_lp500.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_prefill10_launches.csv python tools/prefill_prof.py 10 32 1 > ${O}_lp10.log 2>&1
for k in topp topk greedy; do
  timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:grt_sample --csv --log-file ${O}_sampler_$k.csv python tools/topp_prof.py $k > ${O}_s_$k.log 2>&1
done
# full captures (eager step API of tools/decode_prof.py, 4 layers; launch indices skip layer 0)
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_pair --launch-skip 2 -c 1 -o ${O}_gemv_pair_kernel -f python tools/decode_prof.py 10 4 2 > ${O}_pair.log 2>&1
# gemv_kernel launches: 0 prefill head, then per step q0 d0 q1 d1 q2 d2 q3 d3 head
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_kernel --launch-skip 3 -c 2 -o ${O}_gemv_qkv_down -f python tools/decode_prof.py 10 4 2 > ${O}_gemv_qkv_down.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_kernel --launch-skip 9 -c 1 -o ${O}_gemv_head -f python tools/decode_prof.py 10 4 2 > ${O}_gemv_head.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_decode --launch-skip 2 -c 1 -o ${O}_attn_decode_kernel -f python tools/decode_prof.py 10 4 2 > ${O}_attn10.log 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:attn_decode --launch-skip 2 -c 1 -o ${O}_attn500 -f python tools/decode_prof.py 500 4 2 > ${O}_attn500.log 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:grt_sample --launch-skip 4 -c 1 -o ${O}_sampler_topp -f python tools/topp_prof.py topp > ${O}_sampler_topp_full.log 2>&1
# batched prefill P=500 (4 layers): the four GEMMs of layer 1 and one flash-attention launch
timeout 600 $NCU --set full --clock-control none -k regex:prefill_gemm --launch-skip 4 -c 4 -o ${O}_pfgemm500 -f python tools/prefill_prof.py 500 4 1 > ${O}_pfgemm500.log 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:prefill_fa_tc --launch-skip 1 -c 1 --import-source on -o ${O}_pffa500 -f python tools/prefill_prof.py 500 4 1 > ${O}_pffa500.log 2>&1
