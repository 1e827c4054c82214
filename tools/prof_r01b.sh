# Round-1 profiling refresh (run under gpurun): decode launch list of the bench
# command, a full capture of the dominant decode kernel (fused Wo + gate/up) and
# of the QKV GEMV, and the launch list of one batched prefill at P=10 / P=500
# (32 layers: the TTFT breakdown).
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-profile --sweep= --mixed 0 --ipc 0"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_launches.csv $B > gpurun_out/r01b_launches.log 2>&1; echo launches $?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_pair --launch-skip 200 -c 2 -o gpurun_out/r01b_pair -f $B > gpurun_out/r01b_pair.log 2>&1; echo pair $?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"gemv_kernel" --launch-skip 300 -c 3 -o gpurun_out/r01b_gemv -f $B > gpurun_out/r01b_gemv.log 2>&1; echo gemv $?
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r01b_prefill10.csv python tools/prefill_prof.py 10 32 2 > gpurun_out/r01b_pf10.log 2>&1; echo pf10 $?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_prefill500.csv python tools/prefill_prof.py 500 32 2 > gpurun_out/r01b_pf500.log 2>&1; echo pf500 $?
