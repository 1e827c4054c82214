# Round-1 profiling pass (run under gpurun): launch list of the bench command,
# full ncu captures of the decode GEMVs / attention and of the prefill kernels.
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-profile --sweep= --mixed 0 --ipc 0"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $B > gpurun_out/r01_launches.log 2>&1; echo launches $?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv --launch-skip 400 -c 5 -o gpurun_out/r01_gemv -f $B > gpurun_out/r01_gemv.log 2>&1; echo gemv $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:attn_decode --launch-skip 100 -c 1 -o gpurun_out/r01_attn -f $B > gpurun_out/r01_attn.log 2>&1; echo attn $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:prefill_gemm -c 4 -o gpurun_out/r01_pfgemm500 -f python tools/prefill_prof.py 500 1 1 > gpurun_out/r01_pf.log 2>&1; echo pfgemm $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:prefill_gemm -c 4 -o gpurun_out/r01_pfgemm10 -f python tools/prefill_prof.py 10 1 1 >> gpurun_out/r01_pf.log 2>&1; echo pfgemm10 $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:prefill_attn -c 1 -o gpurun_out/r01_pfattn -f python tools/prefill_prof.py 500 1 1 >> gpurun_out/r01_pf.log 2>&1; echo pfattn $?
timeout 300 python tools/op_trace.py 32 80 > gpurun_out/r01_op_trace.txt 2>&1; echo trace $?
