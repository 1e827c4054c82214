NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-profile --sweep= --mixed 0 --ipc 0"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $B > gpurun_out/r01_launches.log 2>&1; echo launches $?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv --launch-skip 400 -c 5 -o gpurun_out/r01_gemv -f $B > gpurun_out/r01_gemv.log 2>&1; echo gemv $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:attn_decode --launch-skip 100 -c 1 -o gpurun_out/r01_attn -f $B > gpurun_out/r01_attn.log 2>&1; echo attn $?
