NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_impl1.csv -c 3000 $B --pass-impl 1 > gpurun_out/ncu_b1.log 2>&1; echo l1 $?
timeout 300 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_impl0.csv -c 400 $B --pass-impl 0 > gpurun_out/ncu_b0.log 2>&1; echo l0 $?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_kernel --launch-skip 1600 -c 5 -o gpurun_out/gemv_full -f $B --pass-impl 1 > gpurun_out/ncu_f1.log 2>&1; echo f1 $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:attn_decode --launch-skip 300 -c 1 -o gpurun_out/attn_full -f $B --pass-impl 1 > gpurun_out/ncu_f2.log 2>&1; echo f2 $?
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:decode_pass --launch-skip 12 -c 1 -o gpurun_out/pass_full -f $B --pass-impl 0 > gpurun_out/ncu_f3.log 2>&1; echo f3 $?
