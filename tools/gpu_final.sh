cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo rc=$? >> gpurun_out/final_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
timeout 700 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo rc=$? >> gpurun_out/final_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-profile --sweep= --mixed 0 --ipc 0"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_launches.csv $B > gpurun_out/r01e_launches.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn_decode --launch-skip 100 -c 1 -o gpurun_out/r01e_attn -f $B > gpurun_out/r01e_attn.log 2>&1
