cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_checkpoint.py tests/test_gpu_parity.py -m gpu -x -q -k "checkpoint or dump or strict or f16 or device_loop or ipc" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
/usr/bin/time -v timeout 700 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$? >> gpurun_out/bench2.err
timeout 900 bash tools/multi_ab.sh 2 "GRT_GEMV_PAIR=2" "GRT_GEMV_PAIR=1" "GRT_GEMV_PAIR=1 GRT_PAIR_CHMAX_A=1408 GRT_PAIR_CHMAX_B=1024" "GRT_GEMV_PAIR=1 GRT_PAIR_CHMAX_A=2048 GRT_PAIR_CHMAX_B=1024" > gpurun_out/ab2.txt 2>&1
timeout 300 python bench.py --mode device_loop --no-cpu-baseline --no-profile --sweep "" --mixed 0 --ipc 0 > gpurun_out/bench_dl.json 2> gpurun_out/bench_dl.err
