cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_stream_pass.py tests/test_capture_contract.py -q -x > gpurun_out/r02s1_tests.log 2>&1; echo rc=$? >> gpurun_out/r02s1_tests.log
timeout 300 python tools/stream_trace.py > gpurun_out/r02s1_trace.json 2> gpurun_out/r02s1_trace.err
B="python bench.py --steps 64 --warmup 5 --no-cpu-baseline --sweep= --mixed 0 --ipc 0 --modes= --no-profile"
for i in 1 2; do
  timeout 300 $B --pass-impl 1 > gpurun_out/r02s1_b1_$i.json 2>> gpurun_out/r02s1_b.err
  timeout 300 $B --pass-impl 2 > gpurun_out/r02s1_b2_$i.json 2>> gpurun_out/r02s1_b.err
done
for c in 1024 2048; do
  GRT_STREAM_CHMAX=$c timeout 300 $B --pass-impl 2 > gpurun_out/r02s1_b2_ch$c.json 2>> gpurun_out/r02s1_b.err
done
