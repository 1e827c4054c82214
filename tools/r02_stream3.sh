cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_stream_pass.py tests/test_capture_contract.py -q -x > gpurun_out/r02s3_tests.log 2>&1; echo rc=$? >> gpurun_out/r02s3_tests.log
timeout 300 python tools/stream_trace.py > gpurun_out/r02s3_trace.json 2> gpurun_out/r02s3_trace.err
B="python bench.py --steps 64 --warmup 5 --no-cpu-baseline --sweep= --mixed 0 --ipc 0 --modes= --no-profile"
timeout 300 $B --pass-impl 1 > gpurun_out/r02s3_b1.json 2>> gpurun_out/r02s3_b.err
for a in 0 4 8 12; do for b in 0 2 4; do
  GRT_STREAM_PF_ATT=$a GRT_STREAM_PF_BAR=$b timeout 300 $B --pass-impl 2 > gpurun_out/r02s3_b2_${a}_${b}.json 2>> gpurun_out/r02s3_b.err
done; done
GRT_STREAM_PF_ATT=8 GRT_STREAM_PF_BAR=2 timeout 300 python tools/stream_trace.py > gpurun_out/r02s3_trace82.json 2>> gpurun_out/r02s3_trace.err
