# One GPU pass of the round: the -m gpu suite, smoke(), the default bench line
# and the reference arm (run from the repo root on the GPU box via gpurun).
#   gpurun --timeout 3600 -- 'bash tools/gpu_round.sh TAG'
cd "$GRAFT_REPO_ROOT"
T=${1:-run}
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo rc=$? >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
timeout 900 python bench.py --steps 20 --warmup 5 --trials 100 --mixed 0 --ipc 0 --modes= --no-cpu-baseline > gpurun_out/${T}_sweep100.json 2> gpurun_out/${T}_sweep100.err
