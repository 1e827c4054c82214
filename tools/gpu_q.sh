cd "$GRAFT_REPO_ROOT"
T=${1:-run}
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --section SourceCounters --section WarpStateStats --section SpeedOfLight --import-source on -k regex:grt_sample --launch-skip 4 -c 1 -o gpurun_out/${T}_samp_topp -f python tools/topp_prof.py topp > gpurun_out/${T}_ncu.log 2>&1
