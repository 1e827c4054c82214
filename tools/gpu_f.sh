cd "$GRAFT_REPO_ROOT"
T=${1:-run}


for P in 200 300 500; do timeout 300 python tools/ttft_probe.py $P > gpurun_out/${T}_ttft$P.txt 2>&1; done
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill|gemv" --csv --log-file gpurun_out/${T}_pf500.csv python tools/prefill_prof.py 500 4 1 > gpurun_out/${T}_pf500.log 2>&1
