# bash tools/multi_ab.sh REPS "ENV=a ENV2=b" "ENV=c" ...  -> p50 ms/token per config, reps interleaved
REPS=$1; shift
declare -A vals
for i in $(seq $REPS); do
  for cfg in "$@"; do
    env $cfg timeout 120 python bench.py --steps 128 --warmup 8 --no-cpu-baseline --no-profile --sweep "" --mixed 0 --ipc 0 > gpurun_out/ab.json 2>gpurun_out/ab.err
    v=$(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'], d['p99_ms'])" 2>/dev/null || echo FAIL)
    vals[$cfg]="${vals[$cfg]} | $v"
  done
done
for cfg in "$@"; do echo "$cfg:${vals[$cfg]}"; done
