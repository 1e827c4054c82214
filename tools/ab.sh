# A/B helper: bash tools/ab.sh "ENV=a" "ENV=b" [reps]  -> p50 ms/token per run
REPS=${3:-3}
for cfg in "$1" "$2"; do
  vals=""
  for i in $(seq $REPS); do
    env $cfg timeout 120 python bench.py --steps 128 --warmup 8 --no-cpu-baseline --no-profile --sweep "" --mixed 0 --ipc 0 > gpurun_out/ab.json 2>/dev/null
    vals="$vals $(python -c "import json;print(json.load(open('gpurun_out/ab.json'))['value'])")"
  done
  echo "$cfg:$vals"
done
