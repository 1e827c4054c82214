# A/B of two source trees on the same box: bash tools/ab_builds.sh REPS DIR_A DIR_B
REPS=$1; A=$2; B=$3
for i in $(seq $REPS); do
  for d in $A $B; do
    (cd $d && timeout 120 python bench.py --steps 128 --warmup 8 --no-cpu-baseline --no-profile --sweep "" --mixed 0 --ipc 0 > /tmp/abb.json 2>/tmp/abb.err)
    echo "$d: $(python -c "import json;d=json.load(open('/tmp/abb.json'));print(d['value'], d['p99_ms'])" 2>/dev/null || tail -2 /tmp/abb.err)"
  done
done
