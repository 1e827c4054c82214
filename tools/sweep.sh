# usage: bash tools/sweep.sh VAR "v1 v2 ..." [bench args]  -> gpurun_out/sweep_VAR_v.json
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 64 --warmup 8 --no-cpu-baseline "$@" > gpurun_out/sweep_${VAR}_$v.json 2> gpurun_out/sweep_${VAR}_$v.err
  python -c "import json;d=json.load(open('gpurun_out/sweep_${VAR}_$v.json'));print('$VAR=$v', d['value'], d['p99_ms'], d['decode_hbm_gbs'], {k:v['ms_per_step_isolated'] for k,v in (d['kernels'] or {}).items()})" || tail -3 gpurun_out/sweep_${VAR}_$v.err
done
