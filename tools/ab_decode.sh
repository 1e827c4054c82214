# Same-box A/B of library variants (tools/_ab/NAME/libgraphrt_b200.so, built by
# `python -m paper_2604_23467_b200.build NAME DEFINE...`; "base" = the in-tree build).
#   gpurun -- 'bash tools/ab_decode.sh TAG base if2 if1'
# Prints per variant and repetition: decode p50 ms/token at P=10, the P=500 sweep cell.
cd "$GRAFT_REPO_ROOT"
T=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then L=""; else L="$PWD/tools/_ab/$v/libgraphrt_b200.so"; fi
    GRT_LIB_PATH=$L timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline \
      --sweep 10,500 --trials 3 --modes= --mixed 0 --ipc 0 > gpurun_out/${T}_${v}_${rep}.json 2> gpurun_out/${T}_${v}_${rep}.err
    python - "$T" "$v" "$rep" <<'PY'
import json, sys
T, v, rep = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/{T}_{v}_{rep}.json").read().strip().splitlines()[-1])
    sw = d.get("ttft_sweep", {})
    print(f"{v:10s} rep{rep} p50 {d['value']:.4f}  P10 ttft {sw['10']['ttft_mean_ms']:.3f} p50 {sw['10']['p50_ms']:.4f}  "
          f"P500 ttft {sw['500']['ttft_mean_ms']:.3f} p50 {sw['500']['p50_ms']:.4f}  qkv {d['kernels']['qkv']['gbs']:.0f} "
          f"pair {d['kernels']['wo_residual+gate_up_swiglu']['gbs']:.0f} down {d['kernels']['down_residual']['gbs']:.0f}", flush=True)
except Exception as e:
    print(v, rep, "FAILED", e)
PY
  done
done
# parity of each variant on the GEMV / full-model tests
for v in "$@"; do
  [ "$v" = base ] && continue
  GRT_LIB_PATH=$PWD/tools/_ab/$v/libgraphrt_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
    -k "gemv or llama or device_loop or tp_sharded or all_modes" > gpurun_out/${T}_${v}_tests.log 2>&1
  echo "$v tests: $(tail -1 gpurun_out/${T}_${v}_tests.log)"
done
