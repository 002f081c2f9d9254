# C4 bench kernel table under SpMM variants (env), one line per kernel: tools/spmv_variants.sh "VAR=a" "VAR=b" ...
for v in "$@"; do
  echo "=== $v"
  env $v WL_SPMV_SPLIT=1 timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e ${BENCHARGS} \
      2>gpurun_out/var.err > gpurun_out/var.json || tail -3 gpurun_out/var.err
  python - <<'PY'
import json
d = json.load(open("gpurun_out/var.json"))
print("value", round(d["value"], 3), "ms/step", round(d["ms_per_step"], 1), "spmv.b1", json.dumps(d.get("spmv", {}).get("b1", {}))[:200])
for k, v in d["kernels"].items():
    if v["ms_per_step"] > 0.5:
        print(f'  {k:20s} ms/step={v["ms_per_step"]:9.2f} n={v["launches_per_step"]:5.0f} ' + (f'frac={v["frac"]:.3f}' if "frac" in v else ""))
PY
done
