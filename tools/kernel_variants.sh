# C4 bench kernel table (every kernel > 0.5 ms/step) for compile-time variants: tools/kernel_variants.sh "-DA=1" ...
# (BENCHARGS: extra bench flags, e.g. "--fp32 1"); the tree is rebuilt with the defaults at the end
for v in "$@"; do
  echo "=== WL_EXTRA_NVCC=$v"
  WL_EXTRA_NVCC="$v" python -c "from paper_2601_11338_b200 import build; build.build(force=True)" || continue
  WL_SPMV_SPLIT=1 timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e ${BENCHARGS} \
      2>gpurun_out/var.err > gpurun_out/var.json || tail -3 gpurun_out/var.err
  python - <<'PY'
import json
d = json.load(open("gpurun_out/var.json"))
print("value", round(d["value"], 3), "ms/step", round(d["ms_per_step"], 1), "clocks", d.get("clocks"))
for k, v in d["kernels"].items():
    if v["ms_per_step"] > 0.5:
        print(f'  {k:20s} ms/step={v["ms_per_step"]:9.2f} n={v["launches_per_step"]:5.0f} ' + (f'frac={v["frac"]:.3f}' if "frac" in v else ""))
PY
done
python -c "from paper_2601_11338_b200 import build; build.build(force=True)"
