# C4 bench kernel table for compile-time SpMM variants: tools/build_variants.sh "-DA=1" "-DB=2" ...
for v in "$@"; do
  echo "=== WL_EXTRA_NVCC=$v"
  WL_EXTRA_NVCC="$v" python -c "from paper_2601_11338_b200 import build; build.build(force=True)" || continue
  WL_SPMV_SPLIT=1 timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e ${BENCHARGS} \
      2>gpurun_out/var.err > gpurun_out/var.json || tail -3 gpurun_out/var.err
  python - <<'PY'
import json
d = json.load(open("gpurun_out/var.json"))
b1 = d.get("spmv", {}).get("b1", {})
print("value", round(d["value"], 3), "ms/step", round(d["ms_per_step"], 1), "spmv.b1 ms", round(b1.get("ms_per_launch", 0), 3),
      {k: round(v, 3) for k, v in b1.get("class_ms_per_launch", {}).items()}, "clocks", d.get("clocks"))
for k, v in d["kernels"].items():
    if k.startswith("spmv"):
        print(f'  {k:20s} ms/step={v["ms_per_step"]:9.2f} n={v["launches_per_step"]:5.0f}')
PY
done
python -c "from paper_2601_11338_b200 import build; build.build(force=True)"
