# rebuild with each set of compile-time flags (args) and time the plain C4 step (no per-class split)
for flags in "$@"; do
  WL_EXTRA_NVCC="$flags" python -c "from paper_2601_11338_b200 import build; build.build(force=True)" || exit 1
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vb.json 2>/dev/null
  python - "$flags" <<'PY'
import json, sys
d = json.load(open("gpurun_out/vb.json"))
print("==", sys.argv[1], "ms/step", round(d["ms_per_step"], 1), "spmv", round(d["kernels"]["spmv_binned"]["ms_per_step"], 1), "sm_mhz", d["clocks"].get("sm_mhz"))
PY
done
python -c "from paper_2601_11338_b200 import build; build.build(force=True)"
