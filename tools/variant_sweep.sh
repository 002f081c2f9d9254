# rebuild with each set of compile-time flags (args) and time the C4 step (per-class SpMM split);
# BENCH_ARGS (e.g. "--diffusion") selects another bench workload
i=0
for flags in "$@"; do
  i=$((i+1))
  WL_EXTRA_NVCC="$flags" python -c "from paper_2601_11338_b200 import build; build.build(force=True)" || exit 1
  WL_SPMV_SPLIT=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/variant_$i.json 2>/dev/null
  python - "$flags" $i <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/variant_{sys.argv[2]}.json"))
print("==", sys.argv[1], "ms/step", round(d["ms_per_step"], 1), {k: round(v["ms_per_step"], 1) for k, v in d["kernels"].items() if v["share"] > 0.05})
PY
done
python -c "from paper_2601_11338_b200 import build; build.build(force=True)"
