# parity tests, then the C4 bench under several experiment knobs (env assignments as args)
[ -z "$SKIPTESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x --timeout 180 -p no:cacheprovider 2>&1 | tail -${TESTLINES:-3}
for cfg in "$@"; do
  env $cfg timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e ${BENCHARGS} 2>gpurun_out/bench_sweep.err > gpurun_out/bench_sweep.json || tail -5 gpurun_out/bench_sweep.err
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/bench_sweep.json"))
print("==", sys.argv[1], "value", round(d["value"], 3), "ms/step", round(d["ms_per_step"], 1))
for k, v in d["kernels"].items():
    if v["share"] > 0.01:
        print(f'   {k:20s} ms/step={v["ms_per_step"]:9.2f} share={v["share"]:.3f} ' + (f'GB/s={v["achieved_gbs"]:8.1f} frac={v["frac"]:.3f}' if "frac" in v else ""))
PY
done
