# quick GPU iteration: parity tests + C4 bench kernel table
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -${TESTLINES:-3}
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e ${BENCHARGS} 2>gpurun_out/bench_c4.err > gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_c4.json"))
print("value", round(d["value"], 3), "ms/step", round(d["ms_per_step"], 1), "launches", d["gpu_launches"])
for k, v in d["kernels"].items():
    print(f'{k:20s} ms/step={v["ms_per_step"]:9.2f} share={v["share"]:.3f} n={v["launches_per_step"]:5.0f} '
          + (f'GB/s={v["achieved_gbs"]:8.1f} frac={v["frac"]:.3f}' if "frac" in v else ""))
PY
