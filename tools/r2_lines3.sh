# the headline lines on the final tree (clock sampler started before the timed region)
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4_final.json 2>gpurun_out/k0.err; tail -2 gpurun_out/k0.err
timeout 900 python bench.py --steps 20 --warmup 5 --fp32 1 > gpurun_out/r02_bench_c4_fp32.json 2>gpurun_out/k1.err; tail -2 gpurun_out/k1.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 > gpurun_out/r02_bench_c4_adaptive.json 2>gpurun_out/k2.err; tail -2 gpurun_out/k2.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 --fp32 1 > gpurun_out/r02_bench_c4_adaptive_fp32.json 2>gpurun_out/k3.err; tail -2 gpurun_out/k3.err
timeout 900 python bench.py --rhoz --steps 5 --warmup 3 > gpurun_out/r02_bench_rhoz_c4.json 2>gpurun_out/k4.err; tail -2 gpurun_out/k4.err
