# the fp32-mode lines on the final tree
set -x
timeout 900 python bench.py --steps 20 --warmup 5 --fp32 1 > gpurun_out/r02_bench_c4_fp32.json 2>gpurun_out/p1.err; tail -1 gpurun_out/p1.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 --fp32 1 > gpurun_out/r02_bench_c4_adaptive_fp32.json 2>gpurun_out/p2.err; tail -1 gpurun_out/p2.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --walk --fp32 1 > gpurun_out/r02_bench_c4_walk_fp32.json 2>gpurun_out/p3.err; tail -1 gpurun_out/p3.err
timeout 900 python bench.py --diffusion --steps 3 --warmup 3 --no-cpu-baseline --fp32 1 > gpurun_out/r02_bench_diffusion_c3_fp32.json 2>gpurun_out/p4.err; tail -1 gpurun_out/p4.err
timeout 1200 python bench.py --trace --steps 2 --warmup 1 --fp32 1 > gpurun_out/r02_bench_trace_rational_c3_fp32.json 2>gpurun_out/p5.err; tail -1 gpurun_out/p5.err
timeout 1200 python bench.py --trace --adaptive 1e-13 --steps 2 --warmup 1 --fp32 1 > gpurun_out/r02_bench_trace_rational_c3_adaptive_fp32.json 2>gpurun_out/p6.err; tail -1 gpurun_out/p6.err
