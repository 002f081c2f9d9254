# headline lines with the committed ncu traffic tables, the fp32 secondary lines, and the gather ceilings
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4_final.json 2>gpurun_out/g0.err; tail -2 gpurun_out/g0.err
timeout 900 python bench.py --steps 20 --warmup 5 --fp32 1 > gpurun_out/r02_bench_c4_fp32.json 2>gpurun_out/g1.err; tail -2 gpurun_out/g1.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 > gpurun_out/r02_bench_c4_adaptive.json 2>gpurun_out/g2.err; tail -2 gpurun_out/g2.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 --fp32 1 > gpurun_out/r02_bench_c4_adaptive_fp32.json 2>gpurun_out/g3.err; tail -2 gpurun_out/g3.err
timeout 900 python bench.py --diffusion --steps 3 --warmup 3 --no-cpu-baseline --fp32 1 > gpurun_out/r02_bench_diffusion_c3_fp32.json 2>gpurun_out/g4.err; tail -2 gpurun_out/g4.err
timeout 1200 python bench.py --trace --adaptive 1e-13 --steps 2 --warmup 1 --fp32 1 > gpurun_out/r02_bench_trace_rational_c3_adaptive_fp32.json 2>gpurun_out/g5.err; tail -2 gpurun_out/g5.err
timeout 600 ./tools/gather_ceiling > gpurun_out/r02_gather_ceiling.txt 2>&1; tail -8 gpurun_out/r02_gather_ceiling.txt
