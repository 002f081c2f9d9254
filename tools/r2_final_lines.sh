# round-2 bench lines (profiles/r02_bench_*.json) on the final tree
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4_final.json 2>gpurun_out/f0.err; tail -2 gpurun_out/f0.err
timeout 900 python bench.py --steps 20 --warmup 5 --fp32 1 > gpurun_out/r02_bench_c4_fp32.json 2>gpurun_out/f10.err; tail -2 gpurun_out/f10.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 > gpurun_out/r02_bench_c4_adaptive.json 2>gpurun_out/f1.err; tail -2 gpurun_out/f1.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --adaptive 1e-13 --fp32 1 > gpurun_out/r02_bench_c4_adaptive_fp32.json 2>gpurun_out/f14.err; tail -2 gpurun_out/f14.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --walk > gpurun_out/r02_bench_c4_walk_lanczos1.json 2>gpurun_out/f11.err; tail -2 gpurun_out/f11.err
timeout 900 python bench.py --b 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c4_b8.json 2>gpurun_out/f9.err; tail -2 gpurun_out/f9.err
timeout 900 python bench.py --diffusion --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_diffusion_c3.json 2>gpurun_out/f2.err; tail -2 gpurun_out/f2.err
timeout 900 python bench.py --diffusion --adaptive 1e-13 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_diffusion_c3_adaptive.json 2>gpurun_out/f3.err; tail -2 gpurun_out/f3.err
timeout 900 python bench.py --diffusion --steps 3 --warmup 3 --no-cpu-baseline --fp32 1 > gpurun_out/r02_bench_diffusion_c3_fp32.json 2>gpurun_out/f12.err; tail -2 gpurun_out/f12.err
timeout 1200 python bench.py --trace --adaptive 1e-13 --steps 2 --warmup 1 > gpurun_out/r02_bench_trace_rational_c3_adaptive.json 2>gpurun_out/f4.err; tail -2 gpurun_out/f4.err
timeout 1200 python bench.py --trace --adaptive 1e-13 --steps 2 --warmup 1 --fp32 1 > gpurun_out/r02_bench_trace_rational_c3_adaptive_fp32.json 2>gpurun_out/f13.err; tail -2 gpurun_out/f13.err
timeout 900 python bench.py --solver cg --config c4 --steps 5 --warmup 3 > gpurun_out/r02_bench_cg_c4.json 2>gpurun_out/f5.err; tail -2 gpurun_out/f5.err
timeout 900 python bench.py --solver cg --config c3 --steps 5 --warmup 3 > gpurun_out/r02_bench_cg_c3.json 2>gpurun_out/f8.err; tail -2 gpurun_out/f8.err
timeout 900 python bench.py --markov --steps 3 --warmup 3 > gpurun_out/r02_bench_markov_c4.json 2>gpurun_out/f6.err; tail -2 gpurun_out/f6.err
timeout 900 python bench.py --rhoz --steps 3 --warmup 3 > gpurun_out/r02_bench_rhoz_c4.json 2>gpurun_out/f7.err; tail -2 gpurun_out/f7.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02_bench_reference.json 2>gpurun_out/f15.err; tail -2 gpurun_out/f15.err
