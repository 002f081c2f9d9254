# secondary bench lines of round 2 (profiles/r02_bench_*.json)
set -x
timeout 900 python bench.py --diffusion --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_diffusion_c3.json 2>gpurun_out/l1.err; tail -2 gpurun_out/l1.err
timeout 900 python bench.py --diffusion --adaptive 1e-13 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_diffusion_c3_adaptive.json 2>gpurun_out/l2.err; tail -2 gpurun_out/l2.err
timeout 900 python bench.py --b 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c4_b8.json 2>gpurun_out/l3.err; tail -2 gpurun_out/l3.err
timeout 900 python bench.py --solver cg --config c3 --steps 5 --warmup 3 > gpurun_out/r02_bench_cg_c3.json 2>gpurun_out/l4.err; tail -2 gpurun_out/l4.err
timeout 900 python bench.py --rhoz --steps 3 --warmup 3 > gpurun_out/r02_bench_rhoz_c4.json 2>gpurun_out/l5.err; tail -2 gpurun_out/l5.err
timeout 900 python bench.py --markov --steps 3 --warmup 3 > gpurun_out/r02_bench_markov_c4.json 2>gpurun_out/l6.err; tail -2 gpurun_out/l6.err
