set -x
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 python bench.py --diffusion --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/diff_final.json 2> gpurun_out/diff_final.err
timeout 300 python bench.py --diffusion --relabel 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/diff_norelabel.json 2> gpurun_out/diff_norelabel.err
timeout 300 python bench.py --trace --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/trace_final.json 2> gpurun_out/trace_final.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/launches_bench.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests5.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests5.log
