# full GPU test suite, the full bench line (cpu_baseline + e2e), then the ncu launch list of the bench command
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -3 gpurun_out/bench_full.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c ${NLAUNCH:-4000} --csv \
    --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/launches_bench.log 2>&1
tail -2 gpurun_out/launches_bench.log
