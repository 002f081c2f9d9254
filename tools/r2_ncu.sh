# ncu launch list (device time + DRAM bytes per launch) of the C4 bench command, after it exited 0 without ncu
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r02_launches_bench_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
