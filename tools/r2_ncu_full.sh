# launch list (time + DRAM bytes per launch) of the C4 bench command, then one --set full capture of the B=11 row
# kernel (32-byte lanes) — each only after the same command exited 0 without ncu
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r02_launches_bench_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -1 gpurun_out/ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"spmv_binned_kernelILi4ELb0ELi4ELb0E" -s 10 -c 1 -o gpurun_out/r02_prof_spmv $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
