# final round-2 ncu evidence on the current tree: launch lists (time + DRAM bytes per launch) of the C4 bench in
# both storage modes, then --set full captures of the SpMM row kernels and the fp32 ring passes — each only after
# the same command exited 0 without ncu
for mode in 0 1; do
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --fp32 $mode"
  tag=$([ $mode = 1 ] && echo _fp32 || echo "")
  $CMD > gpurun_out/ncu_plain$tag.json 2> gpurun_out/ncu_plain$tag.err && \
  timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
      --log-file gpurun_out/r02_launches_bench_c4$tag.csv $CMD > gpurun_out/ncu_launch$tag.log 2>&1
  tail -1 gpurun_out/ncu_launch$tag.log
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"spmv_binned_kernelILi4ELb0ELi4ELb0Ed" -s 10 -c 1 -o gpurun_out/r02_prof_spmv $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"(spmv_binned_kernelILi4ELb0ELi8ELb0Ef|dcgs2_dots_ringIf|toar_update_ringILi3Ef)" -s 20 -c 3 \
  -o gpurun_out/r02_prof_fp32 $CMD --fp32 1 > gpurun_out/ncu_full_fp32.log 2>&1
tail -1 gpurun_out/ncu_full_fp32.log
