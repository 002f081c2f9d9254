# one ncu --set full capture of the B=11 (VW=4) SpMM rows kernel and the batched small-row kernel in the C4 bench
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"spmv_(binned_kernelILi4ELb0ELi4E|small_batched_kernelILi2ELb0ELi4E)" -s 10 -c 2 \
  -o gpurun_out/prof_spmv $CMD > gpurun_out/ncu_spmv.log 2>&1
tail -3 gpurun_out/ncu_spmv.log
