# ncu --set full of the fp32-storage Gram passes (dots, 3-output update) in the C4 --fp32 bench
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --fp32 1"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"(dcgs2_dots_ringIf|toar_update_ringILi3EfE)" -s 20 -c 2 \
  -o gpurun_out/prof_fp32 $CMD > gpurun_out/ncu_fp32.log 2>&1
tail -3 gpurun_out/ncu_fp32.log
