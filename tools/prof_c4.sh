set -x
python tools/prof_run.py c4 30 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spmv_binned|gram_update_proj|gram_proj|gram_update_norm" -s 130 -c 8 -o gpurun_out/prof_c4_r2 python tools/prof_run.py c4 30 2 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
