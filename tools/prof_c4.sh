set -x
python tools/prof_run.py ${CFG:-c4} ${KDIM:-12} 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-spmv_binned|dcgs2}" -s ${SKIP:-60} -c ${COUNT:-6} -o gpurun_out/prof_c4_${TAG:-r3} python tools/prof_run.py ${CFG:-c4} ${KDIM:-12} 2 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
