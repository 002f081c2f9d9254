# launch list of one C4 action: per-launch device time + DRAM bytes (cold-cache, serialised)
python tools/prof_run.py ${CFG:-c4} ${KDIM:-30} 1 > gpurun_out/launches_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${CFG:-c4}.csv python tools/prof_run.py ${CFG:-c4} ${KDIM:-30} 1 > gpurun_out/launches_ncu.log 2>&1
tail -2 gpurun_out/launches_ncu.log
