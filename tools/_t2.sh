mkdir -p gpurun_out/t2
timeout 300 python tools/trace_v2.py --workload c5 > gpurun_out/t2/trace_c5.txt 2>&1
timeout 600 ncu --replay-mode range --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none python tools/step_range.py --workload c5 > gpurun_out/t2/step_range_c5.txt 2>&1; echo range=$?
tail -20 gpurun_out/t2/step_range_c5.txt
