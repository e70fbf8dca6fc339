mkdir -p gpurun_out/t3
timeout 300 python tools/trace_v2.py --workload c5 > gpurun_out/t3/trace_c5.txt 2>&1
