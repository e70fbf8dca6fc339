mkdir -p gpurun_out/r1
timeout 900 python -m pytest tests/test_gpu_tvtdf.py tests/test_gpu_tvdf.py tests/test_gpu_tv.py -q -p no:cacheprovider > gpurun_out/r1/t.log 2>&1; echo tests=$?; tail -15 gpurun_out/r1/t.log
