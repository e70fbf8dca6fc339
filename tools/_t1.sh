mkdir -p gpurun_out/t1
timeout 900 python -m pytest tests/test_gpu_diag.py tests/test_gpu_rec.py -q -p no:cacheprovider > gpurun_out/t1/t.log 2>&1; echo tests=$?; tail -4 gpurun_out/t1/t.log
for w in f1m4 f3m4; do
timeout 200 python bench.py --workload $w > gpurun_out/t1/bench_$w.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/t1/bench_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['ms_per_step']*1e3,1), 'us/step', r['kernel'], round(r['frac'],3), {k:round(v*1e3,1) for k,v in r['kernel_ms'].items()})" 2>&1 | tail -1
done
timeout 600 ncu --replay-mode range --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none python tools/step_range.py --workload c5 > gpurun_out/t1/step_range_c5.txt 2>&1; echo range=$?
tail -20 gpurun_out/t1/step_range_c5.txt
