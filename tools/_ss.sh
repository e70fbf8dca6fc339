mkdir -p gpurun_out/ss
timeout 900 python -m pytest tests/test_gpu_tv.py tests/test_gpu_tvdf.py tests/test_gpu_tvtdf.py tests/test_gpu_robust.py -x -q -p no:cacheprovider > gpurun_out/ss/t.log 2>&1; echo tests=$?; tail -2 gpurun_out/ss/t.log
for w in c3 f2; do
timeout 120 python bench.py --workload $w --no-cpu-baseline --steps 20 > gpurun_out/ss/b_$w.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ss/b_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['ms_per_step']*1e3,1), 'us/step', r['kernel'], round(r['frac'],3), {k:round(v*1e3,1) for k,v in r['kernel_ms'].items()}, 'e2e', d['e2e']['value'])" 2>&1 | tail -1
done
