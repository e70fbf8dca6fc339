mkdir -p gpurun_out/u1
timeout 900 python -m pytest tests/test_gpu_lti_engines.py tests/test_gpu_lti.py tests/test_gpu_robust.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/u1/t.log 2>&1; echo tests=$?; tail -2 gpurun_out/u1/t.log
for w in c5 c4; do
timeout 120 python bench.py --workload $w --no-cpu-baseline --steps 100 > gpurun_out/u1/b_$w.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/u1/b_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['ms_per_step']*1e3,1), 'us/step', r['kernel'], round(r['frac'],3), {k:round(v*1e3,1) for k,v in r['kernel_ms'].items()})" 2>&1 | tail -1
done
