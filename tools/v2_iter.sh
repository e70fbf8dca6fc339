#!/usr/bin/env bash
# one iteration on the GPU box: LTI parity + robust tests, C5/C2/C4 bench lines, optional ncu of c5
TAG=${1:-v}; PROF=${2:-0}
timeout 900 python -m pytest tests/test_gpu_lti.py tests/test_gpu_robust.py -x -q 2>&1 | tail -6 > gpurun_out/t_$TAG.log; cat gpurun_out/t_$TAG.log
for w in c5 c2 c4; do
  timeout 120 python bench.py --workload $w --no-cpu-baseline --steps 50 > gpurun_out/b_${TAG}_$w.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/b_${TAG}_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['ms_per_step']*1e3,1), 'us/step', r['kernel'], round(r['frac'],3), {k:round(v*1e3,1) for k,v in r['kernel_ms'].items()})" 2>&1 | tail -1
done
if [ "$PROF" = "1" ]; then tools/prof_v2.sh p_$TAG c5 > /dev/null 2>&1; head -30 gpurun_out/p_$TAG/summary.txt; fi
