#!/usr/bin/env bash
# quick iteration loop on the GPU box: LTI parity tests, per-workload bench, phase traces
TAG=${1:-q}
shift || true
WLS=${*:-"c2 c4 c5 c1"}
timeout 600 python -m pytest tests/test_gpu_lti.py -x -q > gpurun_out/t_$TAG.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_$TAG.log
for w in $WLS; do
  timeout 120 python bench.py --workload $w --no-cpu-baseline > gpurun_out/b_${TAG}_$w.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/b_${TAG}_$w.json').read().splitlines()[-1]); r=d['roofline']
print('$w', round(d['ms_per_step']*1e3,1), 'us/step', r['kernel'], round(r['frac'],3), {k:round(v*1e3,1) for k,v in r['kernel_ms'].items()})"
done
for w in $WLS; do python tools/trace_phases.py --workload $w > gpurun_out/trace_${TAG}_$w.log 2>&1; done
