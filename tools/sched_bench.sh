#!/usr/bin/env bash
# Compare the LTI scan schedules per workload: bench line summaries for auto / 1p / 3p.
#   usage: tools/sched_bench.sh TAG [workloads...]
TAG=${1:-s}
shift || true
WLS=${*:-"c2 c4 c5 c1"}
for w in $WLS; do
  for sc in 1p 3p; do
    timeout 180 python bench.py --workload $w --scan $sc --no-cpu-baseline > gpurun_out/b_${TAG}_${w}_${sc}.json 2> gpurun_out/b_${TAG}_${w}_${sc}.err
    python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/b_${TAG}_${w}_${sc}.json').read().splitlines()[-1]); r = d['roofline']
    print('$w $sc', round(d['ms_per_step'] * 1e3, 1), 'us/step', r['kernel'], round(r['frac'], 3),
          {k: round(v * 1e3, 1) for k, v in r['kernel_ms'].items()})
except Exception as e:
    print('$w $sc failed', e, open('gpurun_out/b_${TAG}_${w}_${sc}.err').read()[-800:])
PY
  done
done
