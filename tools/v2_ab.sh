#!/usr/bin/env bash
# A/B of library variants on the GPU box: parity tests on the default build, then C5/C2/C4 per variant.
#   tools/v2_ab.sh TAG variant1 variant2 ...   ("default" = lib/libiirgrad.so)
TAG=$1; shift
timeout 900 python -m pytest tests/test_gpu_lti.py tests/test_gpu_robust.py -x -q 2>&1 | tail -4 > gpurun_out/t_$TAG.log; cat gpurun_out/t_$TAG.log
for v in "$@"; do
  if [ "$v" = "default" ]; then lib=paper_2511_14390_b200/lib/libiirgrad.so; else lib=paper_2511_14390_b200/lib/libiirgrad_$v.so; fi
  for w in c5 c2 c4; do
    IIRG_LIB=$PWD/$lib timeout 120 python bench.py --workload $w --no-cpu-baseline --steps 50 > gpurun_out/b_${TAG}_${v}_$w.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/b_${TAG}_${v}_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $w', round(d['ms_per_step']*1e3,1), 'us/step', r['kernel'], round(r['frac'],3), {k:round(v*1e3,1) for k,v in r['kernel_ms'].items()})" 2>&1 | tail -1
  done
done
