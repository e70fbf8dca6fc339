#!/usr/bin/env bash
# GPU box: full GPU test suite, then one bench line per workload (summary lines to stdout).
#   tools/gpu_all.sh TAG [workloads...]
TAG=${1:-g}; shift || true
WLS=${*:-"c5 c2 c4 c1 c3 f1 f2 f3"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo tests=$?; tail -3 $OUT/tests.log
fi
for w in $WLS; do
  timeout 300 python bench.py --workload $w ${BENCH_ARGS:-} > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python - "$OUT/bench_$w.json" "$w" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], round(d["ms_per_step"] * 1e3, 1), "us/step", r.get("kernel"), round(r["frac"], 3),
          {k: round(v * 1e3, 1) for k, v in r.get("kernel_ms", {}).items()}, "e2e", d.get("e2e", {}).get("value"))
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
