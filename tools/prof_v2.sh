#!/usr/bin/env bash
# ncu --set full of the v2 LTI kernels on one workload (GPU box): summaries + per-line shares.
#   tools/prof_v2.sh TAG WORKLOAD [kernel-regex]
TAG=${1:-p}; W=${2:-c5}; KRE=${3:-lti2_(fwd|bwd)}
OUT=gpurun_out/$TAG; mkdir -p $OUT
IIRG_LIB=${IIRG_LIB:-} timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$KRE" -s ${SKIP:-2} -c ${CNT:-2} \
  -o $OUT/full python bench.py --workload $W --steps 2 --warmup 1 --no-graph --no-cpu-baseline > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
python profiles/ncu_summary.py $OUT/full.ncu-rep $OUT/summary.txt > /dev/null 2>&1
for k in lti2_fwd lti2_bwd; do python tools/ncu_lines.py $OUT/full.ncu-rep $k 45 > $OUT/lines_$k.txt 2>&1; done
ncu -i $OUT/full.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
[ -n "$KEEP" ] || rm -f $OUT/full.ncu-rep
cat $OUT/summary.txt
