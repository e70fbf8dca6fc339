#!/usr/bin/env bash
# One gpurun call's worth of round evidence (run from the repo root on the GPU box):
#   bench lines for every workload, the reference (oracle) arm, per-launch ncu
#   lists (duration + DRAM bytes) and one `--set full` capture of each
#   workload family's dominant kernel.  Output: gpurun_out/$TAG/.
#   usage: tools/profile_round.sh TAG [workloads...]
set -u
TAG=${1:-r01}
shift || true
WLS=${*:-"c2 c1 c4 c5 c3 f1"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
for w in $WLS; do
  timeout 600 python bench.py --workload "$w" > "$OUT/bench_$w.json" 2> "$OUT/bench_$w.err"
  echo "bench $w rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/ref_c2.json" 2> "$OUT/ref_c2.err"
for w in $WLS; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file "$OUT/launches_$w.csv" \
    python bench.py --workload "$w" --steps 2 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
  echo "launches $w rc=$?"
done
if [[ " $WLS " == *" c2 "* ]]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lti_bwd -s 4 -c 1 \
    -o "$OUT/full_c2_lti_bwd" python bench.py --workload c2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline \
    > "$OUT/full_c2.log" 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lti_fwd -s 4 -c 1 \
    -o "$OUT/full_c2_lti_fwd" python bench.py --workload c2 --steps 2 --warmup 3 --no-graph --no-cpu-baseline \
    > "$OUT/full_c2f.log" 2>&1
  echo "full c2 rc=$?"
fi
if [[ " $WLS " == *" c3 "* ]]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tv_seq_kernel -s 2 -c 1 \
    -o "$OUT/full_c3_tv_bwd" python bench.py --workload c3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline \
    > "$OUT/full_c3.log" 2>&1
  echo "full c3 rc=$?"
fi
