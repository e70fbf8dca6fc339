#!/usr/bin/env bash
# One gpurun call's worth of round evidence (run from the repo root on the GPU box):
#   bench lines for every workload, the reference (oracle) arm, per-launch ncu
#   lists (duration + DRAM bytes) and `--set full` captures of the dominant
#   kernels (C2 lti_fwd / lti_bwd, C5 lti_fwd / lti_bwd, C3 tv_bwd).
#   Output: gpurun_out/$TAG/.   usage: tools/profile_round.sh TAG [workloads...]
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
full() {   # workload kernel-regex skip name
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s "$3" -c 1 \
    -o "$OUT/full_$4" python bench.py --workload "$1" --steps 2 --warmup 3 --no-graph --no-cpu-baseline \
    > "$OUT/full_$4.log" 2>&1
  echo "full $4 rc=$?"
}
[[ " $WLS " == *" c2 "* ]] && { full c2 lti_bwd 4 c2_lti_bwd; full c2 lti_fwd 4 c2_lti_fwd; }
[[ " $WLS " == *" c5 "* ]] && { full c5 lti_bwd 4 c5_lti_bwd; full c5 lti_fwd 4 c5_lti_fwd; }
[[ " $WLS " == *" c3 "* ]] && full c3 "tv_seq_kernel" 2 c3_tv_bwd
# summarise the captures here (gpurun copies back <= 64 MiB): text only, reports dropped
for r in "$OUT"/full_*.ncu-rep; do
  [ -e "$r" ] || continue
  n=$(basename "$r" .ncu-rep)
  python profiles/ncu_summary.py "$r" "$OUT/${n}_summary.txt" > /dev/null 2>&1
  python tools/ncu_lines.py "$r" "." 40 > "$OUT/${n}_lines.txt" 2>&1
  ncu -i "$r" --page raw --csv > "$OUT/${n}_raw.csv" 2>/dev/null
  rm -f "$r"
done
exit 0
