#!/usr/bin/env bash
# Round-2 evidence on the GPU box (one call): bench lines for every workload, the reference
# (oracle) arm, ncu launch lists (duration + DRAM bytes per launch) and --set full captures of
# the dominant kernels, per-tile phase traces.  Output: gpurun_out/$TAG/.
TAG=${1:-ev}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
for w in c5 c4 c2 c1 c3 f1 f2 f2t f3 f1m4 f3m4; do
  timeout 300 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "bench $w rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_c5.json 2> $OUT/ref.err; echo "ref rc=$?"
for w in c5 c4 c2 c1 c3 f1 f2 f2t f3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
  echo "launches $w rc=$?"
done
full() {   # workload kernel-regex skip name
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s "$3" -c 1 \
    -o $OUT/full_$4 python bench.py --workload "$1" --steps 2 --warmup 3 --no-graph --no-cpu-baseline \
    > $OUT/full_$4.log 2>&1
  echo "full $4 rc=$?"
  python profiles/ncu_summary.py $OUT/full_$4.ncu-rep $OUT/ncu_$4.txt > /dev/null 2>&1
  python tools/ncu_lines.py $OUT/full_$4.ncu-rep "$2" 40 > $OUT/ncu_$4_lines.txt 2>&1
  rm -f $OUT/full_$4.ncu-rep
}
full c5 lti2_bwd 4 c5_lti_bwd
full c5 lti2_fwd 4 c5_lti_fwd
full c2 lti_bwd 4 c2_lti_bwd
full c3 tv_seq_kernel 2 c3_tv_bwd
for w in c5 c4; do timeout 300 python tools/trace_v2.py --workload $w > $OUT/trace_$w.txt 2>&1; done
timeout 600 ncu --replay-mode range --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none python tools/step_range.py --workload c5 > $OUT/step_range_c5.txt 2>&1
exit 0
