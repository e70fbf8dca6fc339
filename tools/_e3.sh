OUT=gpurun_out/ev3; mkdir -p $OUT
for w in c3 f2 f2t; do
  timeout 300 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "bench $w rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1; echo "launches $w rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:tv_phi" -s 1 -c 1 -o $OUT/full_phi python bench.py --workload c3 --steps 2 --warmup 3 --no-graph --no-cpu-baseline > $OUT/full_phi.log 2>&1
python profiles/ncu_summary.py $OUT/full_phi.ncu-rep $OUT/ncu_c3_tv_phi.txt > /dev/null 2>&1; rm -f $OUT/full_phi.ncu-rep
