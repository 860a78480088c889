# Round-2 capture (run under gpurun): headline line, all configs with CPU baseline + parity,
# the reference arm, launch list, ncu of the top kernels (summarised on the box).
set -x
D=gpurun_out/r2c; mkdir -p $D
timeout 900 python bench.py > $D/bench_c2.json 2> $D/bench_c2.err
timeout 2400 python bench.py --all --steps 10 --warmup 3 > $D/bench_all.json 2> $D/bench_all.err
for c in c2 c1; do timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $D/ref_$c.json 2> $D/ref_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launch.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name kernel-regex skip count workload reps
  timeout 900 $NCU -k "regex:$2" -s $3 -c $4 -o $D/$1 python tools/prof_step.py $5 $6 > $D/ncu_$1.log 2>&1
  python tools/ncu_summary.py $D/$1.ncu-rep $D/$1.json --label "$1" > /dev/null 2>&1
  ncu -i $D/$1.ncu-rep --page source --csv --print-source sass > $D/$1.sass.csv 2>/dev/null; gzip -f $D/$1.sass.csv
  rm -f $D/$1.ncu-rep
}
cap k_nn_c2 'k_nn<' 1 1 c2 2
cap k_lb_matrix_c2 'lb_matrix' 1 1 c2 2
cap k_nn_c4m 'k_nn<' 3 1 c4m 1
cap k_nn_c4t 'k_nn<' 3 1 c4t 1
cap k_triangle_c3w 'k_triangle' 1 1 c3w 2
cap k_triangle_c3e 'k_triangle' 1 1 c3e 2
cap k_subseq_lb_c5 'k_subseq_lb' 0 1 c5 1
cap k_subseq_c5 'k_subseq<' 1 1 c5 1
du -sh $D
echo done
