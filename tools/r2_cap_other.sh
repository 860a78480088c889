# ncu --set full captures of the non-headline hot kernels (run under gpurun, one GPU).
# Reports are summarised on the box (tools/ncu_summary.py) and only the summaries plus
# the raw CSV pages come back (gpurun returns <= 64 MiB).
set -x
D=gpurun_out/r2o
mkdir -p $D
timeout 900 python bench.py --all --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_all.json 2> $D/bench_all.err
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base function"
cap() {  # name regex skip count workload reps
  timeout 600 $NCU -k "regex:$2" -s $3 -c $4 -o $D/$1 python tools/prof_step.py $5 $6 > $D/ncu_$1.log 2>&1
  python tools/ncu_summary.py $D/$1.ncu-rep $D/$1.json --label "$1" > /dev/null 2>&1
  ncu -i $D/$1.ncu-rep --page source --csv > $D/$1.source.csv 2>/dev/null
  gzip -f $D/$1.source.csv
  rm -f $D/$1.ncu-rep
}
cap k_triangle_c3w '^k_triangle$' 1 1 c3w 2
cap k_triangle_c3e '^k_triangle$' 1 1 c3e 2
cap k_lb_matrix_c2 '^k_lb_matrix$' 4 1 c2 2
cap k_subseq_lb_c5 '^k_subseq_lb$' 0 1 c5 1
cap k_subseq_c5 '^k_subseq$' 0 2 c5 1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c5.csv python tools/prof_step.py c5 2 > $D/ncu_c5l.log 2>&1
du -sh $D
echo done
