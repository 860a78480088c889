# Round-2 closing capture (run under gpurun): headline line, all configs (CPU baseline + parity),
# the reference arm, the C2 launch list, ncu --set full summaries of the hot kernels.
set -x
D=gpurun_out/r2g; mkdir -p $D
timeout 900 python bench.py > $D/bench_c2.json 2> $D/bench_c2.err
timeout 2400 python bench.py --all --steps 10 --warmup 3 > $D/bench_all.json 2> $D/bench_all.err
for c in c2 c1; do timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $D/ref_$c.json 2> $D/ref_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_launch.log 2>&1
python tools/ncu_summary.py --launches $D/launches_c2.csv $D/launches_c2.json > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
cap() {  # name kernel-regex skip workload reps label
  timeout 900 $NCU -k "regex:$2" -s $3 -c 1 -o $D/$1 python tools/prof_step.py $4 $5 > $D/ncu_$1.log 2>&1
  python tools/ncu_summary.py $D/$1.ncu-rep $D/$1.json --label "$6" > /dev/null 2>&1
  rm -f $D/$1.ncu-rep
}
cap c2_k_nn2 'k_nn2<' 1 c2 2 "round2 closing C2 CDTW phase B: k_nn2, two pairs per warp (P=8 half-warps, series through L1 from padded HBM copies, per-query work counters)"
cap c2_k_lb_matrix 'k_lb_matrix<' 1 c2 2 "round2 closing C2 LB_Keogh key matrix"
cap c4m_k_nn 'k_nn<\(int\)4, \(int\)0, \(int\)16>' 0 c4m 1 "round2 closing C4 MSM k_nn phase B tail ranks (guarded P=4 band +-61, slot-0 result mask, split/merge factor by IMAD)"
cap c4t_k_nn 'k_nn<\(int\)5, \(int\)0, \(int\)16>' 0 c4t 1 "round2 closing C4 TWE k_nn phase B tail ranks (guarded P=4 band +-61, slot-0 result mask, bulk candidate staging)"
ls -la $D
echo done
