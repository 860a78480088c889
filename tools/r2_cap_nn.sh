set -x
D=gpurun_out/r2d; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "subseq" > $D/pytest_subseq.log 2>&1; tail -2 $D/pytest_subseq.log
cp paper_2102_05221_b200/libelastik_b200.so /tmp/cur.so
cp absx/live.so paper_2102_05221_b200/libelastik_b200.so
timeout 600 python tools/live_cells.py c2 c4m c4t > $D/live_cells.txt 2>&1
cp /tmp/cur.so paper_2102_05221_b200/libelastik_b200.so
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name kernel-regex skip count workload reps
  timeout 900 $NCU -k "regex:$2" -s $3 -c $4 -o $D/$1 python tools/prof_step.py $5 $6 > $D/ncu_$1.log 2>&1
  python tools/ncu_summary.py $D/$1.ncu-rep $D/$1.json --label "$1" > /dev/null 2>&1
  ncu -i $D/$1.ncu-rep --page source --csv --print-source sass > $D/$1.sass.csv 2>/dev/null; gzip -f $D/$1.sass.csv
  rm -f $D/$1.ncu-rep
}
cap k_nn_c2 '^k_nn$' 1 1 c2 2
cap k_nn_c4m '^k_nn$' 3 1 c4m 2
cap k_nn_c4t '^k_nn$' 3 1 c4t 2
cap k_subseq_c5 '^k_subseq$' 1 1 c5 1
cat $D/live_cells.txt
echo done
