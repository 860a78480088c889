# one ncu --set full capture with SASS source counts (run under gpurun): $1 name, $2 kernel regex, $3 skip, $4 workload, $5 reps
D=gpurun_out/cap; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k "regex:$2" -s $3 -c 1 -o $D/$1 python tools/prof_step.py $4 $5 > $D/ncu_$1.log 2>&1
python tools/ncu_summary.py $D/$1.ncu-rep $D/$1.json --label "$1" > /dev/null 2>&1
ncu -i $D/$1.ncu-rep --page source --csv --print-source sass > $D/$1.sass.csv 2>/dev/null; gzip -f $D/$1.sass.csv
ncu -i $D/$1.ncu-rep --page raw --csv > $D/$1.raw.csv 2>/dev/null; gzip -f $D/$1.raw.csv
rm -f $D/$1.ncu-rep
