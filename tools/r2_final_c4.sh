D=gpurun_out/r2f; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
cap() {
  timeout 900 $NCU -k "regex:$2" -s $3 -c 1 -o $D/$1 python tools/prof_step.py $4 $5 > $D/ncu_$1.log 2>&1
  python tools/ncu_summary.py $D/$1.ncu-rep $D/$1.json --label "$6" > /dev/null 2>&1
  rm -f $D/$1.ncu-rep
}
cap c4m_k_nn 'k_nn<\(int\)4, \(int\)0, \(int\)16>' 0 c4m 1 "round2 C4 MSM k_nn phase B tail ranks (guarded P=4 band, split/merge choice as FMA)"
cap c4t_k_nn 'k_nn<\(int\)5, \(int\)0, \(int\)16>' 0 c4t 1 "round2 C4 TWE k_nn phase B tail ranks (guarded P=4 band, bulk candidate staging)"
ls $D/*.json
