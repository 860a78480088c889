# per-kernel device times of one C2 step (second of two), from ncu's gpu__time_duration
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_step.py ${1:-c2} 2 > gpurun_out/lt.csv 2>/dev/null
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/lt.csv")) if len(r)>10]
h=rows[0]; iN=h.index("Kernel Name"); iV=h.index("Metric Value")
data=[(r[iN][:48], float(r[iV].replace(",",""))) for r in rows[1:]]
for nm,v in data[len(data)//2:]: print(f"{v/1000:8.1f} us  {nm}")
PY
