mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:partial -c 40 --csv --log-file gpurun_out/partial_launches.csv python tools/partial_split2.py c5 > gpurun_out/partial_ncu.log 2>&1; echo ncu=$?
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/partial_launches.csv') if l.startswith('"'))]
from collections import defaultdict
d=defaultdict(list)
for r in rows:
    if r.get('Metric Name')=='gpu__time_duration.sum':
        d[r['Kernel Name'][:40]].append(float(r['Metric Value'].replace(',','')))
for k,v in d.items(): print(k, len(v), 'mean', sum(v)/len(v), r['Metric Unit'])
PY
