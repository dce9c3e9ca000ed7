mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/setup_c3.csv python tools/setup_breakdown.py c3 > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/setup_c3.csv') if not l.startswith('=='))]
import collections
k=collections.OrderedDict()
for r in rows:
    d=k.setdefault(r['ID'],{'name':r['Kernel Name'].split('(')[0][:70]})
    d[r['Metric Name']]=float(r['Metric Value'].replace(',',''))
for i,d in k.items():
    t=d.get('gpu__time_duration.sum',0)/1e6
    if t>0.2: print(i, '%-70s %8.3f ms  R %6.2f GB W %6.2f GB'%(d['name'],t,d.get('dram__bytes_read.sum',0)/1e9,d.get('dram__bytes_write.sum',0)/1e9))
PY
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_2308_00106_b200 import synth
A = synth.rmat(24, 22, cap=1024)
L = (A.d_row_ptr[1:] - A.d_row_ptr[:-1]).long()
for lo, hi in [(0,32),(33,256),(257,512),(513,1024),(1025,1<<30)]:
    m = (L >= lo) & (L <= hi)
    print(f"rows {lo}..{hi}: {int(m.sum()):,} rows, {int(L[m].sum()):,} nnz")
PY
