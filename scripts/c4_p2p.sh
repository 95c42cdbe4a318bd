python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "p2p" > gpurun_out/pt.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pt.log
timeout 300 python bench.py --workload config4 --shard-mode p2p --steps 256 --warmup 8 > gpurun_out/c4_p2p.json 2> gpurun_out/c4_p2p.err; python -c "import json;d=json.load(open(\"gpurun_out/c4_p2p.json\"));print('p2p', round(d[\"ms_per_step\"]*1e3,2),\"us\",round(d[\"roofline\"][\"frac\"],3))"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|p2p" -c 30 --csv --log-file gpurun_out/launches_c4p2p.csv python bench.py --workload config4 --shard-mode p2p --steps 8 --warmup 3 --graph-steps 4 > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_c4p2p.csv')))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; data=rows[i+1:]; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in data:
    if len(r)==len(h): d[r[ki].split('(')[0].replace('void ','')].append(float(r[vi].replace(',','')))
for k,v in d.items(): print(k, len(v), round(sum(v)/len(v)/1e3,2),'us')
PY
