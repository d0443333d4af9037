cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/bench_toynet.py --n ${N:-65536} --reps 3 > gpurun_out/toynet_bench.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/toynet_launches.csv python tools/bench_toynet.py --n ${N:-65536} --reps 0 > /dev/null 2>&1
cat gpurun_out/toynet_bench.json
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/toynet_launches.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[i]; kn=hdr.index('Kernel Name'); mv=hdr.index('Metric Value')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[i+1:]:
    if len(r)<=mv: continue
    name=r[kn].split('(')[0][:60]; agg[name][0]+=1; agg[name][1]+=float(r[mv].replace(',',''))
tot=sum(v[1] for v in agg.values())
print('total us', tot/1e3)
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:25]: print(f"{v[1]/1e3:9.1f} us {v[0]:5d}x {k}")
PY
