# per-kernel DRAM bytes in the steady state (no cache flush between kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/${NAME:-warm}.csv python tools/iter_driver.py --reps 3 --config ${CFG:-3d_1m} > gpurun_out/${NAME:-warm}.log 2>&1
python - <<'PY'
import csv,os,collections
name=os.environ.get('NAME','warm')
rows=list(csv.reader(open(f'gpurun_out/{name}.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[i]; d=collections.defaultdict(dict)
for r in rows[i+1:]:
    if len(r)<len(hdr): continue
    rec=dict(zip(hdr,r)); d[(int(rec['ID']),rec['Kernel Name'][:40])][rec['Metric Name']]=rec['Metric Value']
for (id_,k),m in sorted(d.items())[-16:]:
    print(id_,k.ljust(40),{a.split('__')[1][:18]:m[a] for a in m})
PY
