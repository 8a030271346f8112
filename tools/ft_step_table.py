"""Per-kernel table of one fine-tune step (dev tool) from an ncu launch list of
tools/ft_steps.py (gpu__time_duration + dram bytes, --clock-control none):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file L.csv python tools/ft_steps.py 4
    python tools/ft_step_table.py L.csv > profiles/<tag>_finetune_kernels.json"""
import csv, collections, json, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); ii=h.index('ID'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
sc={'nsecond':1e-3,'ns':1e-3,'usecond':1,'us':1,'msecond':1e3,'ms':1e3,'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
per=collections.OrderedDict()
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    d=per.setdefault(r[ii],{'k':r[ki]})
    d[r[mi]]=float(r[vi].replace(',',''))*sc.get(r[ui],1)
L=list(per.values())
idx=[j for j,d in enumerate(L) if 'k_composite_bwd' in d['k']]
a,b=idx[-2]+1, idx[-1]+1   # one full step: from after the previous backward to this one
agg=collections.OrderedDict()
for d in L[a:b]:
    name=d['k'].split('(')[0].replace('void ','').replace('g6r::','')
    x=agg.setdefault(name,[0,0.0,0.0]); x[0]+=1; x[1]+=d.get('gpu__time_duration.sum',0); x[2]+=d.get('dram__bytes_read.sum',0)+d.get('dram__bytes_write.sum',0)
tot=sum(v[1] for v in agg.values())
out={"note":"one DeviceTrainer.step on the 1M-Gaussian scene at 512x512 (tools/ft_steps.py), ncu --clock-control none launch list: serialised, cold-cache per-launch durations; shares, not absolute wall time","total_us":round(tot,1),"kernels":[]}
for k,(n,us,by) in sorted(agg.items(), key=lambda x:-x[1][1]):
    out["kernels"].append({"kernel":k,"launches":n,"us":round(us,1),"share":round(us/tot,3),"dram_MB":round(by/1e6,1)})
print(json.dumps(out,indent=1))
