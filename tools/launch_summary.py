import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size'); bi=h.index('Block Size')
agg=collections.defaultdict(lambda:[0,0.0])
tot=0
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',',''))
    n=r[ki].split('(')[0].split('<')[0]+' g='+r[gi].replace(', 1, 1)',')')+' b='+r[bi].replace(', 1, 1)',')')
    agg[n][0]+=1; agg[n][1]+=v; tot+=v
for n,(c,t) in sorted(agg.items(),key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]: print(f"{n[:52]:52s} {c:5d} {t/1e6:9.3f} ms {t/c/1e3:9.1f} us/l {t/tot*100:5.1f}%")
print('total',tot/1e6)
