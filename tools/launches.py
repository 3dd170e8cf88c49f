import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if r and r[0]=='ID')
hdr = rows[hdr_i]; data = rows[hdr_i+1:]
ci = {h:i for i,h in enumerate(hdr)}
k = collections.OrderedDict()
for r in data:
    if len(r) < len(hdr): continue
    kid=(int(r[ci['ID']]), r[ci['Kernel Name']][:55])
    k.setdefault(kid, {})[r[ci['Metric Name']]] = float(r[ci['Metric Value']].replace(',',''))
for (i,n),m in k.items():
    t = m.get('gpu__time_duration.sum',0); rd=m.get('dram__bytes_read.sum',0); wr=m.get('dram__bytes_write.sum',0)
    print(f"{i:4d} {n:55s} {t/1000:9.1f}us rd {rd/1e6:8.1f}MB wr {wr/1e6:8.1f}MB  {(rd+wr)/max(t,1):7.0f}GB/s")
