# per-kernel durations of one 512^3 transport RHS, this tree and round 1's
for d in . build/r1; do
  (cd $d && ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/transport_once.py 2>/dev/null) | python3 -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and r[12]=='gpu__time_duration.sum']
half=len(rows)//2
agg={}
for r in rows[half:]:
    k=r[4].split('(')[0]; agg.setdefault(k,[]).append(float(r[14].replace(',',''))/1e3)
tot=sum(sum(v) for v in agg.values())
print('$d total_us', round(tot,1))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])): print('  ', k, len(v), [round(x,1) for x in v])
"
done
