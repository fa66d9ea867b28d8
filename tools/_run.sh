for fl in "--flush" ""; do echo "== stamps $fl"; TA_NO_EVENTS=1 python tools/step_times.py --phases --mini --decide-only $fl --ticks 60 2>&1 | python -c "
import sys,re,statistics
acc={}
cur=None
for l in sys.stdin:
    l=l.strip()
    m=re.match(r'(\w+)\s*:\s*(.*)',l)
    if not m or m.group(1) in ('tick','phases','spans'): continue
    nm=m.group(1)
    for i,v in re.findall(r'(\d+):([\d.]+)',m.group(2)):
        acc.setdefault((nm,int(i)),[]).append(float(v))
for (nm,i),v in sorted(acc.items()):
    if len(v)>20: print(nm,i,round(statistics.median(v),1))
"; done
