import csv, sys, subprocess, collections
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; agg = collections.Counter(); src = {}; stall = collections.defaultdict(collections.Counter); hdr = None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] in ("Function Name",) or not r[0]: continue
    try: ln = int(r[0])
    except ValueError: continue
    try: smp = float(r[4] or 0)
    except ValueError: smp = 0
    if smp:
        agg[(cur, ln)] += smp; src[(cur, ln)] = r[1].strip()[:100]
        for ci, name in enumerate(hdr):
            if name.startswith("stall_") and "Not Issued" not in name:
                try: v = float(r[ci] or 0)
                except ValueError: v = 0
                if v: stall[(cur, ln)][name[6:]] += v
tot = sum(agg.values())
print(f"total samples {tot:.0f}")
for (f, ln), s in agg.most_common(n):
    top = ", ".join(f"{k}:{int(v)}" for k, v in stall[(f, ln)].most_common(3))
    print(f"{100*s/tot:5.1f}% {f}:{ln}  {src[(f, ln)]}  [{top}]")
