import csv, sys, subprocess
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(lines[1:]))
h = rows[0]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source"); iE = h.index("Instructions Executed")
data = []
for r in rows[1:]:
    try: data.append((int(r[iS]), r[iSrc].strip(), int(r[iE]), r[0]))
    except: pass
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", sum(d[2] for d in data))
for i,(s,src,e,a) in enumerate(data):
    pass
for s, src, e, a in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{s:6d} {100*s/tot:5.1f}% {e:9d} {a[-5:]} {src[:90]}")
