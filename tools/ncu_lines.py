"""Aggregate ncu source-page stall samples per CUDA source line (file:line)."""
import csv, sys, subprocess, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = collections.Counter(); stalls = collections.defaultdict(collections.Counter)
cur_file = None; hdr = None; src_line = {}
for row in csv.reader(out):
    if not row: continue
    if row[0] == "File Path": cur_file = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or len(row) < 6: continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    if row[1].strip():
        src_line[(cur_file, ln)] = row[1].strip()
    try: s = int(row[4])
    except ValueError: continue
    key = (cur_file, ln)
    agg[key] += s
    for i, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try: stalls[key][name] += int(row[i])
            except (ValueError, IndexError): pass
tot = sum(agg.values())
print("total samples", tot)
for (f, ln), s in agg.most_common(top):
    st = ", ".join(f"{k[6:]}={v}" for k, v in stalls[(f, ln)].most_common(3) if v)
    print(f"{s:7d} {100*s/tot:5.1f}%  {f}:{ln}  [{st}]  {src_line.get((f, ln), '')[:70]}")
