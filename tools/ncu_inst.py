"""Per CUDA source line: warp instructions executed, shared wavefronts (and excessive ones) from an
ncu source page (cuda,sass).  Usage: ncu_inst.py report.ncu-rep [top]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
inst = collections.Counter(); wf = collections.Counter(); wfx = collections.Counter(); src = {}
cur = None; hdr = None
for row in csv.reader(out):
    if not row: continue
    if row[0] == "File Path": cur = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or len(row) < 8: continue
    try: ln = int(row[0])
    except ValueError: continue
    if row[1].strip(): src[(cur, ln)] = row[1].strip()
    def col(name):
        try: return int(row[hdr.index(name)])
        except (ValueError, IndexError): return 0
    inst[(cur, ln)] += col("Instructions Executed")
    wf[(cur, ln)] += col("L1 Wavefronts Shared")
    wfx[(cur, ln)] += col("L1 Wavefronts Shared Excessive")
tot = sum(inst.values())
print(f"total warp instructions {tot}, shared wavefronts {sum(wf.values())} (excessive {sum(wfx.values())})")
for k, v in inst.most_common(top):
    print(f"{v:12d} {100*v/tot:5.1f}%  wf {wf[k]:11d} x {wfx[k]:10d}  {k[0]}:{k[1]}  {src.get(k, '')[:80]}")
