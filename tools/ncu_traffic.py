"""DRAM traffic per launch of the kernels in ncu reports -> JSON {name: {dram_bytes_read, dram_bytes_write,
duration_ns}} (the `traffic` field of bench.py's roofline).  usage: ncu_traffic.py out.json name=rep ..."""
import csv, io, json, subprocess, sys
out = {}
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def num(k):
        v = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
                 "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(u[k], 1)
        return v * scale
    out[name] = {"kernel": d.get("Kernel Name", "")[:80], "dram_bytes_read": num("dram__bytes_read.sum"),
                 "dram_bytes_write": num("dram__bytes_write.sum"), "duration_ns": num("gpu__time_duration.sum")}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out))
