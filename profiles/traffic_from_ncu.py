"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
of kernels from an `ncu --set full` report into profiles/traffic.json, which
bench.py reports as roofline.traffic for the dominant kernel.

    python profiles/traffic_from_ncu.py gpurun_out/prof_X.ncu-rep [tag]"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(rep)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    rd = float(d["dram__bytes_read.sum"]) * scale[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(d["dram__bytes_write.sum"]) * scale[units[hdr.index("dram__bytes_write.sum")]]
    dur = d.get("gpu__time_duration.sum")
    db[name] = {"dram_bytes": int(rd + wr), "read": int(rd), "write": int(wr), "source": f"{tag}",
                "ncu_duration": dur}
    print(name, db[name])
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
