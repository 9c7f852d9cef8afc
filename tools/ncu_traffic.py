"""Per-launch DRAM traffic (dram__bytes_read + write) of the bench's kernel groups
from an `ncu --set full` report -> profiles/ncu_traffic.json[workload]."""
import csv, io, json, subprocess, sys, os, collections
rep, workload = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name"); ri = hdr.index("dram__bytes_read.sum"); wi = hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
groups = {"accumulate": ["k_prep", "Onesweep", "k_reduce", "Histogram", "Scan"], "pool": ["k_box_y", "k_box_x", "k_pool_count"],
          "gather_mlp": ["k_gather_mlp"]}
per = collections.defaultdict(list)
for r in rows[2:]:
    b = float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
    per[r[ki].split("(")[0].replace("void ", "")].append(b)
res = {}
for g, keys in groups.items():
    tot = 0.0
    for k, v in per.items():
        if any(x in k for x in keys):
            tot += sum(v) / len(v) * (3 if "Onesweep" in k else 1)   # three onesweep passes per launch group
    res[g] = tot
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[workload] = res
json.dump(data, open(path, "w"), indent=1)
print(workload, {k: round(v / 1e6, 1) for k, v in res.items()}, "MB per launch")
