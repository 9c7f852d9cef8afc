"""Per-launch DRAM traffic and warp instructions of the bench's kernel groups
from an `ncu --set full` report of one step -> profiles/ncu_traffic.json and
profiles/ncu_instr.json [workload][group]."""
import collections, csv, io, json, os, subprocess, sys

rep, workload = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name"); ri = hdr.index("dram__bytes_read.sum"); wi = hdr.index("dram__bytes_write.sum")
ii = hdr.index("smsp__inst_executed.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
groups = {"accumulate": ["k_prep", "Radix", "k_scatter", "k_runsort", "k_longsort", "k_reduce", "Scan"],
          "pool": ["k_box_y", "k_box_x", "k_pool_count"], "gather_mlp": ["k_gather_mlp"]}
traffic = collections.defaultdict(float)
instr = collections.defaultdict(float)
for r in rows[2:]:
    name = r[ki]
    for g, keys in groups.items():
        if any(k in name for k in keys):
            traffic[g] += float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
            instr[g] += float(r[ii].replace(",", ""))
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
for fname, data in (("ncu_traffic.json", traffic), ("ncu_instr.json", instr)):
    path = os.path.join(root, fname)
    allv = json.load(open(path)) if os.path.exists(path) else {}
    allv[workload] = dict(data)
    json.dump(allv, open(path, "w"), indent=1)
print(workload, "traffic MB", {k: round(v / 1e6, 1) for k, v in traffic.items()},
      "warp-instr M", {k: round(v / 1e6, 1) for k, v in instr.items()})
