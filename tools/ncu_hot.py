"""Top SASS lines by warp-stall samples for one kernel of an .ncu-rep."""
import csv, subprocess, sys, io, collections
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)"); src = hdr.index("Source"); ie = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try: data.append((int(r[si] or 0), r[src], int(r[ie] or 0)))
    except Exception: pass
tot = sum(d[0] for d in data) or 1
print("samples", tot, "warp-instrs", sum(d[2] for d in data))
for i, d in enumerate(data):
    pass
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:6d} {100*d[0]/tot:5.1f}% {d[2]:>9} {d[1][:100]}")
ops = collections.Counter()
for d in data:
    t = d[1].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += d[2]
print(ops.most_common(20))
