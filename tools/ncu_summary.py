"""Summarise an ncu launch list (csv) and a --set full report (.ncu-rep)."""
import csv, subprocess, sys, collections, io

def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        k = r[ki].split("(")[0].replace("void ", "")[:48]
        agg.setdefault(k, []).append(float(r[vi]) / 1e3)
    return agg

def full(path, kernels_filter=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]; units = rows[1]
    ki = hdr.index("Kernel Name")
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = r[ki].split("(")[0].replace("void ", "")[:40]
        st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v))
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        def g(m, scale=1.0):
            try: return float(d[m].replace(",", "")) * scale
            except Exception: return None
        res.append(dict(kernel=name, dur_us=g("gpu__time_duration.sum", 1e-3),
                        dram_rd_MB=g("dram__bytes_read.sum"), dram_wr_MB=g("dram__bytes_write.sum"),
                        dram_pct=g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                        sm_pct=g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                        tensor_pct=g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed") or g("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                        occ=g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                        regs=g("launch__registers_per_thread"),
                        stalls=[(a, round(b, 2)) for a, b in st[:4]],
                        units=dict(rd=units[hdr.index("dram__bytes_read.sum")], dur=units[hdr.index("gpu__time_duration.sum")])))
    return res

if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            for k, v in launches(p).items():
                print(f"{k:50s} n={len(v):3d} mean={sum(v)/len(v):9.2f} us")
        else:
            for r in full(p):
                print(r)
