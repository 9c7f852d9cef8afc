"""Per-launch-sequence roofline inputs from a `tools/gpu_metrics.sh` capture.

    python tools/ncu_roofline.py gpurun_out/metrics_<tag>_<wl>.csv <wl> [--write]

Splits the launch list into launch sequences (one per `k_prep*` launch), keeps
the last 5 (the bench's profiled calls, one launch sequence each), and sums
per kernel group: DRAM bytes, warp instructions, FMA / ALU / XU / tensor-pipe
instructions, duration; tensor-pipe activity of the MLP kernel.  With
--write the results go to profiles/ncu_traffic.json, ncu_instr.json and
ncu_pipes.json under the workload's key (read by bench.py's roofline).
"""
import csv
import io
import json
import os
import sys

GROUPS = {
    "accumulate": ("k_prep", "Scan", "k_scatter", "k_runsort", "k_longsort", "Onesweep", "Histogram", "k_reduce",
                   "k_order", "k_bin", "k_rank"),
    "pool": ("k_box", "k_pool_count"),
    "gather_mlp": ("k_gather_mlp", "k_features", "k_mlp_ffma"),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6,
         "Ginst": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "hz": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "": 1, "%": 1,
         "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "Kcycle/second": 1e3,
         "Mcycle/second": 1e6, "Gcycle/second": 1e9}


def load(path):
    with open(path) as fh:
        txt = fh.read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr, units = rows[0], rows[1]

    def val(r, name):
        if name not in hdr:
            return 0.0
        j = hdr.index(name)
        s = r[j].replace(",", "")
        try:
            return float(s) * SCALE.get(units[j], 1)
        except ValueError:
            return 0.0
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        out.append((r[hdr.index("Kernel Name")], lambda name, r=r: val(r, name)))
    return out


def group_of(name):
    for g, keys in GROUPS.items():
        if any(k in name for k in keys):
            return g
    return None


def analyse(path, keep=5):
    ks = load(path)
    seqs = []
    for name, v in ks:
        if name.startswith("vkm::k_prep") or "k_prep" in name.split("(")[0]:
            seqs.append([])
        if seqs:
            seqs[-1].append((name, v))
    seqs = seqs[-keep:]
    res = {g: {"dram_bytes": 0.0, "warp_instr": 0.0, "fma_instr": 0.0, "alu_instr": 0.0, "xu_instr": 0.0,
               "tc_instr": 0.0, "ms_serialised": 0.0, "fmaheavy_pct": 0.0, "alu_pct": 0.0, "issue_pct": 0.0}
           for g in GROUPS}
    tensor = []
    for seq in seqs:
        for name, v in seq:
            g = group_of(name)
            if g is None:
                continue
            r = res[g]
            r["dram_bytes"] += v("dram__bytes_read.sum") + v("dram__bytes_write.sum")
            r["warp_instr"] += v("smsp__inst_executed.sum")
            r["fma_instr"] += v("sm__inst_executed_pipe_fma.sum")
            r["alu_instr"] += v("sm__inst_executed_pipe_alu.sum")
            r["xu_instr"] += v("sm__inst_executed_pipe_xu.sum")
            r["tc_instr"] += v("sm__inst_executed_pipe_tc.sum")
            ms = v("gpu__time_duration.sum") * 1e3
            r["ms_serialised"] += ms
            # duration-weighted pipe activity (normalised below)
            r["fmaheavy_pct"] += ms * v("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active")
            r["alu_pct"] += ms * v("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active")
            r["issue_pct"] += ms * v("smsp__issue_active.avg.pct_of_peak_sustained_active")
            if "k_gather_mlp" in name:
                tensor.append((v("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                               v("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"),
                               v("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                               v("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                               v("gpu__time_duration.sum") * 1e3))
    n = max(1, len(seqs))
    for r in res.values():
        for k in ("fmaheavy_pct", "alu_pct", "issue_pct"):
            r[k] = r[k] / r["ms_serialised"] if r["ms_serialised"] > 0 else 0.0
        for k in r:
            if not k.endswith("_pct"):
                r[k] /= n
    if tensor:
        m = len(tensor)
        res["gather_mlp"]["tensor_pipe_pct"] = sum(t[0] for t in tensor) / m
        res["gather_mlp"]["tensor_hmma_pct"] = sum(t[1] for t in tensor) / m
        res["gather_mlp"]["fma_pipe_pct"] = sum(t[2] for t in tensor) / m
        res["gather_mlp"]["mlp_issue_pct"] = sum(t[3] for t in tensor) / m
    per_kernel = {}
    for seq in seqs:
        for name, v in seq:
            short = name.split("(")[0].replace("void ", "")[:60]
            d = per_kernel.setdefault(short, {"n": 0, "us": 0.0, "dram_mb": 0.0, "minstr": 0.0, "fma_pct": 0.0,
                                              "alu_pct": 0.0, "fmaheavy_pct": 0.0, "issue_pct": 0.0, "warps_pct": 0.0, "tensor_pct": 0.0})
            d["n"] += 1
            d["us"] += v("gpu__time_duration.sum") * 1e6
            d["dram_mb"] += (v("dram__bytes_read.sum") + v("dram__bytes_write.sum")) / 1e6
            d["minstr"] += v("smsp__inst_executed.sum") / 1e6
            d["fma_pct"] += v("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")
            d["alu_pct"] += v("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active")
            d["fmaheavy_pct"] += v("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active")
            d["issue_pct"] += v("smsp__issue_active.avg.pct_of_peak_sustained_active")
            d["warps_pct"] += v("sm__warps_active.avg.pct_of_peak_sustained_active")
            d["tensor_pct"] += v("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    for d in per_kernel.values():
        for k in list(d):
            if k != "n":
                d[k] = round(d[k] / d["n"], 3)
    return res, per_kernel, len(seqs)


def main():
    path, wl = sys.argv[1], sys.argv[2]
    res, per_kernel, nseq = analyse(path)
    print(f"{wl}: {nseq} launch sequences")
    for k, d in per_kernel.items():
        print(f"  {k:60s} n/seq={d['n'] / max(1, nseq):.1f} {d['us']:9.1f} us  dram {d['dram_mb']:8.1f} MB  "
              f"{d['minstr']:7.2f} Minstr  fma {d['fma_pct']:5.1f}% (heavy {d['fmaheavy_pct']:5.1f}%)  alu {d['alu_pct']:5.1f}%  issue "
              f"{d['issue_pct']:5.1f}%  warps {d['warps_pct']:5.1f}%  tensor {d['tensor_pct']:5.1f}%")
    for g, r in res.items():
        print(f"  [{g}] " + " ".join(f"{k}={v:.4g}" for k, v in r.items()))
    if "--write" in sys.argv:
        root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
        for fname, pick in (("ncu_traffic.json", lambda r: r["dram_bytes"]),
                            ("ncu_instr.json", lambda r: r["warp_instr"]),
                            ("ncu_pipes.json", lambda r: {k: v for k, v in r.items()})):
            p = os.path.join(root, fname)
            data = json.load(open(p)) if os.path.exists(p) else {}
            data[wl] = {g: pick(r) for g, r in res.items()}
            with open(p, "w") as fh:
                json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
