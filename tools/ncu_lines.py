"""Per-CUDA-source-line warp-stall samples of one kernel (ncu --page source --print-source cuda,sass).
usage: python tools/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import csv, collections, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samples, ie, src, stalls = collections.Counter(), collections.Counter(), {}, collections.defaultdict(collections.Counter)
fname, hdr, cur = "?", None, None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) - 5: continue
    if r[0]: cur = (fname, int(r[0])); src[cur] = r[1]; continue
    try: s = int(r[4] or 0); n = int(r[7] or 0)
    except ValueError: continue
    samples[cur] += s; ie[cur] += n
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("", "-", "0"):
            try: stalls[cur][h[6:]] += int(r[i])
            except ValueError: pass
tot = sum(samples.values()) or 1
print("samples", tot, "instructions", sum(ie.values()))
for k, s in samples.most_common(top):
    st = ",".join(f"{a}:{b}" for a, b in stalls[k].most_common(3))
    print(f"{k[0][:14]:14s}:{k[1]:<4d} {100*s/tot:5.1f}% ie={ie[k]:>9} [{st}] {src[k].strip()[:70]}")
