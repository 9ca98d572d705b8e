"""Per-source-line shared-memory wavefronts (total / ideal / excessive) of one
ncu report launch.  usage: python tools/ncu_smem.py REPORT"""
import csv, io, subprocess, sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, fname, rows = None, None, []
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] and r[0] != "Function Name":
        d = dict(zip(hdr[2:], r[2:]))
        try:
            wf = int(d["L1 Wavefronts Shared"]); ex = int(d["L1 Wavefronts Shared Excessive"])
            ideal = int(d["L1 Wavefronts Shared Ideal"]); smp = int(d["# Samples"])
        except (KeyError, ValueError):
            continue
        rows.append((wf, ideal, ex, smp, fname, r[0], r[1].strip()[:80]))
tw = sum(x[0] for x in rows) or 1
print("total shared wavefronts", tw, "excessive", sum(x[2] for x in rows))
for wf, ideal, ex, smp, f, ln, s in sorted(rows, reverse=True)[:25]:
    if wf:
        print("%5.1f%%  wf %9d ideal %9d excess %9d  %s:%s  %s" % (100 * wf / tw, wf, ideal, ex, f, ln, s))
