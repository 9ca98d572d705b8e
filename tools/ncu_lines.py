"""Per-source-line shared-memory wavefronts, instructions and stall samples of
one kernel in an ncu report (--set full --import-source on).
usage: python tools/ncu_lines.py REPORT [records]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nrec = float(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
          "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
          "smsp__issue_active.avg.pct_of_peak_sustained_active"):
    print(k, d.get(k))
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "")) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v}
tot = sum(st.values()) or 1
print("stalls:", ", ".join("%s %.0f%%" % (k, 100 * v / tot) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.OrderedDict()
hdr = None
fname = None
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0] or r[2] not in ("-", ""):
        continue
    m = dict(zip(hdr[4:], r[4:]))

    def f(k):
        try:
            return float(m.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    agg[(fname, r[0], r[1][:90])] = (f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal"),
                                     f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"))
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[2] for v in agg.values()) or 1
ts = sum(v[3] for v in agg.values()) or 1
if nrec:
    print("per record: %.3f shared wavefronts, %.3f warp instructions" % (tw / nrec, ti / nrec))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:24]:
    print("%5.1f%% wf (x%.2f ideal) %5.1f%% inst %5.1f%% stall  %s:%s %s" % (
        100 * v[0] / tw, v[0] / max(v[1], 1), 100 * v[2] / ti, 100 * v[3] / ts, k[0], k[1], k[2].strip()))
print("--- by instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:20]:
    print("%5.1f%% inst %5.1f%% wf %5.1f%% stall  %s:%s %s" % (
        100 * v[2] / ti, 100 * v[0] / tw, 100 * v[3] / ts, k[0], k[1], k[2].strip()))
