"""Summarise an ncu report: stall reasons + hottest source lines of one launch.
usage: python tools/ncu_src.py REPORT [launch_index]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, r = rows[0], rows[2 + li]
vals = dict(zip(hdr, r))
st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for h, v in vals.items()
      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v}
tot = sum(st.values()) or 1
print("stalls:", ", ".join("%s %.0f%%" % (k, 100 * v / tot) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]))
for h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
          "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
    if h in vals:
        print(h, vals[h])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(li), "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
fname = None
seen = set()
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    key = (r[0], r[2])
    if key in seen:
        continue
    seen.add(key)
    try:
        s, i = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg[(fname, r[0])]
    a[0] += s
    a[1] += i
    if r[1].strip():
        a[2] = r[1].strip()[:90]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print("samples", ts, "inst", ti)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print("%5.1f%% %5.1f%%  %s:%s  %s" % (100 * v[0] / ts, 100 * v[1] / ti, k[0], k[1], v[2]))
