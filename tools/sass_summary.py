"""Instruction-mnemonic summary of selected kernels in the built library
(cuobjdump -sass): proves the TMA bulk copies (UBLKCP), mbarrier ops (SYNCS),
asynchronous copies (LDGSTS) and shared-memory traffic of each kernel.
usage: python tools/sass_summary.py [lib.so] > profiles/r02/sass_summary.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2209_06909_b200/libpowersort_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and cur:
        funcs[cur][m.group(1) + (m.group(2) or "")] += 1
want = ("merge_pipe_kernel", "xs_merge_kernel", "merge_tiny_kernel", "form_leaves_kernel", "rd_types_kernel")
keys = ("UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "LDG", "STG", "BAR", "SHFL", "VOTE", "total")
print("# cuobjdump -sass %s (sm_100a); counts of static SASS instructions per kernel" % lib)
for f, c in funcs.items():
    if not any(w in f for w in want):
        continue
    agg = collections.Counter()
    for op, n in c.items():
        for k in keys[:-1]:
            if op == k or op.startswith(k + "."):
                agg[k] += n
        agg["total"] += n
    detail = sorted((op for op in c if op.split(".")[0] in ("UBLKCP", "SYNCS", "LDGSTS")), key=lambda o: -c[o])
    print("%s\n  %s\n  %s" % (f, "  ".join("%s=%d" % (k, agg[k]) for k in keys),
                             "  ".join("%s x%d" % (o, c[o]) for o in detail)))
