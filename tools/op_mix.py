"""Executed-instruction mix of an ncu report by SASS opcode (source page):
    python tools/op_mix.py gpurun_out/x.ncu-rep"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
isrc = hdr.index("Source"); ie = hdr.index("Instructions Executed"); iw = hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.Counter(); smp = collections.Counter()
for r in data:
    s = r[isrc].strip()
    if s.startswith("@"): s = s.split(None, 1)[1]
    op = s.split()[0] if s else "?"
    agg[op] += int(r[ie] or 0); smp[op] += float(r[iw] or 0)
tot = sum(agg.values()); ts = sum(smp.values())
for op, n in agg.most_common(40):
    print("%-28s %12d %5.1f%%  stall-samples %5.1f%%" % (op, n, 100*n/tot, 100*smp[op]/ts))
