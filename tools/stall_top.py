"""Top warp-stall instructions of an ncu report (source page, SASS view):
    python tools/stall_top.py gpurun_out/x.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw = hdr.index("Warp Stall Sampling (All Samples)")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iw] or 0) for r in data)
agg = {}
for r in data:
    for i in cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print("samples", int(tot))
print(", ".join("%s %.1f%%" % (k[6:], 100 * v / tot) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
for j, r in sorted(enumerate(data), key=lambda x: -float(x[1][iw] or 0))[:n]:
    st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in cols), reverse=True)[:2]
    prev = data[j - 1][isrc].strip()[:40] if j else ""
    print("%s %5.2f%%  %-55s %s   <- %s" % (r[ia][-5:], 100 * float(r[iw]) / tot, r[isrc].strip()[:55],
                                           [(h, int(v)) for v, h in st if v > 0], prev))
