"""Summarize ncu captures into profiles/ (run in the dev container).

    python tools/summarize_ncu.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --tag r01 --kernel k_fused_tma --traffic-key "k_fused_tma<15,6>@256x256x256"

Writes profiles/<tag>_<kernel>_ncu.md (key metrics + stall reasons of the
--set full capture), profiles/<tag>_launches.md (per-kernel share of the
bench command's launch list) and updates profiles/traffic.json with the
measured DRAM bytes per launch that bench.py reports as roofline.traffic.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("sm__cycles_elapsed.max", "SM cycles elapsed"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts (LSU: LDS/STS)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-memory load wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "shared-memory store wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "L1 data-pipe LSU wavefronts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/TEX throughput % of peak"),
    ("l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed", "LSU writeback % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, r = rows[0], rows[2]
    res = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                res.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "")
                            .replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    return sorted(res, reverse=True)[:8]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--kernel", default="k_fused_tma")
    ap.add_argument("--traffic-key", default=None, help="kernel<..>@NXxNYxNZ (bench.py looks it up per grid)")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.rep:
        hdr, units, rows = raw(a.rep)
        r = rows[0]
        name = r[hdr.index("Kernel Name")]
        lines = ["# %s — ncu --set full (%s)" % (name, a.tag), "",
                 "Capture: `ncu --set full --clock-control none --import-source on` of one launch "
                 "(cold L2, serialised; compare shares, not absolutes).", ""]
        if a.note:
            lines += [a.note, ""]
        lines += ["| metric | value | unit |", "|---|---|---|"]
        vals = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                vals[key] = r[i]
                lines.append("| %s (`%s`) | %s | %s |" % (label, key, r[i], units[i]))
        rd = float(vals.get("dram__bytes_read.sum", "nan"))
        wr = float(vals.get("dram__bytes_write.sum", "nan"))
        unit = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        traffic = (rd + wr) * scale
        if a.algorithmic_bytes:
            lines += ["", "DRAM traffic per launch: %.3f GB; algorithmic %.3f GB; ratio %.3f"
                      % (traffic / 1e9, a.algorithmic_bytes / 1e9, traffic / a.algorithmic_bytes)]
        st = stalls(a.rep)
        if st:
            lines += ["", "Top warp stall reasons (warps stalled per issued instruction):", ""]
            lines += ["| stall | cycles |", "|---|---|"] + ["| %s | %.2f |" % (n, v) for v, n in st]
        fn = os.path.join(PROF, "%s_%s_ncu.md" % (a.tag, a.kernel))
        open(fn, "w").write("\n".join(lines) + "\n")
        print("wrote", fn)
        if a.traffic_key:
            tp = os.path.join(PROF, "traffic.json")
            tj = json.load(open(tp)) if os.path.exists(tp) else {}
            tj[a.traffic_key] = round(traffic)
            json.dump(tj, open(tp, "w"), indent=1)
    if a.launches:
        text = open(a.launches).read()
        start = text.find('"ID"')
        rows = list(csv.DictReader(io.StringIO(text[start:])))
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for row in rows:
            if row.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = row["Kernel Name"].split("(")[0]
            v = float(row["Metric Value"].replace(",", ""))
            mult = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}[row["Metric Unit"]]
            tot[k] += v * mult
            cnt[k] += 1
        all_t = sum(tot.values())
        lines = ["# launch list (%s): `ncu --metrics gpu__time_duration.sum --clock-control none`" % a.tag,
                 "", "Per-launch times are cold-cache and serialised; the SHARE is what matters.", "",
                 "| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
        for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append("| `%s` | %d | %.3f | %.4f | %.1f%% |" % (k, cnt[k], t * 1e3, t * 1e3 / cnt[k],
                                                               100 * t / all_t))
        fn = os.path.join(PROF, "%s_launches.md" % a.tag)
        open(fn, "w").write("\n".join(lines) + "\n")
        print("wrote", fn)


if __name__ == "__main__":
    main()
