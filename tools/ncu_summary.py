"""Summarise ncu outputs into the text files committed under profiles/.

    python tools/ncu_summary.py launches <launches.csv> > profiles/rNN_launches_<cfg>.txt
    python tools/ncu_summary.py full <report.ncu-rep> [kernel-regex] > profiles/rNN_full_<kernel>.txt

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list per
kernel (count, total/avg us, share of all profiled device time).
`full` prints the key metrics of a `--set full` capture: duration, DRAM bytes
read/written (the roofline `traffic`), throughput, IPC, occupancy, pipe
utilisation and the top stall reasons.
"""
import collections
import csv
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("cqg::", "").replace("<unnamed>::", "")
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", ""))
            v_us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
            c, t = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, t + v_us)
    tot = sum(t for _, t in agg.values())
    print(f"# ncu launch list: {path}")
    print(f"# {sum(c for c, _ in agg.values())} launches, {tot:.1f} us total profiled device time")
    print(f"{'kernel':60s} {'count':>6s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {c:6d} {t:10.1f} {t / c:9.2f} {100 * t / tot:5.1f}%")


WANT = [
    "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
    "Compute (SM) Throughput", "Issued Ipc Active", "Issue Slots Busy", "Executed Instructions",
    "Registers Per Thread", "Grid Size", "Block Size", "Theoretical Occupancy", "Achieved Occupancy",
    "L1/TEX Hit Rate", "L2 Hit Rate", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def full(path, kregex=None):
    args = ["ncu", "-i", path, "--page", "details", "--csv"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if kregex and not re.search(kregex, d["Kernel Name"]):
            continue
        key = (d["ID"], d["Kernel Name"])
        per.setdefault(key, {})
        if d["Metric Name"] in WANT:
            per[key][d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rhdr, runits = rr[0], rr[1]
    rawd = {}
    for r in rr[2:]:
        d = dict(zip(rhdr, r))
        rawd[d["ID"]] = {k: f"{d.get(k, '')} {u}".strip() for k, u in zip(rhdr, runits) if k in RAW}
    print(f"# ncu --set full capture: {path}")
    for (kid, kname), m in per.items():
        print(f"\n## [{kid}] {kname}")
        for k in WANT:
            if k in m:
                print(f"  {k:36s} {m[k]}")
        for k in RAW:
            if k in rawd.get(kid, {}):
                print(f"  {k:36s} {rawd[kid][k]}")
    # stall reasons from the source page (first kernel matching)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
                         + (["-k", "regex:" + kregex] if kregex else []), capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    idx = [i for i, r in enumerate(srows) if r and r[0] == "Address"]
    if idx:
        shdr = srows[idx[0]]
        end = idx[1] if len(idx) > 1 else len(srows)
        c = collections.Counter()
        for r in srows[idx[0] + 1:end]:
            if len(r) != len(shdr):
                continue
            d = dict(zip(shdr, r))
            for h in shdr:
                if h.startswith("stall_") and "Not Issued" not in h and d[h].isdigit():
                    c[h[6:]] += int(d[h])
        tot = sum(c.values()) or 1
        print("\n  stall reasons (all samples, first kernel):")
        for k, v in c.most_common(8):
            print(f"    {k:20s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
