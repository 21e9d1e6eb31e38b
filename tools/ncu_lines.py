"""Per-source-line stall samples of one kernel in an ncu --set full capture.

    python tools/ncu_lines.py <report.ncu-rep> [top]

Reads `ncu --page source --print-source cuda,sass --csv` (needs a capture made
with --import-source on and a -lineinfo build) and prints the source lines
with the most warp-stall samples, with their share of all samples.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) >= 5 and r[0].isdigit():
            try:
                samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
                inst = int(r[hdr.index("Instructions Executed")] or 0)
            except ValueError:
                continue
            reasons = {h[6:]: int(r[j] or 0) for j, h in enumerate(hdr)
                       if h.startswith("stall_") and "Not Issued" not in h and r[j] not in ("", "-")}
            top_r = ",".join(f"{k}:{v}" for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:2] if v)
            rows.append((samples, inst, fname, int(r[0]), r[1].strip(), top_r))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(reverse=True)
    print(f"# {rep}: {tot} stall samples over {len(rows)} source lines")
    print(f"{'share':>6s} {'samples':>8s} {'warp_inst':>11s}  location / source")
    for s, i, f, ln, src, rs in rows[:top]:
        print(f"{100 * s / tot:5.1f}% {s:8d} {i:11d}  {f}:{ln} [{rs}]  {src[:80]}")


if __name__ == "__main__":
    main()
