"""Regenerate the committed golden fixtures from the reference itself.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_golden.py

Produces, under tests/golden/:
  acc_61.rgb, acc_62.rgb   40x40 images from the reference fixture generator
                           testsup::synthetic_photo (tests/test_support.hpp:30-89),
                           the inputs of proj/tmp_acceptance/sweep_a.csv.
  sweep_a_rows.csv         the 12 reference rows for (wsm-kpp, wsm-wu, wu) x K=8 x
                           seeds 3,4, produced by the reference run_quantize and
                           asserted byte-identical to proj/tmp_acceptance/sweep_a.csv:2-13.
  wu_init.json             the Wu palettes (precluster.cpp:579-639, out of scope for
                           the product) that seed the wsm-wu rows.
  ref_cases.json           small reference wsm / map_pixels results (centres, SSE
                           trace as hex floats, labels, NDC) for oracle pinning
                           when oracle/_ref is not available.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import RefLib, build  # noqa: E402

SWEEP_A = "/root/reference/proj/tmp_acceptance/sweep_a.csv"


def main() -> None:
    build()
    R = RefLib()
    rows = []
    wu = {}
    for img_seed in (61, 62):
        img = R.synthetic_photo(40, 40, img_seed)
        img.tofile(os.path.join(HERE, f"acc_{img_seed}.rgb"))
        colors, counts, _ = R.histogram(img, 3)
        wu[str(img_seed)] = R.init("wu", colors, counts, 1600, 8, 3).tolist()
        for method in ("wsm-kpp", "wsm-wu", "wu"):
            for run in (0, 1):
                r = R.run_quantize(img, 40, 40, method, 8, 3 + run, name=f"acc_{img_seed}.ppm",
                                   run=run)
                rows.append(r["csv_row"])
    rows.sort()
    header = ("image,method,k,run,seed,sampling,mse,psnr,iterations,ndc_per_point_iter,"
              "time_ms,actual_k,flags")
    text = header + "\n" + "\n".join(rows) + "\n"
    if os.path.exists(SWEEP_A):
        with open(SWEEP_A) as f:
            want = f.read()
        assert text == want, "reference run_quantize no longer reproduces sweep_a.csv"
        print("sweep_a.csv reproduced byte-identically")
    with open(os.path.join(HERE, "sweep_a_rows.csv"), "w") as f:
        f.write(text)
    with open(os.path.join(HERE, "wu_init.json"), "w") as f:
        json.dump(wu, f, indent=1)
    with open(os.path.join(HERE, "wu_init.txt"), "w") as f:  # for tests/cpp/test_dropin.cpp
        for key in ("61", "62"):
            for r, g, b in wu[key]:
                f.write(f"{r!r} {g!r} {b!r}\n")

    # small reference wsm / map cases for oracle pinning
    cases = []
    for (img_seed, K, kind, seed) in [(61, 8, "kpp", 3), (62, 8, "mmx", 4), (61, 16, "kpp", 9)]:
        img = R.synthetic_photo(40, 40, img_seed)
        colors, counts, _ = R.histogram(img, seed)
        init = R.init(kind, colors, counts, 1600, K, seed)
        res = R.wsm(colors, counts, 1600, init, history=True)
        idx, q, mse, mndc = R.map_pixels(img, 40, 40, res.centers)
        cases.append(dict(
            image=img_seed, k=K, init=kind, seed=seed,
            n_unique=int(colors.size),
            hist_colors=colors.tolist(), hist_counts=counts.tolist(),
            init_centers=[float(v).hex() for v in init.reshape(-1)],
            centers=[float(v).hex() for v in res.centers.reshape(-1)],
            sse_trace=[float(v).hex() for v in res.sse_trace],
            iterations=res.iterations, ndc_total=res.ndc_total, repairs=res.repairs,
            labels=res.labels.tolist(),
            history_labels=res.hist_labels.tolist(),
            map_indices=idx.tolist(), map_mse=float(mse).hex(), map_ndc=int(mndc),
        ))
    with open(os.path.join(HERE, "ref_cases.json"), "w") as f:
        json.dump(cases, f)
    print("wrote", len(rows), "rows and", len(cases), "ref cases")


if __name__ == "__main__":
    main()
