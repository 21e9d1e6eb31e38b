"""Run one stage of the hot path once (for ncu / compute-sanitizer captures).

    python tools/prof_stage.py --config cfg5 --stage init|lloyd|hist|map|sweep [--repeat N]

`sweep` runs Lloyd once, then the isolated dense sweep (cqg_bench_sweep, one
warm-up + one timed launch) on its final state: capture with -s 1 -c 1.

Builds the histogram (and init centres for the later stages) first, then runs
the requested stage `repeat` times through the C-ABI.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1101_0395_b200 import cabi, quant  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--stage", default="init")
    ap.add_argument("--repeat", type=int, default=1)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    ctx = cabi.Context(0)
    hist = quant.build_histogram(img, ctx=ctx)
    k = cfg.k
    sc = quant.SeedConfig(k=k, seed=cfg.seed)
    initf = quant.init_kmeanspp if cfg.init == "kpp" else quant.init_maximin
    init = initf(hist, sc, ctx=ctx) if args.stage != "init" else None
    opts = quant.ClusterOptions(quant.Termination(fixed_iterations=cfg.fixed_iterations or None))
    t0 = time.perf_counter()
    for _ in range(args.repeat):
        if args.stage == "init":
            initf(hist, sc, ctx=ctx)
        elif args.stage == "lloyd":
            quant.wsm_hist(hist, init, opts, ctx=ctx)
        elif args.stage == "hist":
            quant.build_histogram(img, ctx=ctx)
        elif args.stage == "map":
            quant.map_pixels(img, init, ctx=ctx)
        elif args.stage == "sweep":
            st = quant.wsm_hist(hist, init, opts, ctx=ctx)
            ctx.bench_sweep(1)
            print(f"lloyd iterations={st.iterations}")
    dt = (time.perf_counter() - t0) / args.repeat
    print(f"{args.config} {args.stage}: N'={hist.size()} {dt * 1e3:.3f} ms/call")


if __name__ == "__main__":
    main()
