"""Do the stages of several library contexts overlap on the device? (design tool, GPU)
N host threads, one context each (SM budget b), run one stage R times; wall time vs N.

    python tools/coop_concurrency.py lloyd|init|hist|map budget n1 n2 ...
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import CONFIGS

stage, budget = sys.argv[1], int(sys.argv[2])
ns = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
cfg = CONFIGS["cfg2"]
img = cfg.image()
R = 20
for n in ns:
    ctxs, work = [], []
    for i in range(n):
        ctx = cabi.Context(0)
        s = torch.cuda.Stream()
        ctx.set_stream(s.cuda_stream)
        if budget:
            ctx.set_sm_budget(budget)
        hist = quant.build_histogram(img, ctx=ctx)
        sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
        init = quant.init_kmeanspp(hist, sc, ctx=ctx)
        opts = quant.ClusterOptions(quant.Termination())
        if stage == "lloyd":
            f = lambda ctx=ctx, hist=hist, init=init, opts=opts: quant.wsm_hist(hist, init, opts, ctx=ctx)
        elif stage == "init":
            f = lambda ctx=ctx, hist=hist, sc=sc: quant.init_kmeanspp(hist, sc, ctx=ctx)
        elif stage == "hist":
            f = lambda ctx=ctx: quant.build_histogram(img, ctx=ctx)
        else:
            f = lambda ctx=ctx, init=init: quant.map_pixels(img, init, ctx=ctx)
        f()
        ctxs.append((ctx, s))
        work.append(f)
    torch.cuda.synchronize()

    def run(f):
        for _ in range(R):
            f()
    ths = [threading.Thread(target=run, args=(f,)) for f in work]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    print(f"{stage} budget {budget} x{n}: {dt / R:.3f} ms per round of {n} ({dt / R / n:.3f} ms per call)", flush=True)
    for ctx, _ in ctxs:
        ctx.close()
