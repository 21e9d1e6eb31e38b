"""Experiment (GPU): does aligning the stages of the concurrent contexts help? 16 cfg2 images through
8 contexts with the staged C-ABI calls (histogram, init, Lloyd, map), free-running vs a thread barrier
between the stages. (design tool)
"""
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS

W, B, N = 8, 32, 16
cfg = CONFIGS["cfg2"]
img = cfg.image()
P = img.shape[0] * img.shape[1]
K = cfg.k
dev = torch.device("cuda", 0)
term = cabi.Term(1e-3, 100, 0, 0)
ctxs = []
for w in range(W):
    c = cabi.Context(0)
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    c.set_sm_budget(B)
    ctxs.append(c)


def mk():
    return dict(src=torch.from_numpy(img).to(dev), col=torch.empty(P, dtype=torch.int32, device=dev),
                cnt=torch.empty(P, dtype=torch.int32, device=dev), ini=torch.empty((K, 3), dtype=torch.float64, device=dev),
                cen=torch.empty((K, 3), dtype=torch.float64, device=dev), lab=torch.empty(P, dtype=torch.int32, device=dev),
                idx=torch.empty(P, dtype=torch.int32, device=dev), q=torch.empty((P, 3), dtype=torch.uint8, device=dev))


bufs = [mk() for _ in range(N)]
pool = ThreadPoolExecutor(W)
for name, sync in [("free-running", False), ("barrier between stages", True), ("free-running", False),
                   ("barrier between stages", True)]:
    bar = threading.Barrier(W)

    def work(w):
        c = ctxs[w]
        sse = np.zeros(128)
        for i in range(w, N, W):
            b = bufs[i]
            n = c.histogram_raw(b["src"], P, b["col"], b["cnt"])
            if sync:
                bar.wait()
            c.init_raw(cabi.INIT_KMEANSPP, b["col"], b["cnt"], n, P, K, cfg.seed, b["ini"])
            if sync:
                bar.wait()
            c.lloyd_raw(b["col"], b["cnt"], n, P, b["ini"], K, term, b["cen"], b["lab"], sse)
            if sync:
                bar.wait()
            c.map_raw(b["src"], P, b["cen"], K, b["idx"], 4, b["q"])
            if sync:
                bar.wait()

    ws = []
    for rep in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        list(pool.map(work, range(W)))
        torch.cuda.synchronize()
        ws.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:24s}: {np.median(ws[2:]):.3f} ms per batch of {N} (min {min(ws[2:]):.3f})", flush=True)
