"""How much of the concurrent cfg2 batch's time is the 16-CTA cluster initialiser's gang scheduling?
The batch with the k-means++ centres given (no initialiser kernels) next to the full one. (design tool, GPU)
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import CONFIGS

W, B, N = 8, 32, 16
cfg = CONFIGS["cfg2"]
img = cfg.image()
P = img.shape[0] * img.shape[1]
dev = torch.device("cuda", 0)
c0 = cabi.Context(0)
hist = quant.build_histogram(img, ctx=c0)
init = np.ascontiguousarray(quant.init_kmeanspp(hist, quant.SeedConfig(k=cfg.k, seed=cfg.seed), ctx=c0), np.float64)
d_init = torch.from_numpy(init.reshape(-1, 3)).to(dev)
ctxs = []
for w in range(W):
    c = cabi.Context(0)
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    c.set_sm_budget(B)
    ctxs.append((c, np.zeros(128)))
bufs = [(torch.from_numpy(img).to(dev), torch.empty(P, dtype=torch.int32, device=dev),
         torch.empty((P, 3), dtype=torch.uint8, device=dev), torch.empty((cfg.k, 3), dtype=torch.float64, device=dev))
        for _ in range(N)]
pool = ThreadPoolExecutor(W)
for name, kind, ini in [("k-means++ on the device", cabi.INIT_KMEANSPP, None), ("centres given", cabi.INIT_GIVEN, d_init)]:
    qc = cabi.QuantizeCfg(kind, cfg.k, cfg.seed, cabi.Term(1e-3, 100, 0, 0), 4)

    def work(w):
        c, sse = ctxs[w]
        for i in range(w, N, W):
            c.quantize_raw(bufs[i][0], P, qc, ini, bufs[i][3], None, sse, bufs[i][1], bufs[i][2])

    ws = []
    for rep in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        list(pool.map(work, range(W)))
        torch.cuda.synchronize()
        ws.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:24s}: {np.median(ws[3:]):.3f} ms per batch of {N} ({np.median(ws[3:]) / N:.3f} ms per image)", flush=True)
