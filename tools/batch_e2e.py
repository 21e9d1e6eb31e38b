"""Which host<->device copy costs the concurrent cfg2 batch its e2e time? (design tool, GPU)
Wall time of a batch of 16 through 8 contexts with host (pinned) or device buffers per argument.
"""
import os
import sys
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
dev = torch.device("cuda", 0)
qc = cabi.QuantizeCfg(cabi.INIT_KMEANSPP, cfg.k, cfg.seed, cabi.Term(1e-3, 100, 0, 0), 4)
ctxs = []
for w in range(W):
    c = cabi.Context(0)
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    c.set_sm_budget(B)
    ctxs.append((c, np.zeros(128)))
pool = ThreadPoolExecutor(W)


def mk(host, shape, dtype):
    t = torch.empty(shape, dtype=dtype)
    return t.pin_memory() if host else t.to(dev)


for name, h_in, h_idx, h_q, h_lab in [("all device", 0, 0, 0, None), ("host image", 1, 0, 0, None),
                                      ("host indices", 0, 1, 0, None), ("host rgb out", 0, 0, 1, None),
                                      ("host labels", 0, 0, 0, 1), ("device labels", 0, 0, 0, 0),
                                      ("host image+idx+rgb", 1, 1, 1, None), ("all host", 1, 1, 1, 1)]:
    src = [torch.from_numpy(img).pin_memory() if h_in else torch.from_numpy(img).to(dev) for _ in range(N)]
    idx = [mk(h_idx, P, torch.int32) for _ in range(N)]
    q = [mk(h_q, (P, 3), torch.uint8) for _ in range(N)]
    pal = [np.empty((cfg.k, 3)) if (h_in and h_idx) else torch.empty((cfg.k, 3), dtype=torch.float64, device=dev)
           for _ in range(N)]
    lab = [None if h_lab is None else mk(h_lab, P, torch.int32) for _ in range(N)]

    def work(w):
        c, sse = ctxs[w]
        for i in range(w, N, W):
            c.quantize_raw(src[i], P, qc, None, pal[i], lab[i], sse, idx[i], q[i])

    ws = []
    for rep in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        list(pool.map(work, range(W)))
        torch.cuda.synchronize()
        ws.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:22s}: {min(ws[2:]):.3f} ms per batch of {N} (median {np.median(ws[2:]):.3f})", flush=True)
