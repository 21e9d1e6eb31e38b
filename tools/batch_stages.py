"""Per-stage elapsed times of the images of a concurrent cfg2 batch (stage events on each
context's stream), next to the same image alone: which stage stretches under concurrency?
(design tool, GPU)    python tools/batch_stages.py [workers] [budget] [batch]
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

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B = int(sys.argv[2]) if len(sys.argv) > 2 else 48
N = int(sys.argv[3]) if len(sys.argv) > 3 else 16
cfg = CONFIGS["cfg2"]
img = cfg.image()
P = img.shape[0] * img.shape[1]
dev = torch.device("cuda", 0)
kind = cabi.INIT_KMEANSPP
qc = cabi.QuantizeCfg(kind, cfg.k, cfg.seed, cabi.Term(1e-3, 100, 0, 0), 4)
bufs = [(torch.from_numpy(img).to(dev), torch.empty(P, dtype=torch.int32, device=dev),
         torch.empty((P, 3), dtype=torch.uint8, device=dev), torch.empty((cfg.k, 3), dtype=torch.float64, device=dev))
        for _ in range(N)]
ctxs = []
for w in range(W):
    c = cabi.Context(0)
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    if B:
        c.set_sm_budget(B)
    c.set_profiling(True)
    ctxs.append((c, s, np.zeros(128)))


def work(w):
    c, s, sse = ctxs[w]
    out = []
    for i in range(w, N, W):
        t0 = time.perf_counter()
        st = c.quantize_raw(bufs[i][0], P, qc, None, bufs[i][3], None, sse, bufs[i][1], bufs[i][2])
        out.append((st.ms_histogram, st.ms_init, st.ms_lloyd, st.ms_map, (time.perf_counter() - t0) * 1e3))
    return out


pool = ThreadPoolExecutor(W)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = [r for part in pool.map(work, range(W)) for r in part]
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
a = np.array(res)
print(f"workers {W} budget {B} batch {N}: wall {wall:.3f} ms; per image mean: hist {a[:,0].mean():.3f} init {a[:,1].mean():.3f} "
      f"lloyd {a[:,2].mean():.3f} map {a[:,3].mean():.3f} sum {a[:,:4].sum(1).mean():.3f} host call {a[:,4].mean():.3f} ms")
print("  max per stage:", a.max(0).round(3).tolist())
