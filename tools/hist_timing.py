"""Device time of the histogram stage (cqg_histogram on a device-resident
image, CUDA events) on the BASELINE configs, checked against the oracle.

    python tools/hist_timing.py [cfg3 cfg5 ...]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.pyoracle import Oracle
from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS

names = sys.argv[1:] or ["cfg3", "cfg5"]
ctx = cabi.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
O = Oracle()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name in names:
    img = CONFIGS[name].image()
    P = img.shape[0] * img.shape[1]
    d_img = torch.from_numpy(img).cuda()
    cap = min(P, 1 << 24)
    col = torch.empty(cap, dtype=torch.int32, device="cuda")
    cnt = torch.empty(cap, dtype=torch.int32, device="cuda")
    fst = torch.empty(cap, dtype=torch.int32, device="cuda")
    for _ in range(3):
        n = ctx.histogram_raw(d_img, P, col, cnt, fst)
    ts = []
    for _ in range(10):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = ctx.histogram_raw(d_img, P, col, cnt, fst)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    c, k, f = O.histogram(img)
    ok = (n == c.size and np.array_equal(col[:n].cpu().numpy().view(np.uint32), c)
          and np.array_equal(cnt[:n].cpu().numpy().view(np.uint32), k)
          and np.array_equal(fst[:n].cpu().numpy().view(np.uint32), f))
    ms = float(np.median(ts))
    alg = 3 * P + 8 * n
    print(f"{name}: P={P} N'={n} median {ms:.4f} ms (min {min(ts):.4f}) "
          f"alg {alg/1e6:.1f} MB -> {alg/ms/1e6:.0f} GB/s  parity={'ok' if ok else 'MISMATCH'}", flush=True)
