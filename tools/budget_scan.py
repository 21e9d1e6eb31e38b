"""Stage times of one image alone on the device as a function of the library
context's SM budget (design tool, GPU): SM-milliseconds per stage tell how many
SMs a context of a concurrent batch should get.

    python tools/budget_scan.py [cfg2] [budgets...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
budgets = [int(x) for x in sys.argv[2:]] or [0, 16, 24, 37, 48, 74, 100]
cfg = CONFIGS[name]
img = cfg.image()
P = img.shape[0] * img.shape[1]
dev = torch.device("cuda", 0)
d_img = torch.from_numpy(img).to(dev)
d_idx = torch.empty(P, dtype=torch.int32, device=dev)
d_q = torch.empty((P, 3), dtype=torch.uint8, device=dev)
d_pal = torch.empty((cfg.k, 3), dtype=torch.float64, device=dev)
kind = cabi.INIT_KMEANSPP if cfg.init == "kpp" else cabi.INIT_MAXIMIN
qc = cabi.QuantizeCfg(kind, cfg.k, cfg.seed, cabi.Term(1e-3, 100, cfg.fixed_iterations, 0), 4)
sse = np.zeros(128)
for b in budgets:
    ctx = cabi.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    if b:
        ctx.set_sm_budget(b)
    for _ in range(3):
        ctx.quantize_raw(d_img, P, qc, None, d_pal, None, sse, d_idx, d_q)
    ctx.set_profiling(True)
    ctx.read_profile(True)
    reps = 10
    ms = np.zeros(4)
    for _ in range(reps):
        st = ctx.quantize_raw(d_img, P, qc, None, d_pal, None, sse, d_idx, d_q)
        ms += [st.ms_histogram, st.ms_init, st.ms_lloyd, st.ms_map]
    ms /= reps
    sms = b or 148
    print(f"{name} budget {sms:3d}: hist {ms[0]:.3f} init {ms[1]:.3f} lloyd {ms[2]:.3f} map {ms[3]:.3f} "
          f"total {ms.sum():.3f} ms | lloyd SM.ms {ms[2] * sms:.1f} total SM.ms {ms.sum() * sms:.1f}", flush=True)
    ctx.close()
