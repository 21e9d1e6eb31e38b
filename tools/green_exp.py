"""Experiment (GPU): cfg2 batch with each library context on its own green context
(a disjoint SM partition) instead of budgets on the shared device.
    python tools/green_exp.py [sms_per_partition] [batch] [flags]
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from cuda.bindings import driver as cu

from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS


def ck(r):
    if r[0] != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(r[0]))
    return r[1:] if len(r) > 2 else (r[1] if len(r) == 2 else None)


SMS = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N = int(sys.argv[2]) if len(sys.argv) > 2 else 18
FLAGS = int(sys.argv[3]) if len(sys.argv) > 3 else 0
torch.cuda.init()
torch.zeros(1, device="cuda")
dev = ck(cu.cuDeviceGet(0))
res = ck(cu.cuDeviceGetDevResource(dev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
print("device SMs:", res.sm.smCount)
groups, nb, rem = ck(cu.cuDevSmResourceSplitByCount(148 // SMS, res, FLAGS, SMS))
print("groups:", nb, [g.sm.smCount for g in groups[:nb]], "remainder", rem.sm.smCount)
streams = []
for g in groups[:nb]:
    desc = ck(cu.cuDevResourceGenerateDesc([g], 1))
    gctx = ck(cu.cuGreenCtxCreate(desc, dev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    st = ck(cu.cuGreenCtxStreamCreate(gctx, cu.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    streams.append((gctx, st, g.sm.smCount))

cfg = CONFIGS["cfg2"]
img = cfg.image()
P = img.shape[0] * img.shape[1]
d = torch.device("cuda", 0)
qc = cabi.QuantizeCfg(cabi.INIT_KMEANSPP, cfg.k, cfg.seed, cabi.Term(1e-3, 100, 0, 0), 4)
bufs = [(torch.from_numpy(img).to(d), torch.empty(P, dtype=torch.int32, device=d),
         torch.empty((P, 3), dtype=torch.uint8, device=d), torch.empty((cfg.k, 3), dtype=torch.float64, device=d))
        for _ in range(N)]
W = len(streams)
ctxs = []
for gctx, st, n in streams:
    c = cabi.Context(0)
    c.set_stream(int(st))
    c.set_sm_budget(n)
    ctxs.append((c, np.zeros(128)))


def work(w, prof=False):
    c, sse = ctxs[w]
    out = []
    for i in range(w, N, W):
        st = c.quantize_raw(bufs[i][0], P, qc, None, bufs[i][3], None, sse, bufs[i][1], bufs[i][2])
        out.append((st.ms_histogram, st.ms_init, st.ms_lloyd, st.ms_map, st.lloyd.iterations))
    return out


pool = ThreadPoolExecutor(W)
# one context alone first
for _ in range(3):
    r1 = work(0)
torch.cuda.synchronize()
t0 = time.perf_counter()
r1 = work(0)
torch.cuda.synchronize()
print(f"context 0 alone: {len(r1)} images in {(time.perf_counter() - t0) * 1e3:.3f} ms")
for nact in range(1, W + 1):
    ws = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        list(pool.map(work, range(nact)))
        torch.cuda.synchronize()
        ws.append((time.perf_counter() - t0) * 1e3)
    print(f"  {nact} contexts active: {min(ws[1:]):.3f} ms for {len(range(0, N, W))} images each")
walls = []
for rep in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = [r for part in pool.map(work, range(W)) for r in part]
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
wall = min(walls[2:])
print(f"{W} green contexts x {SMS} SMs, batch {N}: wall {wall:.3f} ms -> {N * P / wall / 1e3:.1f} MPix/s; iterations "
      f"{sorted(set(int(r[4]) for r in res))}")
ok = all(torch.equal(bufs[i][3], bufs[0][3]) and torch.equal(bufs[i][1], bufs[0][1]) for i in range(1, N))
print("copies equal:", ok)
c0, _ = ctxs[0]
c0.set_profiling(True)
r = work(0)
print("stage ms alone in partition:", [round(float(x), 3) for x in r[-1][:4]])
