import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS
cfg = CONFIGS["cfg2"]; img = cfg.image(); P = img.shape[0]*img.shape[1]
ctx = cabi.Context(0); s = torch.cuda.current_stream(); ctx.set_stream(s.cuda_stream)
d_img = torch.from_numpy(img).cuda(); idx = torch.empty(P, dtype=torch.int32, device="cuda"); q = torch.empty((P,3), dtype=torch.uint8, device="cuda")
pal = torch.empty((256,3), dtype=torch.float64, device="cuda"); sse = np.zeros(128)
qc = cabi.QuantizeCfg(cabi.INIT_KMEANSPP, 256, cfg.seed, cabi.Term(1e-3, 100, 0, 0), 4)
flush = torch.empty(512<<20, dtype=torch.uint8, device="cuda")
def run(prof, stats, n=20):
    ctx.set_profiling(prof)
    ts = []
    for i in range(n+3):
        flush.fill_(i & 255); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if stats: ctx.quantize_raw(d_img, P, qc, None, pal, None, sse, idx, q)
        else:
            st = cabi.QuantizeStats()
            cabi.check(ctx.L.cqg_quantize(ctx.h, cabi.ptr(d_img), P, C.byref(qc), None, cabi.ptr(pal), None, cabi.ptr(sse), cabi.ptr(idx), cabi.ptr(q), None))
        e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    ctx.set_profiling(False)
    return np.median(ts), np.mean(ts)
import ctypes as C
for prof, stats in [(True, True), (False, True), (False, False), (True, True), (False, False)]:
    print("prof", prof, "stats", stats, "median/mean ms", run(prof, stats))
