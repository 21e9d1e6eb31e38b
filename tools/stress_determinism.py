"""Determinism under contention (GPU): the signalling protocols of the cluster
initialiser (st.async + mbarrier), the persistent Lloyd kernel (grid barrier,
rotating delta slots) and the tile initialiser (release flags) are timing
sensitive by construction, and compute-sanitizer is closed on this GPU pool.
This runs the full pipeline many times on 8 concurrent, oversubscribed library
contexts -- every run's timing differs -- and requires every output of every
run to be bit-identical to the oracle-checked first one.

    python tools/stress_determinism.py [rounds]      > profiles/r02_stress_determinism.txt
"""
import hashlib
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.pyoracle import UPDATE_EXACT, Oracle
from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS, synth_image

ROUNDS = int(sys.argv[1]) if len(sys.argv) > 1 else 40
W = 8
dev = torch.device("cuda", 0)
O = Oracle()
cases = [("cfg2 (cluster k-means++, persistent Lloyd)", CONFIGS["cfg2"].image(), 256, "kpp", 202, 0),
         ("cfg1 (cluster maximin, persistent Lloyd)", CONFIGS["cfg1"].image(), 32, "mmx", 101, 0),
         ("1536x1024 noise 0.5 (record / tile initialiser, graph Lloyd, partitioned histogram)",
          synth_image(1536, 1024 * 3, 9, nblobs=16, sigma=25.0, noise=0.5), 64, "kpp", 9, 6)]
for name, img, K, init, seed, fixed in cases:
    P = img.shape[0] * img.shape[1]
    kind = cabi.INIT_KMEANSPP if init == "kpp" else cabi.INIT_MAXIMIN
    qc = cabi.QuantizeCfg(kind, K, seed, cabi.Term(1e-3, 100, fixed, 0), 4)
    c, n, _ = O.histogram(img)
    ini = (O.init_kmeanspp if init == "kpp" else O.init_maximin)(c, n, P, K, seed)
    ref = O.wsm(c, n, P, ini, fixed_it=fixed, mode=UPDATE_EXACT)
    ridx, rq, rmse, _ = O.map_pixels(img, ref.centers, mode=UPDATE_EXACT)
    ctxs = []
    for w in range(W):
        cx = cabi.Context(0)
        s = torch.cuda.Stream()
        cx.set_stream(s.cuda_stream)
        cx.set_sm_budget(32)
        ctxs.append((cx, s, torch.from_numpy(img).to(dev), torch.empty(P, dtype=torch.int32, device=dev),
                     torch.empty((P, 3), dtype=torch.uint8, device=dev),
                     torch.empty((K, 3), dtype=torch.float64, device=dev),
                     torch.empty(P, dtype=torch.int32, device=dev)))

    def digest(w):
        cx, s, src, idx, q, pal, lab = ctxs[w]
        sse = np.zeros(128)
        st = cx.quantize_raw(src, P, qc, None, pal, lab, sse, idx, q)
        s.synchronize()
        h = hashlib.sha1()
        for t in (pal, idx, q, lab[:st.n_unique]):
            h.update(t.cpu().numpy().tobytes())
        h.update(sse[:st.lloyd.iterations].tobytes())
        return (h.hexdigest(), st.n_unique, st.lloyd.iterations, st.lloyd.ndc_total, st.mean_sq_dist, st.map_ndc)

    first = digest(0)
    cx, s, src, idx, q, pal, lab = ctxs[0]
    ok = (first[1] == c.size and first[2] == ref.iterations and first[3] == ref.ndc_total and first[4] == rmse
          and np.array_equal(pal.cpu().numpy(), ref.centers)
          and np.array_equal(idx.cpu().numpy().view(np.uint32), ridx)
          and np.array_equal(lab[:c.size].cpu().numpy().view(np.uint32), ref.labels))
    t0 = time.perf_counter()
    bad = 0
    with ThreadPoolExecutor(W) as ex:
        for r in range(ROUNDS):
            for d in ex.map(digest, range(W)):
                bad += d != first
    print(f"{name}: N'={c.size} K={K} first run equals the oracle: {ok}; {ROUNDS * W} concurrent runs on {W} contexts, "
          f"{bad} differ from the first ({time.perf_counter() - t0:.1f} s)", flush=True)
    for t in ctxs:
        t[0].close()
    if not ok or bad:
        sys.exit(1)
