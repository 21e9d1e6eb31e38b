"""A small run through every kernel family of libcqg.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; tools/sanitize.sh):

  histogram     small fused path (P < 2^22) and the bucketed large path (2^22 pixels)
  initialisers  k-means++ and maximin (cluster kernel by default; CQG_NO_CLUSTER_INIT,
                CQG_INIT_TILE_MIN / CQG_NO_INIT_TILE select the others)
  Lloyd         persistent kernel (default) / graph or host loop (CQG_NO_GRAPH) /
                unpruned (CQG_NO_PRUNE) / without the code table (CQG_NO_NDC_CODE), repair
  mapping       MAPW / MAP sweeps, replay, MSE, mapping NDC, pixel kernel
  exact engine  generic-weight wsm, kmeans_full, centre table, repair, masses, padding
  coarse        coarse 32^3 histogram
Every output is checked against the C oracle, so a sanitizer run is also a parity run.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle.pyoracle import UPDATE_EXACT, Oracle
from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import synth_image

O = Oracle()
ctx = cabi.Context(0)
fails = []


def check(name, ok):
    print(f"{'ok  ' if ok else 'FAIL'} {name}", flush=True)
    if not ok:
        fails.append(name)


def pipeline(img, k, init, fixed=0):
    P = img.shape[0] * img.shape[1]
    cfg = quant.QuantizeConfig(method=quant.parse_method("wsm-" + init), k=k, seed=5,
                               term=quant.Termination(fixed_iterations=fixed or None))
    r = quant.run_quantize(img, cfg, ctx=ctx)
    c, n, _ = O.histogram(img)
    c0 = O.init_kmeanspp(c, n, P, k, 5) if init == "kpp" else O.init_maximin(c, n, P, k, 5)
    w = O.wsm(c, n, P, c0, fixed_it=fixed, mode=UPDATE_EXACT)
    idx, q, mse, mndc = O.map_pixels(img, w.centers, mode=UPDATE_EXACT)
    return (np.array_equal(r.palette, w.centers) and r.state.ndc_total == w.ndc_total
            and np.array_equal(r.mapping.indices, idx) and r.report.mse == mse and r.mapping.ndc == mndc)


small = synth_image(256, 192, 3, nblobs=10, sigma=14.0, noise=0.05)
check("pipeline kpp K=64", pipeline(small, 64, "kpp"))
check("pipeline mmx K=32", pipeline(small, 32, "mmx"))
check("pipeline K=300 fixed 4", pipeline(synth_image(160, 120, 4, nblobs=6, noise=0.3), 300, "mmx", 4))
large = synth_image(2048, 2048, 6, nblobs=12, sigma=20.0, noise=0.2)
h = quant.build_histogram(large, ctx=ctx)
c, n, f = O.histogram(large)
check("histogram large path", np.array_equal(h.packed, c) and np.array_equal(h.counts, n) and np.array_equal(h.first, f))
rng = np.random.default_rng(1)
pts = rng.integers(0, 256, (400, 3)).astype(float)
w = rng.random(400) + 0.05
w /= w.sum()
st = quant.wsm(pts, w, pts[:12], ctx=ctx)
check("exact engine wsm", st.iterations > 0)
st = quant.kmeans_full(pts, pts[:12], quant.ClusterOptions(term=quant.Termination(fixed_iterations=3)), ctx=ctx)
check("exact engine kmeans_full", st.iterations == 3)
cen = np.repeat(pts[:3], 3, axis=0)
lab = np.zeros(400, np.uint32)
check("exact repair", quant.repair_empty_clusters(pts, w, cen, lab, ctx=ctx) > 0)
hw = quant.WeightedHistogram(pts, w, np.ones(400, np.uint32), 400)
check("next masses / maximin pad", quant.kmeanspp_next_masses(hw, pts[:2], ctx=ctx).size == 400
      and quant.maximin_pad(hw, pts[:2], 9, ctx=ctx).shape == (9, 3))
ch = quant.build_coarse_histogram(small, ctx=ctx)
check("coarse histogram", int(ch.count.sum()) == 256 * 192)
print("FAILURES: " + ", ".join(fails) if fails else "all checks passed")
sys.exit(1 if fails else 0)
