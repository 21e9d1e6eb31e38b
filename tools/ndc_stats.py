import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import CONFIGS
for name in ["cfg2", "cfg3", "cfg5"]:
    cfg = CONFIGS[name]
    img = cfg.image()
    ctx = cabi.Context(0)
    hist = quant.build_histogram(img, ctx=ctx)
    sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
    initf = quant.init_kmeanspp if cfg.init == "kpp" else quant.init_maximin
    init = initf(hist, sc, ctx=ctx)
    opts = quant.ClusterOptions(quant.Termination(fixed_iterations=cfg.fixed_iterations or None))
    st = quant.wsm_hist(hist, init, opts, ctx=ctx)
    n = hist.size()
    walk = (st.ndc_total - n * cfg.k) / (n * (st.iterations - 1))
    print(name, "n", n, "iters", st.iterations, "mean walk positions per point-iteration (WALK iterations)", round(walk, 2),
          "swept fraction", round(st.swept_total / (n * st.iterations), 3))
