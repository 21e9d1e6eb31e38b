"""Compare the device initialiser with the oracle on a bench config (GPU).

    python tools/check_init.py cfg3 [cfg5 ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle, build  # noqa: E402
from paper_1101_0395_b200 import cabi, quant  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402

build()
O = Oracle()
ctx = cabi.Context(0)
for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx)
    sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
    if cfg.init == "kpp":
        dev = quant.init_kmeanspp(hist, sc, ctx=ctx)
        ora = O.init_kmeanspp(hist.packed, hist.counts, P, cfg.k, cfg.seed)
    else:
        dev = quant.init_maximin(hist, sc, ctx=ctx)
        ora = O.init_maximin(hist.packed, hist.counts, P, cfg.k, cfg.seed)
    bad = np.nonzero(np.any(dev != ora, axis=1))[0]
    print(name, "N'", hist.counts.size, "equal" if bad.size == 0 else f"FIRST MISMATCH at centre {bad[0]} of {cfg.k}")
