"""Tile initialiser: cost of a warp's round of update_tiles by the number of tiles the new centre reaches
in that warp's share (timing build, tools/init_timing.py build). (design tool, GPU)
    python tools/init_timing.py build && python tools/tile_warp_hist.py [cfg5]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1101_0395_b200 import _build  # noqa: E402

TLIB = os.path.join(_build.PKG, "libcqg_timing.so")
from paper_1101_0395_b200 import cabi, quant  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cabi.load(TLIB)
cfg = CONFIGS[name]
img = cfg.image()
ctx = cabi.Context(0)
hist = quant.build_histogram(img, ctx=ctx)
sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
initf = quant.init_kmeanspp if cfg.init == "kpp" else quant.init_maximin
L = C.CDLL(TLIB)
buf = (C.c_ulonglong * 32)()
initf(hist, sc, ctx=ctx)
L.cqg_dbg_warp_hist(buf, 1)
initf(hist, sc, ctx=ctx)
L.cqg_dbg_warp_hist(buf, 1)
tot = sum(buf[2 * i + 1] for i in range(16))
print(f"{name}: warp-rounds {tot}")
for i in range(16):
    cyc, cnt = buf[2 * i], buf[2 * i + 1]
    if cnt:
        print(f"  reached tiles {i:2d}{'+' if i == 15 else ' '}: {cnt:9d} warp-rounds ({100 * cnt / tot:5.1f}%)  mean {cyc / cnt:9.0f} cycles")
