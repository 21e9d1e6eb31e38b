"""Per-iteration swept (non-pruned) fraction of the Lloyd loop (design tool, GPU).

    python tools/swept_trace.py [cfg2] [lib]
Runs wsm with fixed_iterations = 1..N on the config's substrate and prints the
points that went through the full centre loop in each iteration.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1101_0395_b200 import cabi, quant  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if len(sys.argv) > 2:
    cabi.load(sys.argv[2])
cfg = CONFIGS[name]
img = cfg.image()
ctx = cabi.Context(0)
hist = quant.build_histogram(img, ctx=ctx)
init = quant.init_kmeanspp(hist, quant.SeedConfig(k=cfg.k, seed=cfg.seed), ctx=ctx) if cfg.init == "kpp" else \
    quant.init_maximin(hist, quant.SeedConfig(k=cfg.k, seed=cfg.seed), ctx=ctx)
n = len(hist.counts)
prev = 0
out = []
for it in range(1, 21):
    st = quant.wsm_hist(hist, init, quant.ClusterOptions(quant.Termination(fixed_iterations=it)), ctx=ctx)
    out.append(f"{(st.swept_total - prev) / n:.3f}")
    prev = st.swept_total
print(name, "swept per iteration:", " ".join(out))
