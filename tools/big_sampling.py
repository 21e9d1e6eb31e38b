import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1101_0395_b200 import quant
from paper_1101_0395_b200.synth import CONFIGS
for name, mode in [("cfg3", "none"), ("cfg5", "none"), ("cfg5", "2to1"), ("cfg5", "both")]:
    cfg = CONFIGS[name]
    img = cfg.image()
    qc = quant.QuantizeConfig(method=quant.parse_method("wsm-" + cfg.init), k=cfg.k, seed=cfg.seed, sampling=mode)
    if cfg.fixed_iterations:
        qc.term = quant.Termination(fixed_iterations=cfg.fixed_iterations)
    t0 = time.perf_counter()
    r = quant.run_quantize(img, qc)
    t1 = time.perf_counter()
    print(name, mode, "substrate", r.substrate_points, "it", r.report.iterations, "mse", round(r.report.mse, 4),
          "wall ms", round(1e3 * (t1 - t0), 1), "stages", {k: round(v, 2) for k, v in r.stage_ms.items()})
