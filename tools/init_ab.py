"""A/B timing of the initialiser across build variants (design tool, GPU).

    python tools/init_ab.py run cfg5 base NAME ...   # NAME: libcqg_NAME.so built by tools/sweep_ab.py build
Prints the device-timed init stage (library profiling events) of each build.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(cfg_name):
    from paper_1101_0395_b200 import cabi, quant
    from paper_1101_0395_b200.synth import CONFIGS
    cfg = CONFIGS[cfg_name]
    img = cfg.image()
    ctx = cabi.Context(0)
    hist = quant.build_histogram(img, ctx=ctx)
    sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
    initf = quant.init_kmeanspp if cfg.init == "kpp" else quant.init_maximin
    initf(hist, sc, ctx=ctx)
    ctx.set_profiling(True)
    ctx.read_profile(True)
    reps = 5
    for _ in range(reps):
        initf(hist, sc, ctx=ctx)
    pr = ctx.read_profile(True)
    print(f"{os.path.basename(os.environ.get('CQG_LIB', 'libcqg.so'))}: init {pr.ms[cabi.PROF_INIT] / reps:.4f} ms")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        for name in sys.argv[3:]:
            env = dict(os.environ)
            if name != "base":
                env["CQG_LIB"] = os.path.join(ROOT, "paper_1101_0395_b200", f"libcqg_{name}.so")
            subprocess.run([sys.executable, __file__, "one", sys.argv[2]], env=env)
    else:
        one(sys.argv[2])
