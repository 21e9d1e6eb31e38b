"""A/B timing of build variants of the Lloyd sweep (design tool, GPU).

    python tools/sweep_ab.py build NAME -DFLAG=V ...   # here: builds libcqg_NAME.so
    python tools/sweep_ab.py run cfg3 NAME [NAME...]   # on the GPU box

`run` starts one process per variant (CQG_LIB selects the build) and prints
the dense sweep time (cqg_bench_sweep on the final Lloyd state) and the Lloyd
stage time of one quantize call.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lib_path(name):
    return os.path.join(ROOT, "paper_1101_0395_b200", f"libcqg_{name}.so")


def build(name, flags):
    from paper_1101_0395_b200 import _build
    bdir = os.path.join(_build.PKG, f"build_{name}")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    for src in _build.SOURCES:
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        subprocess.check_call([_build.nvcc(), *_build.flags(flags), "-c", os.path.join(_build.CSRC, src), "-o", o])
        objs.append(o)
    subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "--cudart", "static", "-o", lib_path(name), *objs])


def one(cfg_name):
    from paper_1101_0395_b200 import cabi, quant
    from paper_1101_0395_b200.synth import CONFIGS
    cfg = CONFIGS[cfg_name]
    img = cfg.image()
    ctx = cabi.Context(0)
    hist = quant.build_histogram(img, ctx=ctx)
    sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
    init = (quant.init_kmeanspp if cfg.init == "kpp" else quant.init_maximin)(hist, sc, ctx=ctx)
    opts = quant.ClusterOptions(quant.Termination(fixed_iterations=cfg.fixed_iterations or None))
    quant.wsm_hist(hist, init, opts, ctx=ctx)
    ctx.set_profiling(True)
    ctx.read_profile(True)
    reps = 10
    for _ in range(reps):
        st = quant.wsm_hist(hist, init, opts, ctx=ctx)
    pr = ctx.read_profile(True)
    ctx.set_profiling(False)
    loop = pr.ms[cabi.PROF_LLOYD] / reps
    step = sum(pr.ms[i] for i in range(cabi.PROF_N)) / reps
    ms, units = ctx.bench_sweep(20)
    print(f"{os.path.basename(os.environ.get('CQG_LIB', 'libcqg.so'))}: dense sweep {ms:.4f} ms "
          f"({units * 8 / ms / 1e9:.1f} TFLOP/s)  lloyd loop {loop:.4f} ms  lloyd kernels {step:.4f} ms  "
          f"iters {st.iterations} swept {st.swept_total / (st.iterations * hist.size()):.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "run":
        for name in sys.argv[3:]:
            env = dict(os.environ, CQG_LIB=lib_path(name) if name != "base" else os.path.join(
                ROOT, "paper_1101_0395_b200", "libcqg.so"))
            subprocess.run([sys.executable, __file__, "one", sys.argv[2]], env=env)
    else:
        one(sys.argv[2])
