"""Phase timing of the cluster k-means++ initialiser (design tool, GPU).

Builds a variant of libcqg.so with -DCQG_INIT_TIMING into
paper_1101_0395_b200/build_timing/, runs the init stage of a config and prints
the mean cycles per round of: update, publish, cluster barrier, draw, tail.

    python tools/init_timing.py [cfg2]      # build here, run on the GPU box
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1101_0395_b200 import _build  # noqa: E402

TLIB = os.environ.get("CQG_TIMING_LIB", os.path.join(_build.PKG, "libcqg_timing.so"))


def build(extra=()):
    bdir = os.path.join(_build.PKG, "build_timing")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    for src in _build.SOURCES:
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        subprocess.check_call([_build.nvcc(), *_build.flags(["-DCQG_INIT_TIMING", *extra]), "-c",
                               os.path.join(_build.CSRC, src), "-o", o])
        objs.append(o)
    subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "--cudart", "static", "-o", TLIB, *objs])


def run(name):
    from paper_1101_0395_b200 import cabi, quant
    from paper_1101_0395_b200.synth import CONFIGS
    cabi.load(TLIB)  # the timing variant becomes the process's libcqg
    cfg = CONFIGS[name]
    img = cfg.image()
    ctx = cabi.Context(0)
    hist = quant.build_histogram(img, ctx=ctx)
    sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
    initf = quant.init_kmeanspp if cfg.init == "kpp" else quant.init_maximin
    L = C.CDLL(TLIB)
    buf = (C.c_ulonglong * 8)()
    initf(hist, sc, ctx=ctx)
    L.cqg_dbg_init_timing(buf, 1)
    reps = 5
    for _ in range(reps):
        initf(hist, sc, ctx=ctx)
    L.cqg_dbg_init_timing(buf, 1)
    rounds = reps * (cfg.k - 1)
    names = ["update", "publish", "cluster_sync", "draw", "tail"]
    tot = sum(buf[i] for i in range(5))
    if tot:  # cluster kernel (small substrates)
        for i, nm in enumerate(names):
            print(f"{nm:14s} {buf[i] / rounds:8.0f} cycles/round  {100 * buf[i] / tot:5.1f}%")
        print(f"{'total':14s} {tot / rounds:8.0f} cycles/round")
    # cooperative record kernel (large substrates; forced with CQG_NO_CLUSTER_INIT=1)
    L.cqg_dbg_coop_timing(buf, 1)
    tr = (C.c_ulonglong * 2048)()
    lp = (C.c_ulonglong * 4)()
    if hasattr(L, "cqg_dbg_tile_rounds"):
        L.cqg_dbg_tile_rounds(tr, 1)
        L.cqg_dbg_loc_phase(lp, 1)
    initf(hist, sc, ctx=ctx)
    L.cqg_dbg_coop_timing(buf, 1)
    if hasattr(L, "cqg_dbg_tile_rounds"):
        L.cqg_dbg_tile_rounds(tr, 0)
        L.cqg_dbg_loc_phase(lp, 0)
        if lp[0]:
            r1 = cfg.k - 1
            print(f"tile locate: segment sums {lp[0] / r1:8.0f}  owner run {lp[1] / r1:8.0f}  "
                  f"points {lp[2] / r1:8.0f} cycles/round")
        sel = [1, 2, 3, 5, 8, 12, 20, 40, 80, 160, cfg.k - 1]
        if any(tr[2 * r] for r in sel if r < 1024):
            print("tile rounds (slowest block update / block-0 locate, cycles): " +
                  "  ".join(f"r{r}:{tr[2 * r]}/{tr[2 * r + 1]}" for r in sel if r < min(cfg.k, 1024)))
    names = ["update", "grid_sync_1", "locate", "grid_sync_2", "tail"]
    tot = sum(buf[i] for i in range(5))
    if tot:
        rounds1 = cfg.k - 1
        for i, nm in enumerate(names):
            print(f"coop {nm:14s} {buf[i] / rounds1:8.0f} cycles/round  {100 * buf[i] / tot:5.1f}%")
        if buf[5]:  # tile layout
            print(f"coop tiles updated {buf[5] / rounds1:10.0f}/round  points changed {buf[6] / rounds1:10.0f}/round  "
                  f"slowest block update {buf[7] / rounds1:8.0f} cycles/round")
    # persistent Lloyd kernel phases (block 0, thread 0), per WALK iteration
    init = initf(hist, sc, ctx=ctx)
    opts = quant.ClusterOptions(quant.Termination(fixed_iterations=cfg.fixed_iterations or None))
    quant.wsm_hist(hist, init, opts, ctx=ctx)
    L.cqg_dbg_lloyd_timing(buf, 1)
    L.cqg_dbg_block_timing((C.c_ulonglong * (1024 * 3))(), 1)
    if hasattr(L, "cqg_dbg_sweep_timing"):
        L.cqg_dbg_sweep_timing((C.c_ulonglong * 8)(), 1)
    st = None
    for _ in range(reps):
        st = quant.wsm_hist(hist, init, opts, ctx=ctx)
    L.cqg_dbg_lloyd_timing(buf, 1)
    its = reps * (st.iterations - 1)
    bt = (C.c_ulonglong * (1024 * 3))()
    L.cqg_dbg_block_timing(bt, 0)
    import numpy as np
    arr = np.array(bt[:], dtype=np.float64).reshape(1024, 3)
    arr = arr[arr.sum(1) > 0] / its
    for j, nm in enumerate(["ndc", "sweep", "replay"]):
        col = arr[:, j]
        print(f"  per-block {nm:7s} min {col.min():8.0f} mean {col.mean():8.0f} max {col.max():8.0f}")
    tot_b = arr.sum(1)
    print(f"  per-block total   min {tot_b.min():8.0f} mean {tot_b.mean():8.0f} max {tot_b.max():8.0f}")
    names = ["ndc", "sweep", "flush+replay", "grid_sync_1", "iter_end", "grid_sync_2"]
    tot = sum(buf[i] for i in range(6))
    if not tot:
        return
    for i, nm in enumerate(names):
        print(f"{nm:14s} {buf[i] / its:8.0f} cycles/iter  {100 * buf[i] / tot:5.1f}%")
    print(f"{'total':14s} {tot / its:8.0f} cycles/iter  (swept {st.swept_total / (st.iterations * len(hist.counts)):.3f})")
    print(f"  finalise (from the barrier): pass 1 {buf[6] / its:8.0f}  + SSE tree and status {buf[7] / its:8.0f} cycles/iter")
    if hasattr(L, "cqg_dbg_sweep_timing"):
        sb = (C.c_ulonglong * 8)()
        L.cqg_dbg_sweep_timing(sb, 0)
        calls = max(sb[3], 1)
        print(f"  pruned sweep (block 0): filter {sb[0] / calls:8.0f}  whole {sb[1] / calls:8.0f} cycles/call, "
              f"survivors {sb[2] / calls:6.0f}")
        print(f"  list tiles (block 0, thread 0): loads {sb[4] / calls:8.0f}  centre loop {sb[5] / calls:8.0f}  "
              f"resolve {sb[6] / calls:8.0f} cycles/call")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "build":
        build(sys.argv[2:])  # e.g. -DCQG_EXP_SKIP_UPDATE=1 (timing experiments, wrong results)
    else:
        run(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
