"""Benchmark: quantized MPixel/s (and Lloyd colour-centre distances/s) of the
B200-native hot path on BASELINE.json's configurations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg1|cfg3|cfg3k64|cfg4|cfg5] [--sharded]

A step is one pass of the hot path (histogram -> init -> weighted Lloyd ->
mapping + MSE, i.e. quant::run_quantize) over one batch of synthetic input.
The line's `value` is BASELINE.json configs[1] (cfg2: 512x512, K=256,
k-means++), the K=256 configuration the reference's CPU build also runs in
seconds. One step quantizes a batch of 16 copies of the cfg2 image (separate
buffers) through 8 concurrent library contexts of 32 SMs each -- the same
batch the reference arm runs, one copy per host thread; one cfg2 image alone
is two latency chains (255 dependent k-means++ draws on a 16-SM cluster, 20
grid-synchronised Lloyd iterations) that leave most of the device idle. The
single-image run (one context on the whole device) is measured first in the
same process and reported under `single_image`; the per-kernel profile and
the roofline come from it. The other single-GPU K=256 configurations are
reported in the same line under `by_config` (N=1: cfg3 4096^2 maximin, cfg5
8192^2 k-means++, one image per step, each with its own roofline fractions,
e2e, parity digest and 1-core reference baseline); cfg1 is the reference's own
small case.

Multi-GPU (one rank per GPU; `--gpus N` starts torch.distributed.run itself
when WORLD_SIZE is unset): cfg2 runs one independent replica per rank (the
path does not shard below ~1M colours: "replicas only"); by_config then adds
cfg4 (64 images sharded across ranks, no collective) and cfg5 sharded by
unique colour (one NCCL allreduce of the int64 moments per iteration).
Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events
on the launching stream with an L2 flush (write of a 512 MiB buffer) between
steps outside the timed events; the per-rank device time is max-reduced.

--impl reference times the reference's own CPU implementation (the reference
sources compiled in place: oracle/_ref/libquantref.so, through its public
run_quantize / stage API) on this box's host cores, one image per host thread.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
from concurrent.futures import ThreadPoolExecutor
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# concurrent library contexts use 3 streams each: 32 hardware queues instead of the default 8,
# so their streams do not alias (read at CUDA context creation: set before torch initialises CUDA)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "Lloyd color-center distances/s and quantized MPixel/s at K=256, 1-8 B200"
UNIT = "MPixel/s"


BATCH_DEFAULT = 16  # copies of a small image per step (both arms)


def config_dict(cfg, images_per_step):
    """The workload both arms print as `config` (the same dictionary on the GPU and the reference arm)."""
    return {"workload": cfg.name, "image": f"{cfg.width}x{cfg.height}", "images_per_step": int(images_per_step),
            "k": cfg.k if not cfg.k_cycle else list(cfg.k_cycle), "init": cfg.init,
            "fixed_iterations": cfg.fixed_iterations or None}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region.

    Uses NVML (nvidia-ml-py) every 2 ms from a background thread (the cfg2
    timed region is only ~25 ms); falls back to `nvidia-smi -lms 50`."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x0000000000000008: "hw_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000004: "sw_power_cap",
    }

    def __init__(self, device: int):
        self.device = device
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.mx.append(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run_nvml, daemon=True)
        except Exception:
            self.nvml = None
            self.t = threading.Thread(target=self._run_smi, daemon=True)
        self.t.start()
        time.sleep(0.005)
        return self

    def _run_nvml(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def _run_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}",
                                     "--format=csv,noheader,nounits", "-lms", "50"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            return
        for line in proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except ValueError:
                    pass
                for nm, v in zip(names, parts[2:6]):
                    if v.lower() == "active":
                        self.reasons.add(nm)
            if self.stop.is_set():
                break
        proc.terminate()

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": max(self.mx) if self.mx else None,
                    "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml 2 ms" if self.nvml else "nvidia-smi 50 ms"}


# ---------------------------------------------------------------------------
# reference arm (CPU)

def ref_pipeline_once(R, img, cfg, k, kind):
    h, w = img.shape[:2]
    t0 = time.perf_counter()
    out = R.time_pipeline(img, w, h, kind, k, cfg.seed, fixed_it=cfg.fixed_iterations)
    t1 = time.perf_counter()
    return t1 - t0, out


def run_reference(args, cfg):
    from concurrent.futures import ThreadPoolExecutor
    from oracle.pyoracle import RefLib, have_ref, Oracle
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    if have_ref():
        R = RefLib()
        kind = "reference"
    else:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    # one step = the GPU arm's batch (args.batch copies of the image; a batched config: its images), one
    # image per host thread; with more host threads than images, whole batches run side by side
    per_batch = cfg.images if cfg.images > 1 else max(1, args.batch)
    nimg = per_batch * max(1, threads // per_batch)
    base = cfg.image(0) if cfg.images == 1 else None
    imgs = [base if base is not None else cfg.image(i % cfg.images) for i in range(nimg)]
    ks = [cfg.k_for(i) for i in range(nimg)]
    P = imgs[0].shape[0] * imgs[0].shape[1]

    def one(i):
        return ref_pipeline_once(R, imgs[i], cfg, ks[i], cfg.init)

    times, dist, lloyd_s = [], 0.0, 0.0
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = list(ex.map(one, range(nimg)))
            t1 = time.perf_counter()
            if s >= args.warmup:
                times.append(t1 - t0)
                for (_, o), k in zip(res, ks):
                    dist += o["n_unique"] * k * o["iterations"]
                    lloyd_s += o["stage_s"][2]
    step = sum(times) / len(times)
    value = nimg * P / step / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, per_batch),
        "run": {"note": "reference sources compiled -O3 -DNDEBUG (oracle/Makefile), one image per host thread",
                "host_threads": threads, "batches_side_by_side": nimg // per_batch},
        "lloyd_distances_per_s": dist / lloyd_s * min(threads, nimg) if lloyd_s > 0 else None,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(threads, nimg), "kind": kind,
                         "sample": f"{nimg} {cfg.name} run_quantize pipelines per step on {threads} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(cfg, budget_s: float):
    """Reference pipeline (oracle/_ref) on 1 core, bounded sample."""
    try:
        from oracle.pyoracle import RefLib, have_ref, Oracle, UPDATE_REFERENCE
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "unavailable", "sample": str(e)}
    img = cfg.image(0)
    h, w = img.shape[:2]
    P = w * h
    k = cfg.k_for(0)
    if not have_ref():
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "unavailable",
                "sample": "oracle/_ref not built"}
    R = RefLib()
    runs, tot, st_sum = 0, 0.0, np.zeros(4)
    t_start = time.perf_counter()
    while True:
        dt, out = ref_pipeline_once(R, img, cfg, k, cfg.init)
        runs += 1
        tot += dt
        st_sum += out["stage_s"]
        if time.perf_counter() - t_start >= budget_s or runs >= 50:
            break
    return {"value": runs * P / tot / 1e6, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{runs} full {cfg.name} pipelines ({w}x{h}, K={k}, {cfg.init}) in {tot:.1f} s",
            "stage_s_mean": (st_sum / runs).round(6).tolist(),
            "lloyd_distances_per_s": (out["n_unique"] * k * out["iterations"]) / out["stage_s"][2]}


# ---------------------------------------------------------------------------
# our arm

def cpp_dropin(cfg, batch, workers, sms):
    """The same workload through the C++ drop-in (libquant_b200.so: quant::run_quantize with pageable
    std::vector buffers and the full QuantizeResult; quant::run_bench over `batch` copies with the cells
    shared out over worker threads): tools/cpp_e2e, wall clock."""
    import tempfile
    from paper_1101_0395_b200 import _build
    if not os.path.exists(_build.CPP_E2E_BIN):
        return {"unavailable": "tools/cpp_e2e not built"}
    img = cfg.image(0)
    h, w = img.shape[:2]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, f"{cfg.name}.ppm")
        with open(path, "wb") as f:
            f.write(b"P6\n%d %d\n255\n" % (w, h))
            f.write(np.ascontiguousarray(img, np.uint8).tobytes())
        method = "wsm-kpp" if cfg.init == "kpp" else "wsm-mmx"
        r = subprocess.run([_build.CPP_E2E_BIN, path, str(cfg.k), method, "20", str(batch), str(workers), str(sms)],
                           capture_output=True, text=True, timeout=300)
    if r.returncode != 0:
        return {"error": (r.stdout + r.stderr)[-400:]}
    return json.loads(r.stdout)


def parity_digest(cfg, img, k, image_id, st, pal, didx, dq):
    """The bench step's outputs (host copies) against the C oracle
    (UPDATE_EXACT) on the same input."""
    import hashlib
    from oracle.pyoracle import UPDATE_EXACT, Oracle
    t0 = time.perf_counter()
    O = Oracle()
    P = img.shape[0] * img.shape[1]
    c, n, _ = O.histogram(img)
    init = O.init_kmeanspp(c, n, P, k, cfg.seed) if cfg.init == "kpp" else O.init_maximin(c, n, P, k, cfg.seed)
    r = O.wsm(c, n, P, init, fixed_it=cfg.fixed_iterations, mode=UPDATE_EXACT)
    idx, q, mse, mndc = O.map_pixels(img, r.centers, mode=UPDATE_EXACT)
    out = {
        "checker": "oracle/cq_oracle.c (C restatement, exact moments)", "image": image_id,
        "palette_sha1": hashlib.sha1(pal.tobytes()).hexdigest()[:16],
        "palette_equal": bool(np.array_equal(pal.view(np.uint64), r.centers.view(np.uint64))),
        "n_unique_equal": int(st.n_unique) == int(c.size),
        "iterations_equal": int(st.lloyd.iterations) == r.iterations,
        "ndc_equal": int(st.lloyd.ndc_total) == r.ndc_total,
        "indices_equal": bool(np.array_equal(didx, idx)),
        "quantized_equal": bool(np.array_equal(dq, q)),
        "mse_equal": float(st.mean_sq_dist) == mse,
        "map_ndc_equal": int(st.map_ndc) == mndc,
        "oracle_s": round(time.perf_counter() - t0, 2),
    }
    out["ok"] = all(v for key, v in out.items() if key.endswith("_equal"))
    return out


def sharded_measure(args, cfg, env, steps, warmup):
    """One huge image (cfg5 / cfg3) over the ranks: histogram and init per
    rank, Lloyd sharded by unique colour with one allreduce of the int64
    moment partials per iteration (parallel.sharded_wsm; NCCL over NVLink),
    mapping of this rank's rows, the global MSE by an allreduce of the per-rank
    squared-distance sums. Total work is fixed as ranks are added (strong
    scaling). Device time per step is the max over ranks; e2e adds the H2D of
    the image and the D2H of this rank's rows from / to pinned host memory."""
    import torch
    import torch.distributed as dist
    from paper_1101_0395_b200 import cabi, parallel
    world, rank, local, dev, stream = env["world"], env["rank"], env["local"], env["dev"], env["stream"]
    ctx = cabi.Context(local)
    ctx.set_stream(stream.cuda_stream)
    img = cfg.image()
    H, W = img.shape[:2]
    P = H * W
    K = cfg.k
    kind = cabi.INIT_KMEANSPP if cfg.init == "kpp" else cabi.INIT_MAXIMIN
    d_img = torch.from_numpy(img).to(dev)
    cap = min(P, 1 << 24)
    d_col = torch.empty(cap, dtype=torch.int32, device=dev)
    d_cnt = torch.empty(cap, dtype=torch.int32, device=dev)
    d_init = torch.empty((K, 3), dtype=torch.float64, device=dev)
    r0, r1 = parallel.shard_bounds(H, world, rank)
    Pr = (r1 - r0) * W
    d_idx = torch.empty(max(Pr, 1), dtype=torch.int32, device=dev)
    d_q = torch.empty((max(Pr, 1), 3), dtype=torch.uint8, device=dev)
    term = cabi.Term(1e-3, 100, cfg.fixed_iterations, 0)
    eng = parallel.CudaShardEngine(ctx, dev)
    info = {}

    def step(src=d_img, idx=d_idx, q=d_q):
        if src is not d_img:
            d_img.copy_(src, non_blocking=True)
        n = ctx.histogram_raw(d_img, P, d_col, d_cnt)
        ctx.init_raw(kind, d_col, d_cnt, n, P, K, cfg.seed, d_init)
        r = parallel.sharded_wsm(eng, d_col[:n], d_cnt[:n], P, d_init, K, term, labels=False)
        pal = np.ascontiguousarray(r.centers)
        mse_r = ctx.map_raw(d_img[r0:r1], Pr, pal, K, d_idx, 4, d_q) if Pr else 0.0
        if idx is not d_idx and Pr:
            idx[:Pr].copy_(d_idx[:Pr], non_blocking=True)
            q[:Pr].copy_(d_q[:Pr], non_blocking=True)
        tot = torch.tensor([mse_r * Pr], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)  # global MSE: sum of the ranks' squared-distance sums / P
        info.update(n=n, it=r.iterations, ndc=r.ndc_total, mse=float(tot.item()) / P, pal=pal)
        return r

    def timed(run, nsteps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        tot = 0.0
        for s_ in range(nsteps):
            flush.fill_(s_ & 255)
            torch.cuda.synchronize()
            dist.barrier()
            ev0.record(stream)
            run()
            ev1.record(stream)
            torch.cuda.synchronize()
            tot += ev0.elapsed_time(ev1)
        t = torch.tensor([tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / nsteps

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        ms = timed(step, steps)
    launches = ctx.launches - launches0
    h_img = torch.from_numpy(img).pin_memory()
    h_idx = torch.empty(max(Pr, 1), dtype=torch.int32).pin_memory()
    h_q = torch.empty((max(Pr, 1), 3), dtype=torch.uint8).pin_memory()
    e_ms = timed(lambda: step(h_img, h_idx, h_q), steps)
    # roofline of this rank's Lloyd kernel: the dense sweep over its colour shard, back-to-back launches
    # on the final state (cqg_bench_sweep, CUDA events), against the FP32 peak of one GPU
    roofline = None
    try:
        iso_ms, iso_units = ctx.bench_sweep(20)
        peaks, peak_kind = measured_peaks()
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        fp32_peak = sms * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        ach = 8.0 * iso_units / (iso_ms / 1e3) / 1e12
        roofline = {"bound": "fp32", "kernel": "sweep_kernel<WALK> on rank 0's colour shard (dense launch)",
                    "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                    "traffic": None, "avg_launch_ms": iso_ms, "units_per_launch": iso_units,
                    "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 x sm_max_mhz ({peak_kind} MEASURED_PEAKS.json)"}
    except Exception as e:  # the shard engine kept no sweep state
        roofline = {"unavailable": str(e)[:200]}
    ctx.close()
    return {
        "roofline": roofline,
        "workload": cfg.name, "value": P / (ms / 1e3) / 1e6, "unit": UNIT, "n_gpus": world, "steps": steps,
        "ms_per_step": ms, "scaling": "strong",
        "parallelism": (f"unique colours sharded over {world} ranks (int64 moment allreduce per iteration); "
                        "histogram and initialiser replicated per rank; rows sharded for the mapping"),
        "lloyd_distances_per_s": info["n"] * K * info["it"] / (ms / 1e3), "n_unique": info["n"],
        "iterations": info["it"], "ndc_total": info["ndc"], "mse": info["mse"],
        "e2e": {"value": P / (e_ms / 1e3) / 1e6, "unit": UNIT, "ms_per_step": e_ms, "h2d_bytes_per_step": 3 * P,
                "d2h_bytes_per_step": 7 * Pr + 24 * K},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }


def run_sharded_line(args, cfg, env):
    """--sharded: the colour-sharded path as the bench line itself."""
    import torch
    import torch.distributed as dist
    if env["world"] == 1:
        backend = "gloo" if env["share"] else "nccl"
        kw = {} if env["share"] else {"device_id": torch.device("cuda", env["local"])}
        with stdout_to_stderr():
            dist.init_process_group(backend, rank=0, world_size=1, init_method="tcp://127.0.0.1:29533", **kw)
            dist.barrier()
    res = sharded_measure(args, cfg, env, args.steps, args.warmup)
    if env["rank"] == 0:
        line = {"metric": METRIC, "higher_is_better": True, "warmup": args.warmup, "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": cfg.name, "image": f"{cfg.width}x{cfg.height}", "k": cfg.k, "init": cfg.init,
                           "parallelism": res.pop("parallelism"), "l2": "flushed (512 MiB write) between timed steps"},
                "cpu_baseline": None, **res}
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


HOSTPOOL = ThreadPoolExecutor(4)  # parity digests and 1-core CPU baselines, overlapped with device work


class stdout_to_stderr:
    """Rank 0's stdout carries the JSON line only: NCCL prints its "NCCL version ..." banner on stdout when
    the first communicator is created, so file descriptor 1 points at stderr while that happens."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def setup_env(args):
    import torch
    import torch.distributed as dist
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # test hook for the multi-rank logic on a one-GPU box: every rank on device 0,
    # gloo instead of NCCL (NCCL refuses two ranks on one device). Not a bench mode.
    share = os.environ.get("CQG_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        with stdout_to_stderr():
            if share:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
                dist.barrier()  # the communicator exists (and has said so) before anything is printed
    return {"world": world, "rank": rank, "local": local, "share": share,
            "dev": torch.device("cuda", local), "stream": torch.cuda.current_stream()}


def summarize(res, cpu):
    """The by_config entry of one workload."""
    rf = res["roofline"]
    return {
        "workload": res["config"]["workload"], "value": res["value"], "unit": UNIT,
        "ms_per_step": res["ms_per_step"], "steps": res["steps"], "n_unique": res["n_unique"],
        "iterations": res["iterations"], "lloyd_distances_per_s": res["lloyd_distances_per_s"],
        "stage_ms_last_step": res["stage_ms_last_step"],
        "lloyd_kernel": {"kernel": rf["kernel"], "achieved_tflops": rf["achieved"], "frac_fp32": rf["frac"],
                         "dense_sweep_frac_fp32": rf["sweep_isolated"]["frac"]},
        "histogram_hbm_frac": res["byte_kernels"]["histogram"]["frac"],
        "pixel_map_hbm_frac": res["byte_kernels"]["pixel_map"]["frac"],
        "byte_kernels": res["byte_kernels"], "e2e": res["e2e"], "cpu_baseline": cpu,
        "parity": res["parity"], "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
        "config": res["config"], "run": res["run"],
        **({"single_image": res["single_image"]} if "single_image" in res else {}),
    }


def resolve(x):
    return x.result() if hasattr(x, "result") else x


def run_ours(args, cfg):
    import torch.distributed as dist
    from paper_1101_0395_b200.synth import CONFIGS
    env = setup_env(args)
    world, rank = env["world"], env["rank"]
    if args.sharded or (world > 1 and cfg.images == 1 and cfg.name in ("cfg5", "cfg3", "cfg3k64")):
        return run_sharded_line(args, cfg, env)
    cpu_on = rank == 0 and world == 1 and not args.no_cpu_baseline
    extra = [] if args.no_by_config or cfg.name not in ("cfg2",) else (
        ["cfg1", "cfg3", "cfg4", "cfg5"] if world == 1 else ["cfg4"])
    cpu_jobs = {}

    def measure_cfg(c, steps, warmup, batch):
        """A single-image config with batch > 1: the single-image run first (per-kernel profile, roofline,
        stage times; reported under single_image), then `batch` copies of the image per step, quantized
        concurrently by several library contexts (as the reference arm runs one copy per host thread)."""
        line = measure(args, c, env, steps, warmup, not args.no_e2e, not args.no_parity)
        if c.images > 1 or batch <= 1:
            return line
        single = line
        line = measure(args, c, env, steps, warmup, not args.no_e2e, not args.no_parity, batch=batch)
        if rank == 0:
            where = ("the single-image steps of this run (one library context on the whole device), timed before "
                     "the batch steps: in a batch several such kernels share the device, each on its SM budget")
            line["single_image"] = {k: single[k] for k in
                                    ("value", "unit", "ms_per_step", "steps", "e2e", "lloyd_distances_per_s",
                                     "stage_ms_last_step", "gpu_launches", "parity", "clocks")}
            line["single_image"]["parity"] = resolve(line["single_image"]["parity"])
            for k in ("kernels", "byte_kernels", "roofline", "dominant_kernel", "stage_ms_last_step",
                      "lloyd_distances_per_s", "flagged_per_step", "swept_fraction"):
                line[k] = single[k]
            line["roofline"]["measured_on"] = where
            line["kernels_measured_on"] = where
            # the batch as a whole: the Lloyd full-sweep FLOP of all its images over the whole step time
            # (every stage of every image in the denominator), against the device's FP32 peak
            rf = line["roofline"]
            flop = 8.0 * line["n_unique"] * c.k * line["iterations"] * batch
            agg = flop / (line["ms_per_step"] / 1e3) / 1e12
            rf["batch_aggregate"] = {"achieved": agg, "frac": agg / rf["peak"], "unit": "TFLOP/s",
                                     "what": "Lloyd full-sweep FLOP (8 N' K iterations) of the batch's images / "
                                             "the whole batch step time, all stages included"}
        return line

    # the headline runs with the host to itself (its batch is driven by 8 host threads); the 1-core
    # reference baselines then run on host threads while the device measures the by_config workloads,
    # the single-stream ones first
    line = measure_cfg(cfg, args.steps, args.warmup, args.batch)
    if cpu_on:
        cpu_jobs[cfg.name] = HOSTPOOL.submit(cpu_baseline, cfg, args.cpu_seconds)
        for name in extra:
            cpu_jobs[name] = HOSTPOOL.submit(cpu_baseline, CONFIGS[name], 0.0)  # one pipeline
    extra = sorted(extra, key=lambda n: n in ("cfg1", "cfg2", "cfg4"))
    by_config = {}
    for name in extra:
        small = name in ("cfg1", "cfg2")
        res = measure_cfg(CONFIGS[name], 10 if small else 3, 3, BATCH_DEFAULT if small else 1)
        if rank == 0:
            by_config[name] = res
    cpp = None
    if rank == 0 and world == 1 and cfg.images == 1 and not args.no_e2e:
        # after the device measurements (its own process and contexts; the GPU is idle here)
        cpp = cpp_dropin(cfg, max(args.batch, 1), args.batch_workers, args.batch_sm_budget)
    if world > 1 and not args.no_by_config and cfg.name == "cfg2":
        res = sharded_measure(args, CONFIGS["cfg5"], env, 3, 3)
        if rank == 0:
            by_config["cfg5_sharded"] = res  # strong scaling of the huge image
    rc = 0
    if rank == 0:
        line["cpu_baseline"] = resolve(cpu_jobs.get(cfg.name))
        if cpp is not None:
            line["cpp_dropin"] = cpp
        line["parity"] = resolve(line["parity"])
        out = {}
        for name, res in by_config.items():
            if "byte_kernels" in res:  # a measure() line (the sharded result is reported as it is)
                res["parity"] = resolve(res["parity"])
                out[name] = summarize(res, resolve(cpu_jobs.get(name)))
            else:
                out[name] = res
        if out:
            line["by_config"] = out
        print(json.dumps(line))
        bad = [n for n, p in [(cfg.name, line["parity"])] + [(n, r.get("parity")) for n, r in out.items()]
               if p is not None and not p["ok"]]
        if bad:
            print("bench: device outputs differ from the oracle on " + ", ".join(bad), file=sys.stderr)
            rc = 1
    if world > 1:
        dist.destroy_process_group()
    return rc


def measure(args, cfg, env, steps, warmup, e2e_on=True, parity_on=True, batch=1):
    """One workload on this rank: W warm-ups, `steps` timed steps (device
    events, L2 flushed between steps, max over ranks), the stage profile, the
    roofline of the dominant kernel, e2e through the C-ABI with pinned host
    buffers, and the oracle parity digest (a future on the host pool).
    Returns the fields of a bench line."""
    import torch
    import torch.distributed as dist
    from paper_1101_0395_b200 import cabi, quant

    world, rank, local, dev, stream = env["world"], env["rank"], env["local"], env["dev"], env["stream"]
    ctx = cabi.Context(local)
    ctx.set_stream(stream.cuda_stream)

    # work owned by this rank
    batch = max(1, batch) if cfg.images == 1 else 1
    if cfg.images > 1:
        my = list(range(rank, cfg.images, world))
    else:
        my = [0] * batch  # `batch` copies of the image in separate buffers, quantized concurrently
    img0 = cfg.image(my[0])
    imgs = [img0 if i == my[0] else cfg.image(i) for i in my]
    ks = [cfg.k_for(i) for i in my]
    P_list = [im.shape[0] * im.shape[1] for im in imgs]
    kind = cabi.INIT_KMEANSPP if cfg.init == "kpp" else cabi.INIT_MAXIMIN

    def mkcfg(k):
        term = cabi.Term(1e-3, 100, cfg.fixed_iterations, 0)
        return cabi.QuantizeCfg(kind, k, cfg.seed, term, 4)

    d_imgs = [torch.from_numpy(im).to(dev) for im in imgs]
    d_idx = [torch.empty(P, dtype=torch.int32, device=dev) for P in P_list]
    d_q = [torch.empty((P, 3), dtype=torch.uint8, device=dev) for P in P_list]
    d_pal = [torch.empty((k, 3), dtype=torch.float64, device=dev) for k in ks]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    # Batches (cfg4): images are independent, so W library contexts, each on
    # its own CUDA stream and driven by its own host thread, quantize them
    # concurrently (the 16-SM cluster initialisers of different images share
    # the GPU; cooperative kernels are chained by the library). One image:
    # one context on the timing stream.
    want = args.workers if cfg.images > 1 else (args.batch_workers if batch > 1 else 1)
    nworkers = max(1, min(want, len(imgs)))
    ctxs, wstreams = [ctx], [stream]
    for _ in range(nworkers - 1):
        c2 = cabi.Context(local)
        s2 = torch.cuda.Stream(device=dev)
        c2.set_stream(s2.cuda_stream)
        ctxs.append(c2)
        wstreams.append(s2)
    if nworkers > 1:
        s0 = torch.cuda.Stream(device=dev)  # worker 0 off the timing stream too
        ctx.set_stream(s0.cuda_stream)
        # each worker's grids (and cooperative kernels) on its own slice of the SMs
        sm_budget = args.sm_budget if cfg.images > 1 else args.batch_sm_budget
        if sm_budget != 0:
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            budget = sm_budget if sm_budget > 0 else sms // nworkers
            for c in ctxs:
                c.set_sm_budget(budget)
            budget_label = f"{budget} SMs each"
        else:
            budget_label = "the whole device each"
        wstreams[0] = s0
    sses = [np.zeros(128) for _ in range(nworkers)]
    pool = ThreadPoolExecutor(nworkers) if nworkers > 1 else None

    def run_batch(srcs, idxs, qs, pals, labs=None):
        # every worker stream starts after the timing stream's current point
        # and the timing stream waits for all of them; labs: per-image buffers
        # for ClusterState::memberships (the e2e run copies them back too)
        lab = (lambda i: labs[i]) if labs is not None else (lambda i: None)
        if nworkers == 1:
            return [ctx.quantize_raw(srcs[i], P_list[i], mkcfg(ks[i]), None, pals[i], lab(i), sses[0],
                                     idxs[i], qs[i]) for i in range(len(imgs))]
        for ws in wstreams:
            ws.wait_stream(stream)

        def work(w):
            return [(i, ctxs[w].quantize_raw(srcs[i], P_list[i], mkcfg(ks[i]), None, pals[i], lab(i),
                                             sses[w], idxs[i], qs[i]))
                    for i in range(w, len(imgs), nworkers)]
        res = dict(kv for part in pool.map(work, range(nworkers)) for kv in part)
        for ws in wstreams:
            stream.wait_stream(ws)
        return [res[i] for i in range(len(imgs))]

    def step_device():
        return run_batch(d_imgs, d_idx, d_q, d_pal)

    # warm-up
    for _ in range(warmup):
        step_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # timed steps: the library as a user runs it (no kernel-level profiling
    # events between its kernels)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_ms, all_stats = [], []
    launches0 = sum(c.launches for c in ctxs)
    with ClockSampler(local) as clk:
        for s in range(steps):
            flush.fill_(s & 255)  # L2 flush outside the timed events
            torch.cuda.synchronize()
            ev0.record(stream)
            st = step_device()
            ev1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            all_stats.append(st)
    gpu_launches = sum(c.launches for c in ctxs) - launches0
    # then the per-kernel profile (CUDA events around the library's kernels on
    # its stream) over separate, untimed steps
    prof_steps = min(steps, 5)
    for c in ctxs:
        c.set_profiling(True)
        c.read_profile(reset=True)
    prof_stats = []
    for s in range(prof_steps):
        flush.fill_(s & 255)
        torch.cuda.synchronize()
        prof_stats.append(step_device())
        torch.cuda.synchronize()
    profs = [c.read_profile(reset=True) for c in ctxs]
    prof = profs[0]
    for extra in profs[1:]:
        for i in range(cabi.PROF_N):
            prof.ms[i] += extra.ms[i]
            prof.units[i] += extra.units[i]
            prof.launches[i] += extra.launches[i]
    for c in ctxs:
        c.set_profiling(False)
    clocks = clk.summary()

    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    total_ms = float(t.item())
    ms_per_step = total_ms / steps
    pixels_per_step_all = cfg.images * P_list[0] if cfg.images > 1 else batch * P_list[0] * world
    value = pixels_per_step_all / (ms_per_step / 1e3) / 1e6

    # Lloyd distances/s (full-sweep equivalent N'.K.iters over Lloyd device time)
    # (stage times come from the profiled steps: the timed ones record no stage events)
    dist_n = sum(s.n_unique * k * s.lloyd.iterations for st in prof_stats for s, k in zip(st, ks))
    lloyd_ms = sum(s.ms_lloyd for st in prof_stats for s in st)
    lloyd_rate = dist_n / (lloyd_ms / 1e3) if lloyd_ms > 0 else None
    if world > 1:
        v = torch.tensor([lloyd_rate or 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(v)
        lloyd_rate = float(v.item())

    # roofline of the dominant kernel (FP32 pipe). Small substrates run the
    # whole Lloyd loop as ONE persistent kernel (lloyd_persistent_kernel): its
    # launch duration is timed over the timed region. Large substrates run the
    # sweep kernel once per iteration inside a CUDA graph: it is timed by
    # back-to-back launches on the final state (cqg_bench_sweep, CUDA events).
    peaks, peak_kind = measured_peaks()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_peak = sms * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    names = ["sweep", "map_sweep", "histogram", "pixel_map", "init", "replay", "ndc", "lloyd_loop", "map_ndc"]
    stage_share = {}
    for i, nm in enumerate(names):
        stage_share[nm] = {"ms_per_step": prof.ms[i] / prof_steps,
                           "launches_per_step": prof.launches[i] / prof_steps}
    iso_ms, iso_units = ctx.bench_sweep(20)
    iso_achieved = 8.0 * iso_units / (iso_ms / 1e3) / 1e12
    persistent = prof.launches[cabi.PROF_SWEEP] == 0 and prof.launches[cabi.PROF_LLOYD] > 0
    # distance evaluations actually performed: swept points x K, plus one
    # own-centre distance per pruned (skipped or tightened) point-iteration
    swept = sum(s.lloyd.swept_total for st in all_stats for s in st)
    pt_iters = sum(s.n_unique * s.lloyd.iterations for st in all_stats for s in st)
    actual_units = sum(s.lloyd.swept_total * k + (s.n_unique * s.lloyd.iterations - s.lloyd.swept_total)
                       for st in all_stats for s, k in zip(st, ks))
    if persistent:
        # 8 FLOP per (colour, centre) pair of a full sweep, N'.K
        # per iteration, counted whether or not pruning skips it
        kname = "lloyd_persistent_kernel (whole Lloyd loop, one launch per run)"
        k_ms = prof.ms[cabi.PROF_LLOYD] / max(int(prof.launches[cabi.PROF_LLOYD]), 1)
        achieved = 8.0 * prof.units[cabi.PROF_LLOYD] / (prof.ms[cabi.PROF_LLOYD] / 1e3) / 1e12
        achieved_actual = 8.0 * actual_units / (prof.ms[cabi.PROF_LLOYD] / 1e3) / 1e12
        k_share = prof.ms[cabi.PROF_LLOYD] / prof_steps / ms_per_step
    else:
        kname = "sweep_kernel<WALK> (Lloyd assignment, one launch per iteration)"
        k_ms = iso_ms
        achieved = iso_achieved
        achieved_actual = iso_achieved
        iters_all = sum(s.lloyd.iterations for st in all_stats for s in st)
        k_share = iso_ms * iters_all / steps / ms_per_step  # iterations summed over the timed steps
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("dominant_dram_bytes_per_launch")
    roofline = {
        "bound": "fp32", "kernel": kname,
        "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
        "frac": (achieved / fp32_peak) if achieved else None, "traffic": traffic,
        "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 x sm_max_mhz ({peak_kind} MEASURED_PEAKS.json)",
        "algorithmic_unit": ("SURVEY.md 8(d): 8 FP32 FLOP per (unique colour, centre) pair of a full "
                             "sweep, N'.K per iteration, counted whether or not pruning skips it; the "
                             "isolated sweep is the dense N'.K launch"),
        "achieved_actual_work": achieved_actual,  # distances actually evaluated (pruned ones excluded)
        "avg_launch_ms": k_ms,
        "launch_share_of_step": k_share,
        "concurrent_streams": nworkers,  # > 1: shares sum device time over concurrent streams
        "sweep_isolated": {"ms_per_launch": iso_ms, "achieved": iso_achieved,
                           "frac": iso_achieved / fp32_peak, "units_per_launch": iso_units},
    }
    # the kernel with the largest device-time share, when it is not the Lloyd kernel
    dominant = None
    share = {nm: prof.ms[i] / prof_steps / ms_per_step for i, nm in enumerate(names)}
    top = max(share, key=share.get)
    if top == "init" and share["init"] > k_share:
        K0 = ks[0]
        init_ms = prof.ms[cabi.PROF_INIT] / max(int(prof.launches[cabi.PROF_INIT]), 1)
        nu = all_stats[-1][0].n_unique
        small = nu <= 16 * 1024 * 12
        tiled = nu >= (1 << 20)
        dominant = {
            "kernel": ("init_cluster_reg_kernel (16-CTA cluster, register-resident points)" if small
                       else "init_kernel_tile (colour-space tiles, box-pruned rounds)" if tiled
                       else "init_kernel_rec (cooperative grid, in-place records)"),
            "share_of_step": share["init"], "avg_launch_ms": init_ms,
            "bound": "latency" if small or tiled else "hbm",
            "rounds": K0 - 1,
            "us_per_round": 1e3 * init_ms / max(K0 - 1, 1),
            "note": ("a chain of K-1 dependent draws; CTA sums and the pick travel by st.async with mbarrier "
                     "transaction signalling (no cluster barriers); per-round critical path "
                     "(tools/init_timing.py): update ~32%, publish ~15%, draw (wait for sums, locate, "
                     "pick broadcast) ~42%, tail ~11%") if small else
                    ("a round updates only the tiles the new centre can reach; block 0 locates the draw and "
                     "releases the others; see DESIGN.md section 4/8") if tiled else
                    "8 B per point per round streamed; see DESIGN.md section 8",
        }
    hist_ms = prof.ms[cabi.PROF_HIST]
    pix_ms = prof.ms[cabi.PROF_PIXEL]
    hbm = peaks.get("hbm_gbs", 6545.6)
    n_unique = all_stats[-1][0].n_unique
    hist_gbs = ((prof.units[cabi.PROF_HIST] + 8.0 * n_unique * prof_steps * len(imgs)) / (hist_ms / 1e3) / 1e9
                if hist_ms else None)
    pix_gbs = prof.units[cabi.PROF_PIXEL] / (pix_ms / 1e3) / 1e9 if pix_ms else None
    byte_kernels = {  # algorithmic bytes: histogram 3P + 8N', pixel map 3P in + 7P out
        "histogram": {"achieved_gbs": hist_gbs, "peak_gbs": hbm, "frac": hist_gbs / hbm if hist_gbs else None,
                      "ms_per_step": hist_ms / prof_steps},
        "pixel_map": {"achieved_gbs": pix_gbs, "peak_gbs": hbm, "frac": pix_gbs / hbm if pix_gbs else None,
                      "ms_per_step": pix_ms / prof_steps},
    }

    # end-to-end through the C-ABI with pinned HOST buffers (H2D + D2H inside the timed region)
    e2e = None
    if e2e_on:
        h_imgs = [torch.from_numpy(im).pin_memory() for im in imgs]
        h_idx = [torch.empty(P, dtype=torch.int32).pin_memory() for P in P_list]
        h_q = [torch.empty((P, 3), dtype=torch.uint8).pin_memory() for P in P_list]
        h_pal = [np.empty((k, 3)) for k in ks]
        h_lab = [torch.empty(P, dtype=torch.int32).pin_memory() for P in P_list]  # N' <= P memberships
        for _ in range(max(1, warmup // 2)):
            run_batch(h_imgs, h_idx, h_q, h_pal, h_lab)
        e_ms = []
        for s in range(steps):
            flush.fill_(s & 255)
            torch.cuda.synchronize()
            ev0.record(stream)
            run_batch(h_imgs, h_idx, h_q, h_pal, h_lab)
            ev1.record(stream)
            torch.cuda.synchronize()
            e_ms.append(ev0.elapsed_time(ev1))
        et = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_step = float(et.item()) / steps
        h2d = sum(3 * P for P in P_list)
        # indices (u32) + quantized RGB + palette + SSE trace + memberships (u32 per distinct colour)
        nus = [st.n_unique for st in all_stats[-1]] if len(all_stats[-1]) == len(P_list) else [P for P in P_list]
        d2h = sum(7 * P + 24 * k + 8 * 100 + 4 * nu for P, k, nu in zip(P_list, ks, nus))
        e2e = {"value": pixels_per_step_all / (e_step / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e_step,
               "index_layout": "uint32 per pixel (MappingResult::indices)"}

    # a batch holds copies of one image: every copy's outputs must equal image 0's
    batch_equal = None
    if batch > 1:
        torch.cuda.synchronize()
        batch_equal = all(torch.equal(d_pal[i], d_pal[0]) and torch.equal(d_idx[i], d_idx[0]) and
                          torch.equal(d_q[i], d_q[0]) for i in range(1, len(imgs)))
        if not batch_equal:
            raise RuntimeError("bench: the copies of a batch disagree with each other")

    # parity digest of the last timed step's outputs (image 0 of this rank)
    # against the C oracle (exact-moment mode): palette bytes, iterations,
    # NDC, mapping indices / pixels / MSE / mapping NDC. A mismatch fails the run.
    parity = None
    if rank == 0 and parity_on:
        outs = (d_pal[0].cpu().numpy(), d_idx[0].cpu().numpy().view(np.uint32), d_q[0].cpu().numpy().reshape(-1, 3))
        parity = HOSTPOOL.submit(parity_digest, cfg, imgs[0], ks[0], my[0], all_stats[-1][0], *outs)

    line = None
    if rank == 0:
        st0 = all_stats[-1][0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if cfg.images == 1 else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(cfg, len(imgs) if cfg.images == 1 else cfg.images),
            "run": {"images_per_rank": len(imgs),
                    "parallelism": ((f"replicas x{world}" if cfg.images == 1 else f"images sharded over {world}") +
                                    (f"; {nworkers} concurrent library contexts per GPU, {budget_label}"
                                     if nworkers > 1 else "; one library context on the whole device")),
                    "l2": "flushed (512 MiB write) between timed steps",
                    "arithmetic": "FP32 packed sweep + exact FP64 replay of near-ties + int64 moments",
                    "index_layout": "uint32 per pixel", "batch_copies_equal": batch_equal},
            "lloyd_distances_per_s": lloyd_rate,
            "n_unique": int(st0.n_unique), "iterations": int(st0.lloyd.iterations),
            "flagged_per_step": int(st0.lloyd.flagged_total),
            "swept_fraction": swept / pt_iters if pt_iters else None,
            "stage_ms_last_step": {"histogram": prof_stats[-1][0].ms_histogram, "init": prof_stats[-1][0].ms_init,
                                   "lloyd": prof_stats[-1][0].ms_lloyd, "map": prof_stats[-1][0].ms_map,
                                   "note": "from a profiled step (stage events), not a timed one"},
            "kernels": stage_share, "byte_kernels": byte_kernels,
            "roofline": roofline, "dominant_kernel": dominant, "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": int(gpu_launches), "clocks": clocks, "parity": parity,
        }
    if pool:
        pool.shutdown()
    for c in ctxs[1:]:
        c.close()
    ctx.close()
    return line




def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sm-budget", type=int, default=24,
                    help="batched configs: SMs per worker context (-1: SMs / workers, 0: whole device each); "
                         "measured on cfg4: 4 x 37 SMs 608, 8 x 37 880, 16 x 24 982 MPixel/s")
    ap.add_argument("--workers", type=int, default=16,
                    help="batched configs: concurrent library contexts (streams + host threads) per GPU")
    ap.add_argument("--batch", type=int, default=None,
                    help="single-image configs: copies of the image per step, quantized concurrently "
                         "(default: 16 for cfg1 / cfg2, as many as the reference arm's images per step; 1 otherwise)")
    ap.add_argument("--batch-workers", type=int, default=8,
                    help="concurrent library contexts (streams + host threads) for --batch")
    ap.add_argument("--batch-sm-budget", type=int, default=32,
                    help="SMs per library context for --batch (0: whole device each); the budgets may oversubscribe "
                         "the device: kernels of different stages interleave")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle digest of the outputs")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sharded", action="store_true",
                    help="run a single-image config through the colour-sharded multi-GPU path")
    ap.add_argument("--no-by-config", action="store_true",
                    help="skip the by_config measurements (cfg3 / cfg5 at N=1; cfg4 and sharded cfg5 at N>1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched as `python bench.py --gpus N`: start the N ranks ourselves
        # (one process per GPU, torch.distributed over NCCL, rendezvous on 127.0.0.1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "ours" and env_int("WORLD_SIZE", 1) != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={env_int('WORLD_SIZE', 1)}", file=sys.stderr)
        return 2
    from paper_1101_0395_b200.synth import CONFIGS
    cfg = CONFIGS[args.config]
    if args.batch is None:
        args.batch = BATCH_DEFAULT if cfg.name in ("cfg1", "cfg2") else 1
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
