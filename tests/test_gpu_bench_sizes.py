"""Parity at the bench sizes: the full device pipeline (cqg_quantize through
quant.run_quantize) on BASELINE.json's large configurations, against the C
oracle in exact-moment mode and against the reference library itself
(oracle/_ref, the reference's sources compiled in place).

  cfg3     4096^2, 64 blobs + 10% noise, K=256 maximin        (6.3M colours)
  cfg3k64  same image, K=64 maximin
  cfg4     four 768x512 batch images, K = 32/64/128/256, maximin, run through
           four SM-budgeted contexts side by side (the bench's batch layout)
  cfg5     8192^2 uniform noise, K=256 k-means++, 20 fixed iterations (16.47M colours)

Every output is compared: histogram (colours, counts, first index), initial
centres, final labels, iterations, ndc_total, repairs, centres, sse_trace,
mapping indices, quantized pixels, MSE and the mapping NDC.
Bar: bit-exact against the exact-moment oracle; against the
reference: labels, iterations, NDC, histogram, init centres, mapping indices
and pixels bit-exact, centres bit-exact when P is a power of two (else
|d| <= 1e-9), SSE trace and MSE within the rigorous error bound of the reference's recursive FP64
sums of n non-negative terms, (n-1)u with u = 2^-53 (Higham 2002, 4.3;
floored at 1e-12): kmeans.cpp:107-114 sums N' terms, metrics.cpp:51 sums P.
The oracle and the reference run on host threads while the device computes.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle.pyoracle import UPDATE_EXACT
from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import CONFIGS

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


U = 2.0 ** -53


def seq_tol(n):
    """Relative error bound of a recursive FP64 sum of n non-negative terms."""
    return max(1e-12, (n - 1) * U)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def oracle_pipeline(O, img, k, init, seed, fixed):
    P = img.shape[0] * img.shape[1]
    c, n, f = O.histogram(img)
    c0 = O.init_kmeanspp(c, n, P, k, seed) if init == "kpp" else O.init_maximin(c, n, P, k, seed)
    r = O.wsm(c, n, P, c0, fixed_it=fixed, mode=UPDATE_EXACT)
    idx, q, mse, ndc = O.map_pixels(img, r.centers, mode=UPDATE_EXACT)
    return dict(colors=c, counts=n, first=f, init=c0, wsm=r, idx=idx, q=q, mse=mse, map_ndc=ndc)


def ref_pipeline(R, img, k, init, seed, fixed):
    h, w = img.shape[:2]
    P = w * h
    c, n, _ = R.histogram(img)
    c0 = R.init(init, c, n, P, k, seed)
    r = R.wsm(c, n, P, c0, fixed_it=fixed)
    idx, q, mse, ndc = R.map_pixels(img, w, h, r.centers)
    return dict(colors=c, counts=n, init=c0, wsm=r, idx=idx, q=q, mse=mse, map_ndc=ndc)


def device_pipeline(ctx, img, k, init, seed, fixed):
    hist = quant.build_histogram(img, ctx=ctx)
    sc = quant.SeedConfig(k=k, seed=seed)
    c0 = quant.init_kmeanspp(hist, sc, ctx=ctx) if init == "kpp" else quant.init_maximin(hist, sc, ctx=ctx)
    cfg = quant.QuantizeConfig(method=quant.parse_method("wsm-" + init), k=k, seed=seed,
                               term=quant.Termination(fixed_iterations=fixed or None))
    r = quant.run_quantize(img, cfg, ctx=ctx)
    return hist, c0, r


def check_against_oracle(hist, c0, r, o):
    assert hist.size() == o["colors"].size
    assert np.array_equal(hist.packed, o["colors"])
    assert np.array_equal(hist.counts, o["counts"])
    assert np.array_equal(hist.first, o["first"])
    assert np.array_equal(c0.view(np.uint64), o["init"].view(np.uint64))
    w = o["wsm"]
    assert r.substrate_points == o["colors"].size
    assert r.state.iterations == w.iterations
    assert r.state.ndc_total == w.ndc_total
    assert r.state.repair_count == w.repairs
    assert np.array_equal(r.state.memberships, w.labels)
    assert np.array_equal(r.palette.view(np.uint64), w.centers.view(np.uint64))
    assert np.array_equal(r.state.sse_trace.view(np.uint64), w.sse_trace.view(np.uint64))
    assert np.array_equal(r.mapping.indices, o["idx"])
    assert np.array_equal(r.mapping.quantized.reshape(-1, 3), o["q"])
    assert r.report.mse == o["mse"]
    assert r.mapping.ndc == o["map_ndc"]


def check_against_reference(hist, c0, r, ref, P):
    assert np.array_equal(hist.packed, ref["colors"])
    assert np.array_equal(hist.counts, ref["counts"])
    assert np.array_equal(c0, ref["init"])
    w = ref["wsm"]
    assert r.state.iterations == w.iterations
    assert r.state.ndc_total == w.ndc_total
    assert r.state.repair_count == w.repairs
    assert np.array_equal(r.state.memberships, w.labels)
    if P & (P - 1) == 0:
        assert np.array_equal(r.palette, w.centers)
    else:
        assert np.max(np.abs(r.palette - w.centers)) <= 1e-9
    assert rel(r.state.sse_trace, w.sse_trace) <= seq_tol(r.substrate_points)
    assert np.array_equal(r.mapping.indices, ref["idx"])
    assert np.array_equal(r.mapping.quantized.reshape(-1, 3), ref["q"])
    assert rel(r.report.mse, ref["mse"]) <= seq_tol(P)
    assert r.mapping.ndc == ref["map_ndc"]


@pytest.mark.parametrize("name", ["cfg3", "cfg3k64", "cfg5"])
def test_single_image_bench_size(ctx, oracle, reflib, name):
    cfg = CONFIGS[name]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    fixed = cfg.fixed_iterations
    with ThreadPoolExecutor(2) as ex:
        fo = ex.submit(oracle_pipeline, oracle, img, cfg.k, cfg.init, cfg.seed, fixed)
        fr = ex.submit(ref_pipeline, reflib, img, cfg.k, cfg.init, cfg.seed, fixed)
        hist, c0, r = device_pipeline(ctx, img, cfg.k, cfg.init, cfg.seed, fixed)
        o, ref = fo.result(), fr.result()
    check_against_oracle(hist, c0, r, o)
    check_against_reference(hist, c0, r, ref, P)
    if fixed:
        assert r.state.iterations == fixed


def test_batch_images_budgeted_contexts(oracle, reflib):
    """cfg4: one image per K in {32, 64, 128, 256}, four budgeted contexts on
    their own streams and host threads (the bench's batch layout)."""
    cfg = CONFIGS["cfg4"]
    ids = [0, 1, 2, 3]
    imgs = [cfg.image(i) for i in ids]
    ks = [cfg.k_for(i) for i in ids]
    assert sorted(ks) == [32, 64, 128, 256]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctxs, streams = [], []
    for _ in ids:
        c = cabi.Context(0)
        s = torch.cuda.Stream()
        c.set_stream(s.cuda_stream)
        c.set_sm_budget(sms // len(ids))
        ctxs.append(c)
        streams.append(s)
    with ThreadPoolExecutor(len(ids)) as ex:
        dev = list(ex.map(lambda j: device_pipeline(ctxs[j], imgs[j], ks[j], cfg.init, cfg.seed, 0),
                          range(len(ids))))
    with ThreadPoolExecutor(8) as ex:
        fo = [ex.submit(oracle_pipeline, oracle, imgs[j], ks[j], cfg.init, cfg.seed, 0) for j in range(len(ids))]
        fr = [ex.submit(ref_pipeline, reflib, imgs[j], ks[j], cfg.init, cfg.seed, 0) for j in range(len(ids))]
        for j in range(len(ids)):
            hist, c0, r = dev[j]
            P = imgs[j].shape[0] * imgs[j].shape[1]
            check_against_oracle(hist, c0, r, fo[j].result())
            check_against_reference(hist, c0, r, fr[j].result(), P)
    for c in ctxs:
        c.close()
