"""QuantizeConfig::sampling on the device (
pipeline.cpp:91-116, histogram.cpp:60-67) against the reference library.

  unique  distinct colours of the image, count weights          (the default)
  none    every pixel is a point, weight 1/P
  2to1    every pixel at even (x, y) is a point, weight 1/S
  both    distinct colours of the 2:1 subsample, count weights

Initialisers read the histogram of the sampled pixels; the mapping covers the
full image. Bar: iterations and NDC bit-exact, palette bit-exact when the
substrate's pixel count S is a power of two (else |d| <= 1e-9), MSE 1e-12
relative; mapping outputs bit-exact vs the exact oracle on the same palette.
"""
import numpy as np
import pytest

from oracle.pyoracle import UPDATE_EXACT
from paper_1101_0395_b200 import quant
from paper_1101_0395_b200.synth import synth_image

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["none", "2to1", "unique", "both"])
@pytest.mark.parametrize("method,w,h,k,seed", [("wsm-mmx", 128, 128, 16, 5), ("wsm-kpp", 128, 128, 24, 8),
                                               ("wsm-kpp", 97, 61, 12, 3)])
def test_sampling_vs_reference(ctx, oracle, reflib, mode, method, w, h, k, seed):
    img = synth_image(w, h, seed, nblobs=6, sigma=18.0, noise=0.05)
    qc = quant.QuantizeConfig(method=quant.parse_method(method), k=k, seed=seed, sampling=mode)
    r = quant.run_quantize(img, qc, ctx=ctx)
    ref = reflib.run_quantize(img, w, h, method, k, seed, sampling=mode)
    S = ((w + 1) // 2) * ((h + 1) // 2) if mode in ("2to1", "both") else w * h
    assert r.report.iterations == ref["iterations"]
    assert r.report.ndc_per_point_iter == ref["ndc_per_point_iter"]
    if S & (S - 1) == 0:
        assert np.array_equal(r.palette, ref["palette"])
    else:
        assert np.max(np.abs(r.palette - ref["palette"])) <= 1e-9
    assert abs(r.report.mse - ref["mse"]) <= 1e-12 * ref["mse"]
    assert r.report.sampling == mode
    # the substrate: every sampled pixel in the raw modes
    if mode in ("none", "2to1"):
        assert r.substrate_points == S == r.state.memberships.size
    idx, q, mse_e, _ = oracle.map_pixels(img, r.palette, mode=UPDATE_EXACT)
    assert np.array_equal(r.mapping.indices, idx)
    assert np.array_equal(r.mapping.quantized.reshape(-1, 3), q)
    assert r.report.mse == mse_e


def test_sampling_raw_labels_match_the_oracle(ctx, oracle):
    # 'none': the Lloyd substrate is the pixel list itself (duplicates included)
    w, h, k, seed = 64, 48, 10, 2
    img = synth_image(w, h, seed, nblobs=5, sigma=15.0, noise=0.02)
    qc = quant.QuantizeConfig(method=quant.parse_method("wsm-mmx"), k=k, seed=seed, sampling="none")
    r = quant.run_quantize(img, qc, ctx=ctx)
    px = quant.pack_colors(img.reshape(-1, 3))
    hist = quant.build_histogram(img, ctx=ctx)
    init = oracle.init_maximin(hist.packed, hist.counts, w * h, k, seed)
    ora = oracle.wsm(px, np.ones(px.size, np.uint32), w * h, init, mode=UPDATE_EXACT)
    assert np.array_equal(r.state.memberships, ora.labels)
    assert np.array_equal(r.palette.view(np.uint64), ora.centers.view(np.uint64))
    assert r.report.iterations == ora.iterations


def test_sampling_validation(ctx):
    img = synth_image(16, 16, 1)
    with pytest.raises(ValueError, match="unknown sampling mode"):
        quant.run_quantize(img, quant.QuantizeConfig(k=4, sampling="fancy"), ctx=ctx)
