"""Pin the CPU oracle (oracle/cq_oracle.c) against the reference's golden
vectors before trusting it as the GPU checker.

* sweep_a rows: proj/tmp_acceptance/sweep_a.csv:2-13 (committed as
  tests/golden/sweep_a_rows.csv by tests/golden/make_golden.py, which asserts
  it reproduces the reference file byte for byte).
* ref_cases.json: centres / SSE trace / labels / NDC / mapping of the reference
  build on three small cases.
* When oracle/_ref is built (this container), the oracle is also compared with
  the reference library on seeded larger inputs.
"""
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import UPDATE_EXACT, UPDATE_REFERENCE

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load_img(seed):
    return np.fromfile(os.path.join(GOLD, f"acc_{seed}.rgb"), dtype=np.uint8).reshape(40, 40, 3)


def golden_rows():
    with open(os.path.join(GOLD, "sweep_a_rows.csv")) as f:
        lines = f.read().strip().split("\n")
    return lines[0], lines[1:]


def csv_row(image, method, k, run, seed, mse, psnr, iters, ndc_ppi):
    return ",".join([image, method, str(k), str(run), str(seed), "unique", "%.6f" % mse,
                     "%.4f" % psnr, str(iters), "%.4f" % ndc_ppi, "0.000", str(k), ""])


def oracle_row(O, img_seed, method, run, mode):
    img = load_img(img_seed)
    seed = 3 + run
    colors, counts, _ = O.histogram(img)
    P = 1600
    if method == "wsm-kpp":
        init = O.init_kmeanspp(colors, counts, P, 8, seed)
    else:
        with open(os.path.join(GOLD, "wu_init.json")) as f:
            init = np.array(json.load(f)[str(img_seed)])
    res = O.wsm(colors, counts, P, init, mode=mode)
    _, _, mse, _ = O.map_pixels(img, res.centers, mode=mode)
    return csv_row(f"acc_{img_seed}.ppm", method, 8, run, seed, mse, O.psnr(mse), res.iterations,
                   res.ndc_per_point_iter())


@pytest.mark.parametrize("mode", [UPDATE_REFERENCE, UPDATE_EXACT])
def test_oracle_reproduces_sweep_a_rows(oracle, mode):
    _, rows = golden_rows()
    want = {r for r in rows if ",wu," not in r}
    got = set()
    for img_seed in (61, 62):
        for method in ("wsm-kpp", "wsm-wu"):
            for run in (0, 1):
                got.add(oracle_row(oracle, img_seed, method, run, mode))
    assert got == want


def test_oracle_matches_reference_cases_bitwise(oracle):
    with open(os.path.join(GOLD, "ref_cases.json")) as f:
        cases = json.load(f)
    for c in cases:
        img = load_img(c["image"])
        colors, counts, _ = oracle.histogram(img)
        assert colors.tolist() == c["hist_colors"]
        assert counts.tolist() == c["hist_counts"]
        K = c["k"]
        if c["init"] == "kpp":
            init = oracle.init_kmeanspp(colors, counts, 1600, K, c["seed"])
        else:
            init = oracle.init_maximin(colors, counts, 1600, K, c["seed"])
        assert [float(v).hex() for v in init.reshape(-1)] == c["init_centers"]
        r = oracle.wsm(colors, counts, 1600, init, mode=UPDATE_REFERENCE, history=True)
        assert [float(v).hex() for v in r.centers.reshape(-1)] == c["centers"]
        assert [float(v).hex() for v in r.sse_trace] == c["sse_trace"]
        assert r.iterations == c["iterations"]
        assert r.ndc_total == c["ndc_total"]
        assert r.labels.tolist() == c["labels"]
        assert r.hist_labels.tolist() == c["history_labels"]
        idx, _, mse, mndc = oracle.map_pixels(img, r.centers, mode=UPDATE_REFERENCE)
        assert idx.tolist() == c["map_indices"]
        assert float(mse).hex() == c["map_mse"]
        assert mndc == c["map_ndc"]  # MappingResult::ndc (metrics.cpp:36-48)
        # exact-moment mode: same trajectory; P = 1600 is not a power of two so
        # centres may differ in the last bits, SSE within 1e-12
        e = oracle.wsm(colors, counts, 1600, init, mode=UPDATE_EXACT, history=True)
        assert e.iterations == c["iterations"] and e.ndc_total == c["ndc_total"]
        assert e.hist_labels.tolist() == c["history_labels"]
        ref_sse = np.array([float.fromhex(v) for v in c["sse_trace"]])
        assert np.max(np.abs(e.sse_trace - ref_sse) / ref_sse) < 1e-12
        ref_c = np.array([float.fromhex(v) for v in c["centers"]])
        assert np.max(np.abs(e.centers.reshape(-1) - ref_c)) < 1e-9


def test_oracle_histogram_reference_case(oracle):
    # tests/test_histogram.cpp:102-118
    A, B, C = (10, 20, 30), (200, 100, 50), (0, 0, 0)
    img = np.array([A, B, A, C, B, A], np.uint8)
    colors, counts, first = oracle.histogram(img)
    assert colors.tolist() == [0x0A141E, 0xC86432, 0]
    assert counts.tolist() == [3, 2, 1]
    assert first.tolist() == [0, 1, 3]
    w = oracle.weights(counts, 6)
    assert w[0] == 0.5


def test_oracle_rng_matches_std_mt19937_64(oracle):
    # std::mt19937_64 default-seed (5489) 10000th output is 9981545732273789042
    r = oracle.rng(5489)
    for _ in range(9999):
        oracle.L.cqo_rng_u64(r)
    assert oracle.L.cqo_rng_u64(r) == 9981545732273789042


@pytest.mark.parametrize("seed,K,kind", [(7, 16, "kpp"), (8, 32, "mmx"), (9, 64, "kpp")])
def test_oracle_vs_reference_library(oracle, reflib, seed, K, kind):
    from paper_1101_0395_b200.synth import synth_image
    img = synth_image(128, 96, seed, nblobs=6, sigma=10.0, noise=0.01)
    P = 128 * 96
    colors, counts, first = oracle.histogram(img)
    rc, rn, rw = reflib.histogram(img, seed)
    assert np.array_equal(colors, rc) and np.array_equal(counts, rn)
    assert np.array_equal(oracle.weights(counts, P), rw)
    init = (oracle.init_kmeanspp if kind == "kpp" else oracle.init_maximin)(colors, counts, P, K, seed)
    assert np.array_equal(init, reflib.init(kind, colors, counts, P, K, seed))
    a = oracle.wsm(colors, counts, P, init, mode=UPDATE_REFERENCE, history=True)
    b = reflib.wsm(colors, counts, P, init, history=True)
    assert np.array_equal(a.centers, b.centers)
    assert np.array_equal(a.sse_trace, b.sse_trace)
    assert np.array_equal(a.hist_labels, b.hist_labels)
    assert a.ndc_total == b.ndc_total and a.repairs == b.repairs
    i1, q1, m1, n1 = oracle.map_pixels(img, b.centers, mode=UPDATE_REFERENCE)
    i2, q2, m2, n2 = reflib.map_pixels(img, 128, 96, b.centers)
    assert np.array_equal(i1, i2) and np.array_equal(q1, q2) and m1 == m2 and n1 == n2
