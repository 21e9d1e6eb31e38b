"""Batched quantisation (the cfg4 shape) with several library contexts, each on
its own CUDA stream and host thread and restricted to a slice of the SMs
(cqg_set_sm_budget), so their cooperative kernels -- the persistent Lloyd
loop and the grid initialisers -- run side by side. Every image's outputs
must equal a whole-device context's, bit for bit.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import synth_image

pytestmark = pytest.mark.gpu


def test_budgeted_contexts_side_by_side(ctx):
    imgs = [synth_image(768, 512, 300 + i, nblobs=12 + 3 * i, sigma=20.0, noise=0.12) for i in range(8)]
    ks = [32, 64, 128, 256] * 2
    cfgs = [quant.QuantizeConfig(method=quant.parse_method("wsm-mmx" if i % 2 else "wsm-kpp"), k=k, seed=i)
            for i, k in enumerate(ks)]
    ref = [quant.run_quantize(im, c, ctx=ctx) for im, c in zip(imgs, cfgs)]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    workers = 4
    ctxs, streams = [], []
    for _ in range(workers):
        c = cabi.Context(0)
        s = torch.cuda.Stream()
        c.set_stream(s.cuda_stream)
        c.set_sm_budget(sms // workers)
        ctxs.append(c)
        streams.append(s)

    def work(w):
        return [(i, quant.run_quantize(imgs[i], cfgs[i], ctx=ctxs[w])) for i in range(w, len(imgs), workers)]

    with ThreadPoolExecutor(workers) as ex:
        out = dict(kv for part in ex.map(work, range(workers)) for kv in part)
    for i, r0 in enumerate(ref):
        r = out[i]
        assert r.substrate_points == r0.substrate_points
        assert r.state.iterations == r0.state.iterations
        assert r.state.ndc_total == r0.state.ndc_total
        assert np.array_equal(r.palette, r0.palette)
        assert np.array_equal(r.state.memberships, r0.state.memberships)
        assert np.array_equal(r.mapping.indices, r0.mapping.indices)
        assert r.report.mse == r0.report.mse
    for c in ctxs:
        c.close()


def test_sm_budget_validation(ctx):
    with pytest.raises(cabi.CqgError):
        ctx.set_sm_budget(-1)
    ctx.set_sm_budget(0)  # whole device


def test_oversubscribed_contexts_batch_of_copies(ctx, oracle):
    # the bench's cfg2 shape: copies of one image through more contexts than the
    # SM budgets leave room for (8 x 32 SMs), outputs into pageable host arrays
    # (small results travel through the pinned bounce buffer, api.cu copy_out)
    # and into device buffers; every copy must equal the oracle's result
    from oracle.pyoracle import UPDATE_EXACT
    img = synth_image(320, 256, 77, nblobs=14, sigma=12.0, noise=0.02)
    P, K = 320 * 256, 64
    c, n, _ = oracle.histogram(img)
    init = oracle.init_kmeanspp(c, n, P, K, 5)
    ref = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT)
    ridx, rq, rmse, _ = oracle.map_pixels(img, ref.centers, mode=UPDATE_EXACT)
    workers, copies = 8, 16
    ctxs = []
    for _ in range(workers):
        cx = cabi.Context(0)
        s = torch.cuda.Stream()
        cx.set_stream(s.cuda_stream)
        cx.set_sm_budget(32)
        ctxs.append((cx, s))
    qc = cabi.QuantizeCfg(cabi.INIT_KMEANSPP, K, 5, cabi.Term(1e-3, 100, 0, 0), 4)
    host = [i % 2 == 0 for i in range(copies)]
    src = [torch.from_numpy(img) if h else torch.from_numpy(img).cuda() for h in host]
    pal = [np.empty((K, 3)) if h else torch.empty((K, 3), dtype=torch.float64, device="cuda") for h in host]
    idx = [np.empty(P, np.uint32) if h else torch.empty(P, dtype=torch.int32, device="cuda") for h in host]
    q = [np.empty((P, 3), np.uint8) if h else torch.empty((P, 3), dtype=torch.uint8, device="cuda") for h in host]
    lab = [np.empty(P, np.uint32) if h else None for h in host]

    def work(w):
        cx, _ = ctxs[w]
        sse = np.zeros(128)
        return [(i, cx.quantize_raw(src[i], P, qc, None, pal[i], lab[i], sse, idx[i], q[i]), sse[:ref.iterations].copy())
                for i in range(w, copies, workers)]

    for _ in range(2):  # the second round runs on warm contexts
        with ThreadPoolExecutor(workers) as ex:
            out = [r for part in ex.map(work, range(workers)) for r in part]
    torch.cuda.synchronize()
    for i, st, sse in out:
        assert st.n_unique == c.size and st.lloyd.iterations == ref.iterations
        assert st.lloyd.ndc_total == ref.ndc_total
        p = pal[i] if host[i] else pal[i].cpu().numpy()
        assert np.array_equal(p, ref.centers)
        assert np.array_equal(sse, np.asarray(ref.sse_trace)[:ref.iterations])
        ii = idx[i] if host[i] else idx[i].cpu().numpy().view(np.uint32)
        assert np.array_equal(ii, ridx)
        qq = q[i] if host[i] else q[i].cpu().numpy()
        assert np.array_equal(qq.reshape(-1, 3), rq)
        assert st.mean_sq_dist == rmse
        if host[i]:
            assert np.array_equal(lab[i][:c.size], ref.labels)
    for cx, _ in ctxs:
        cx.close()
