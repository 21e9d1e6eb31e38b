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
