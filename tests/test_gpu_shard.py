"""The CUDA shard engine (cqg_shard_* through parallel.CudaShardEngine).

* two engines on one GPU (two contexts, two colour slices) driven in lockstep
  with a host-side sum standing in for the allreduce (the kernels never wait on
  each other, so this is safe on one device), incl. the repair protocol;
* the real parallel.sharded_wsm over a 1-rank NCCL group.
Both must match the single-process exact-moment oracle bit for bit."""
import os
import socket

import numpy as np
import pytest

from oracle.pyoracle import UPDATE_EXACT
from paper_1101_0395_b200 import cabi, parallel
from paper_1101_0395_b200.synth import synth_image

pytestmark = pytest.mark.gpu


def case(oracle, seed, K, w=160, h=120, adversarial=False):
    img = synth_image(w, h, seed, nblobs=8, sigma=11.0, noise=0.03)
    colors, counts, _ = oracle.histogram(img)
    P = w * h
    init = (np.full((K, 3), 128.0) if adversarial
            else oracle.init_kmeanspp(colors, counts, P, K, seed))
    return colors, counts, P, init


def lockstep(engines, slices, colors, counts, P, init, K, term):
    import torch
    for e, (lo, hi) in zip(engines, slices):
        e.begin(colors[lo:hi], counts[lo:hi], P, init, K, term)
    ndc = rep = 0
    while True:
        glob = sum(e.assign().cpu() for e in engines)
        ndc += int(glob[5 * K])
        states = [e.finalize(glob.cuda())[0] for e in engines]
        assert len(set(states)) == 1
        while states[0] == parallel.STATE_EMPTY:
            gs = sum(e.sizes().cpu() for e in engines)
            while (gs == 0).any():
                ee = int((gs == 0).nonzero()[0])
                cands = []
                for r, (e, (lo, hi)) in enumerate(zip(engines, slices)):
                    v, li, col, lab = e.donor(gs, False)
                    cands.append((v, (lo + li) if li is not None else 1 << 60, r, li, col, lab))
                v, gi, r, li, col, lab = max(cands, key=lambda t: (t[0], -t[1]))
                assert v > 0
                for rr, e in enumerate(engines):
                    e.move(li if rr == r else None, ee, col)
                gs[lab] -= 1
                gs[ee] += 1
                rep += 1
            glob = sum(e.moments().cpu() for e in engines)
            states = [e.finalize(glob.cuda())[0] for e in engines]
        if states[0] == parallel.STATE_DONE:
            break
    outs = [e.end(term.max_iterations) for e in engines]
    return outs, ndc, rep


@pytest.mark.parametrize("seed,K,adv", [(7, 32, False), (8, 16, True)])
def test_two_shards_one_gpu(oracle, seed, K, adv):
    import torch
    colors, counts, P, init = case(oracle, seed, K, adversarial=adv)
    ref = oracle.wsm(colors, counts, P, init, max_it=60, mode=UPDATE_EXACT)
    n = colors.size
    slices = [parallel.shard_bounds(n, 2, r) for r in range(2)]
    engines = [parallel.CudaShardEngine(cabi.Context(0), torch.device("cuda", 0)) for _ in range(2)]
    outs, ndc, rep = lockstep(engines, slices, colors, counts, P, init, K, cabi.Term(1e-3, 60, 0, 0))
    labels = np.concatenate([o[1] for o in outs])
    for cen, lab, sse, it in outs:
        assert it == ref.iterations
        assert np.array_equal(cen, ref.centers)
        assert np.array_equal(sse.view(np.uint64), ref.sse_trace.view(np.uint64))
    assert np.array_equal(labels, ref.labels)
    assert ndc == ref.ndc_total and rep == ref.repairs
    if adv:
        assert rep > 0


def test_sharded_wsm_nccl_single_rank(oracle):
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        colors, counts, P, init = case(oracle, 9, 48)
        ref = oracle.wsm(colors, counts, P, init, max_it=60, mode=UPDATE_EXACT)
        eng = parallel.CudaShardEngine(cabi.Context(0), torch.device("cuda", 0))
        r = parallel.sharded_wsm(eng, colors, counts, P, init, 48, cabi.Term(1e-3, 60, 0, 0))
        assert r.iterations == ref.iterations and r.ndc_total == ref.ndc_total
        assert np.array_equal(r.centers, ref.centers)
        assert np.array_equal(r.labels_local, ref.labels)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("adv", [False, True])
def test_sharded_wsm_fixed_iterations_no_host_sync(oracle, adv):
    # fixed iteration counts (BASELINE cfg5) take the asynchronous path: the
    # states are logged on the device and read once; an empty cluster (the
    # adversarial init) sends the run to the synchronous repair protocol
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        colors, counts, P, init = case(oracle, 21, 24, adversarial=adv)
        ref = oracle.wsm(colors, counts, P, init, fixed_it=12, mode=UPDATE_EXACT)
        eng = parallel.CudaShardEngine(cabi.Context(0), torch.device("cuda", 0))
        r = parallel.sharded_wsm(eng, colors, counts, P, init, 24, cabi.Term(1e-3, 100, 12, 0))
        assert r.iterations == 12 == ref.iterations
        assert r.ndc_total == ref.ndc_total and r.repair_count == ref.repairs
        assert np.array_equal(r.centers, ref.centers)
        assert np.array_equal(r.sse_trace.view(np.uint64), ref.sse_trace.view(np.uint64))
        assert np.array_equal(r.labels_local, ref.labels)
        if adv:
            assert ref.repairs > 0
    finally:
        dist.destroy_process_group()


def test_two_shards_async_finalize(oracle):
    # two engines in lockstep, every finalise without a host read
    import torch
    colors, counts, P, init = case(oracle, 31, 40)
    ref = oracle.wsm(colors, counts, P, init, fixed_it=9, mode=UPDATE_EXACT)
    n = colors.size
    slices = [parallel.shard_bounds(n, 2, r) for r in range(2)]
    engines = [parallel.CudaShardEngine(cabi.Context(0), torch.device("cuda", 0)) for _ in range(2)]
    term = cabi.Term(1e-3, 100, 9, 0)
    for e, (lo, hi) in zip(engines, slices):
        e.begin(colors[lo:hi], counts[lo:hi], P, init, 40, term)
    ndc = 0
    for _ in range(9):
        glob = sum(e.assign().cpu() for e in engines).cuda()
        ndc += int(glob[5 * 40])
        for e in engines:
            e.finalize_async(glob)
    assert all(e.status()[0] == parallel.STATE_DONE for e in engines)
    outs = [e.end(9) for e in engines]
    for cen, lab, sse, it in outs:
        assert it == 9 and np.array_equal(cen, ref.centers)
    assert np.array_equal(np.concatenate([o[1] for o in outs]), ref.labels)
    assert ndc == ref.ndc_total
