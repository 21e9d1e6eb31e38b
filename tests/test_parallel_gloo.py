"""The multi-rank protocol of paper_1101_0395_b200.parallel (colour-sharded
Lloyd: per-iteration moment allreduce, identical finalisation, cross-rank
empty-cluster repair) on CPU ranks under gloo, against the single-process
exact-moment oracle: labels, centres, SSE trace, iterations, NDC and repairs
must agree bit for bit for any world size."""
import multiprocessing as mp
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    from np_shard_engine import NumpyShardEngine
    from paper_1101_0395_b200 import cabi, parallel
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        colors, counts, P, init, K, fixed = case
        term = cabi.Term(1e-3, 60, fixed, 0)
        r = parallel.sharded_wsm(NumpyShardEngine(), colors, counts, P, init, K, term)
        labels = [None] * world
        dist.all_gather_object(labels, r.labels_local)
        q.put((rank, r.centers, np.concatenate(labels), r.sse_trace, r.iterations, r.ndc_total, r.repair_count))
    finally:
        dist.destroy_process_group()


def run_world(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def make_case(oracle, seed, K, adversarial=False, fixed=0):
    from paper_1101_0395_b200.synth import synth_image
    img = synth_image(48, 32, seed, nblobs=5, sigma=9.0, noise=0.03)
    colors, counts, _ = oracle.histogram(img)
    P = 48 * 32
    if adversarial:
        init = np.array([[250.0, 250.0, 250.0 - i] for i in range(K)])
    else:
        init = oracle.init_kmeanspp(colors, counts, P, K, seed)
    return colors, counts, P, init, K, fixed


@pytest.mark.parametrize("world,seed,K,adv", [(2, 3, 12, False), (3, 4, 9, False), (2, 5, 10, True)])
def test_sharded_lloyd_matches_single_process(oracle, world, seed, K, adv):
    from oracle.pyoracle import UPDATE_EXACT
    case = make_case(oracle, seed, K, adv)
    colors, counts, P, init, K, fixed = case
    ref = oracle.wsm(colors, counts, P, init, max_it=60, mode=UPDATE_EXACT)
    outs = run_world(world, case)
    for rank, cen, labels, sse, it, ndc, rep in outs:
        assert it == ref.iterations
        assert ndc == ref.ndc_total
        assert rep == ref.repairs
        assert np.array_equal(cen, ref.centers)
        assert np.array_equal(sse.view(np.uint64), ref.sse_trace.view(np.uint64))
        assert np.array_equal(labels.astype(np.uint32), ref.labels)
    if adv:
        assert ref.repairs > 0


def test_shard_bounds_cover_exactly():
    from paper_1101_0395_b200.parallel import shard_bounds
    for n in (0, 1, 7, 100, 101):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
