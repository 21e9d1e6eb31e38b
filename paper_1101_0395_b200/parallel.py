"""Multi-GPU orchestration: one process per GPU over torch.distributed.

SURVEY.md §8(e):
  * batches (cfg4)  -- sharded by image, no data-path collective (bench.py);
  * small images    -- replicas only (bench.py);
  * one huge image  -- sharded by unique colour: each rank owns a contiguous
    slice of the first-occurrence-ordered histogram and runs the assignment on
    it; one allreduce of the packed int64 moment partials (K x {n, S, Q} + NDC
    + replay count) per iteration (NCCL over NVLink on GPUs, gloo in the CPU
    tests), then every rank finalises identically from the same global
    moments, so centres, termination and walk tables agree bit for bit.

Empty-cluster repair (reference kmeans.cpp:124-169) across ranks: global
cluster sizes by allreduce, each rank's best donor candidate (value, global
index, colour, old label) by all-gather, the lowest global index wins ties,
the owning rank moves its point and every rank plants the centre.

The protocol is written against a small engine interface so the CPU tests can
drive it with a NumPy engine; the product engine is CudaShardEngine (C-ABI).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import cabi

STATE_CONTINUE, STATE_DONE, STATE_EMPTY = 0, 1, 2


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of n items for `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class CudaShardEngine:
    """cqg_shard_* on one GPU; partials live in device tensors for NCCL."""

    def __init__(self, ctx: cabi.Context, device):
        import torch
        self.ctx, self.torch, self.device = ctx, torch, device

    def begin(self, colors, counts, P, init, K, term: cabi.Term):
        """colors/counts/init: numpy arrays or device tensors (used in place)."""
        self.K = K
        def prep(a, dt):
            if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
                return a.contiguous()
            return np.ascontiguousarray(a, dt)
        colors, counts = prep(colors, np.uint32), prep(counts, np.uint32)
        init = prep(init if hasattr(init, "data_ptr") else np.asarray(init, np.float64).reshape(-1, 3), np.float64)
        n = int(colors.numel() if hasattr(colors, "numel") else colors.size)
        cabi.check(self.ctx.L.cqg_shard_begin(self.ctx.h, cabi.ptr(colors) if n else None,
                                              cabi.ptr(counts) if n else None, n,
                                              P, cabi.ptr(init), K, C.byref(term)))
        self.n = n

    def _partial(self, fn):
        t = self.torch.empty(5 * self.K + 2, dtype=self.torch.int64, device=self.device)
        cabi.check(fn(self.ctx.h, t.data_ptr()))
        return t

    def assign(self):
        return self._partial(self.ctx.L.cqg_shard_assign)

    def moments(self):
        return self._partial(self.ctx.L.cqg_shard_moments)

    def finalize(self, glob):
        st, sse = C.c_int(0), C.c_double(0)
        cabi.check(self.ctx.L.cqg_shard_finalize(self.ctx.h, glob.data_ptr(), C.byref(st), C.byref(sse)))
        return st.value, sse.value

    def finalize_async(self, glob):
        """Finalise without a host read (the state is logged on the device)."""
        cabi.check(self.ctx.L.cqg_shard_finalize_async(self.ctx.h, glob.data_ptr()))

    def status(self):
        """(0 continue | 1 done | 2 redo synchronously, iterations) of the logged run."""
        st, it = C.c_int(0), C.c_int(0)
        cabi.check(self.ctx.L.cqg_shard_status(self.ctx.h, C.byref(st), C.byref(it)))
        return st.value, it.value

    def sizes(self):
        t = self.torch.empty(self.K, dtype=self.torch.int32, device=self.device)
        cabi.check(self.ctx.L.cqg_shard_sizes(self.ctx.h, t.data_ptr()))
        return t.to(self.torch.int64)

    def donor(self, global_sizes, fallback):
        gs = global_sizes.to(self.torch.int32).contiguous()
        v, i, c, l = C.c_double(0), C.c_uint64(0), C.c_uint32(0), C.c_uint32(0)
        cabi.check(self.ctx.L.cqg_shard_donor(self.ctx.h, gs.data_ptr(), 1 if fallback else 0, C.byref(v),
                                              C.byref(i), C.byref(c), C.byref(l)))
        idx = i.value if i.value < self.n else None
        return v.value, idx, c.value, l.value

    def move(self, local_index, e, colour):
        idx = (1 << 64) - 1 if local_index is None else int(local_index)
        cabi.check(self.ctx.L.cqg_shard_move(self.ctx.h, idx, int(e), int(colour)))

    def end(self, limit, labels=True):
        K = self.K
        cen = np.empty((K, 3), np.float64)
        lab = np.empty(max(self.n, 1), np.uint32) if labels else None
        sse = np.zeros(max(limit, 1), np.float64)
        it = C.c_int(0)
        cabi.check(self.ctx.L.cqg_shard_end(self.ctx.h, cabi.ptr(cen), cabi.ptr(lab) if labels else None,
                                            cabi.ptr(sse), C.byref(it)))
        return cen, (lab[: self.n] if labels else None), sse[: it.value].copy(), it.value


@dataclass
class ShardedResult:
    centers: np.ndarray
    labels_local: np.ndarray
    lo: int
    hi: int
    sse_trace: np.ndarray
    iterations: int
    ndc_total: int
    repair_count: int
    flagged_total: int


def _repair(engine, lo: int, K: int, dist, group, torch) -> int:
    """Cross-rank replay of repair_empty_clusters (kmeans.cpp:124-169)."""
    gs = engine.sizes()
    dist.all_reduce(gs, group=group)
    dev = gs.device
    gs = gs.cpu()
    world = dist.get_world_size(group)
    repairs = 0
    big = float(1 << 60)
    while True:
        empty = (gs == 0).nonzero()
        if empty.numel() == 0:
            return repairs
        e = int(empty[0])

        def gather(fallback):
            v, li, col, lab = engine.donor(gs, fallback)
            mine = torch.tensor([v, float(lo + li) if li is not None else big, float(col), float(lab)],
                                dtype=torch.float64, device=dev)
            out = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(out, mine, group=group)
            rows = [o.cpu().tolist() for o in out]
            return rows, li

        rows, li = gather(False)
        best = max(range(world), key=lambda r: (rows[r][0], -rows[r][1]))
        if not rows[best][0] > 0.0:
            rows, li = gather(True)
            cands = [r for r in range(world) if rows[r][0] > 0.0]
            if not cands:
                raise RuntimeError("repair_empty_clusters: more clusters than points")
            best = min(cands, key=lambda r: rows[r][1])
        _, gidx, col, lab = rows[best]
        mine = dist.get_rank(group) == best
        engine.move(li if mine else None, e, int(col))
        gs[int(lab)] -= 1
        gs[e] += 1
        repairs += 1


def sharded_wsm(engine, colors, counts, P: int, init, K: int, term: cabi.Term, group=None,
                labels: bool = True) -> ShardedResult:
    """Weighted sort-means over the unique colours sharded across the ranks of
    `group`; every rank returns the same centres / trace and its own labels
    (labels=False leaves them on the device: labels_local is None)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(colors)
    lo, hi = shard_bounds(n, world, rank)
    engine.begin(colors[lo:hi], counts[lo:hi], P, init, K, term)
    if term.fixed_iterations > 0 and hasattr(engine, "finalize_async"):
        # a fixed iteration count needs no per-iteration host round trip: the
        # moments allreduce and every rank's finalise stay on the device (NCCL
        # is ordered on the stream), the states are checked once at the end;
        # an empty cluster (or an early stop) sends the run to the protocol below
        acc = None
        for _ in range(term.fixed_iterations):
            part = engine.assign()
            dist.all_reduce(part, group=group)
            cnt = part[5 * K:5 * K + 2].clone()
            acc = cnt if acc is None else acc + cnt
            engine.finalize_async(part)
        state, _ = engine.status()
        ok = torch.tensor([1 if state == STATE_DONE else 0], dtype=torch.int32, device=part.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 1:
            cen, lab, sse, it = engine.end(term.fixed_iterations, labels)
            tot = acc.cpu().tolist()
            return ShardedResult(cen, lab, lo, hi, sse, it, int(tot[0]), 0, int(tot[1]))
        engine.begin(colors[lo:hi], counts[lo:hi], P, init, K, term)
    ndc, flagged, repairs = 0, 0, 0
    while True:
        part = engine.assign()
        dist.all_reduce(part, group=group)
        ndc += int(part[5 * K])
        flagged += int(part[5 * K + 1])
        state, _ = engine.finalize(part)
        while state == STATE_EMPTY:
            repairs += _repair(engine, lo, K, dist, group, torch)
            part = engine.moments()
            dist.all_reduce(part, group=group)
            state, _ = engine.finalize(part)
        if state == STATE_DONE:
            break
    limit = term.fixed_iterations if term.fixed_iterations > 0 else term.max_iterations
    cen, lab, sse, it = engine.end(limit, labels)
    return ShardedResult(cen, lab, lo, hi, sse, it, ndc, repairs, flagged)
