"""Per-phase wall time of the colour-sharded Lloyd loop at world 1 (GPU).

    python tools/shard_timing.py cfg3
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1101_0395_b200 import cabi, parallel  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
dist.init_process_group("gloo", rank=0, world_size=1, init_method="tcp://127.0.0.1:29544")
dev = torch.device("cuda", 0)
ctx = cabi.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
img = cfg.image()
P = img.shape[0] * img.shape[1]
d_img = torch.from_numpy(img).to(dev).reshape(-1)
cap = min(P, 1 << 24)
d_col = torch.empty(cap, dtype=torch.int32, device=dev)
d_cnt = torch.empty(cap, dtype=torch.int32, device=dev)
n = ctx.histogram_raw(d_img, P, d_col, d_cnt)
K = cfg.k
d_init = torch.empty((K, 3), dtype=torch.float64, device=dev)
ctx.init_raw(cabi.INIT_KMEANSPP if cfg.init == "kpp" else cabi.INIT_MAXIMIN, d_col, d_cnt, n, P, K, cfg.seed, d_init)
term = cabi.Term(1e-3, 100, cfg.fixed_iterations, 0)
eng = parallel.CudaShardEngine(ctx, dev)
for rep in range(2):
    torch.cuda.synchronize()
    eng.begin(d_col[:n], d_cnt[:n], P, d_init, K, term)
    tt = {"assign": 0.0, "allreduce": 0.0, "read": 0.0, "finalize": 0.0}
    its = 0
    while True:
        t0 = time.perf_counter()
        part = eng.assign()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dist.all_reduce(part)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        _ = int(part[5 * K]) + int(part[5 * K + 1])
        t3 = time.perf_counter()
        state, _ = eng.finalize(part)
        t4 = time.perf_counter()
        tt["assign"] += t1 - t0
        tt["allreduce"] += t2 - t1
        tt["read"] += t3 - t2
        tt["finalize"] += t4 - t3
        its += 1
        if state != parallel.STATE_CONTINUE:
            break
    print(f"rep {rep}: {its} iterations, ms per iteration:",
          {k: round(1e3 * v / its, 3) for k, v in tt.items()})
