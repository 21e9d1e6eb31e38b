"""Coarse 32^3 histogram (quant::build_coarse_histogram): device time of the
C-ABI call on a device-resident image (CUDA events on the context stream)
against the reference's CPU build (oracle/_ref, one core), for cfg2 and cfg5.

    python tools/coarse_bench.py > profiles/r01_coarse_histogram.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import RefLib  # noqa: E402  (CPU baseline only)
from paper_1101_0395_b200 import cabi  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402


def main():
    ctx = cabi.Context(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s.cuda_stream)
    ref = RefLib() if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libquantref.so")) else None
    rows = []
    for name in ("cfg2", "cfg5"):
        img = CONFIGS[name].image()
        P = img.shape[0] * img.shape[1]
        d = torch.from_numpy(img).cuda()
        out = torch.empty((5, 32768), dtype=torch.int64, device="cuda")
        for _ in range(3):
            ctx.coarse_histogram_raw(d, P, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            ctx.coarse_histogram_raw(d, P, out)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        row = {"config": name, "pixels": P, "device_ms": ms, "device_mpix_s": P / ms / 1e3}
        if ref is not None:
            t0 = time.perf_counter()
            want = ref.coarse_histogram(rgb=img)
            cpu = time.perf_counter() - t0
            row.update(cpu_ms=cpu * 1e3, cpu_mpix_s=P / cpu / 1e6, cpu_cores=1, cpu_kind="reference",
                       bit_exact=bool(np.array_equal(out.cpu().numpy(), want)))
        rows.append(row)
    print(json.dumps({"metric": "coarse 32^3 histogram, MPixel/s", "rows": rows}))


if __name__ == "__main__":
    main()
