import time, sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1101_0395_b200 import cabi
from paper_1101_0395_b200.synth import CONFIGS
cfg = CONFIGS['cfg4']
ctx = cabi.Context(0)
dev = torch.device('cuda', 0)
imgs = [cfg.image(i) for i in range(8)]
ks = [cfg.k_for(i) for i in range(8)]
d_imgs = [torch.from_numpy(im).to(dev) for im in imgs]
P = imgs[0].shape[0]*imgs[0].shape[1]
d_idx = torch.empty(P, dtype=torch.int32, device=dev); d_q = torch.empty((P,3), dtype=torch.uint8, device=dev)
sse = np.zeros(128)
for rep in range(3):
    for i in range(8):
        d_pal = torch.empty((ks[i],3), dtype=torch.float64, device=dev)
        term = cabi.Term(1e-3, 100, 0, 0)
        c = cabi.QuantizeCfg(cabi.INIT_MAXIMIN, ks[i], cfg.seed, term, 4)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = ctx.quantize_raw(d_imgs[i], P, c, None, d_pal, None, sse, d_idx, d_q)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if rep == 2:
            dsum = st.ms_histogram + st.ms_init + st.ms_lloyd + st.ms_map
            print(f"img {i} K={ks[i]} N'={st.n_unique} wall {1e3*(t1-t0):.3f} ms  device stages {dsum:.3f} ms  it {st.lloyd.iterations}")
