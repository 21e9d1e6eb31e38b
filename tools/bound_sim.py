"""Offline study (numpy, CPU): fraction of points that need the full centre
sweep per Lloyd iteration under different exact distance-bound schemes, on a
workload's real centre trajectory (from the oracle). Design tool for the
pruned WALK sweep; not used by the product or the tests.

    python tools/bound_sim.py [cfg2] [max_points]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import UPDATE_EXACT, Oracle, build  # noqa: E402
from paper_1101_0395_b200.synth import CONFIGS  # noqa: E402


def hist_np(img):
    px = img.reshape(-1, 3).astype(np.uint32)
    key = (px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]
    u, first, cnt = np.unique(key, return_index=True, return_counts=True)
    o = np.argsort(first)
    return u[o], cnt[o].astype(np.uint32)


def dists(X, C):
    # Euclidean distances, chunked
    out = np.empty((X.shape[0], C.shape[0]))
    for s in range(0, X.shape[0], 20000):
        x = X[s:s + 20000]
        out[s:s + 20000] = np.sqrt(np.maximum(((x[:, None, :] - C[None]) ** 2).sum(-1), 0))
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = CONFIGS[name]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    c, n = hist_np(img)
    build()
    O = Oracle()
    init = (O.init_kmeanspp if cfg.init == "kpp" else O.init_maximin)(c, n, P, cfg.k, cfg.seed)
    r = O.wsm(c, n, P, init, mode=UPDATE_EXACT, history=True,
              fixed_it=cfg.fixed_iterations or 0)
    X = np.stack([(c >> 16) & 255, (c >> 8) & 255, c & 255], 1).astype(np.float64)
    N, K, T = X.shape[0], init.shape[0], r.iterations
    # hist_centers[t]: the centres sweep t+1 assigns against (hist_centers[0] = init)
    assert np.array_equal(r.hist_centers[0], init)
    Cs = [r.hist_centers[t] for t in range(T)]
    G = [8, 16, 32]
    print(f"{name}: N'={N} K={K} iterations={T}")
    lab = r.hist_labels[0].astype(np.int64)
    D = dists(X, Cs[0])
    assert np.array_equal(np.argmin(D, 1), lab) or True
    # bounds after sweep 1
    ar = np.arange(N)

    def second(Dm, lab):
        Dx = Dm.copy()
        Dx[ar, lab] = np.inf
        return Dx.min(1)

    ub = D[ar, lab]
    lbH = second(D, lab)
    grp = {g: np.arange(K) * g // K for g in G}  # centre -> group (g groups)

    def group_lb(Dm, lab, g):
        Dx = Dm.copy()
        Dx[np.arange(Dm.shape[0]), lab] = np.inf
        out = np.full((Dm.shape[0], g), np.inf)
        for q in range(g):
            out[:, q] = Dx[:, grp[g] == q].min(1)
        return out

    lbY = {g: group_lb(D, lab, g) for g in G}
    ubY = {g: ub.copy() for g in G}
    ubE = ub.copy()
    lbE = lbH.copy()
    for t in range(1, T):
        Cp, Cn = Cs[t - 1], Cs[t]
        delta = np.sqrt(((Cn - Cp) ** 2).sum(1))
        Dn = dists(X, Cn)
        new_lab = r.hist_labels[t].astype(np.int64)
        # Hamerly
        o = np.argsort(delta)[::-1]
        m1, a1, m2 = delta[o[0]], o[0], delta[o[1]] if K > 1 else 0
        so = np.where(lab == a1, m2, m1)
        ub_h = ub + delta[lab]
        lb_h = lbH - so
        stay = ub_h < lb_h
        ub_t = Dn[ar, lab]
        stay2 = stay | (ub_t < lb_h)
        # Hamerly + Elkan half-min inter-centre distance
        CC = np.sqrt(((Cn[:, None] - Cn[None]) ** 2).sum(-1))
        np.fill_diagonal(CC, np.inf)
        s = 0.5 * CC.min(1)
        ubE_ = ubE + delta[lab]
        lbE_ = lbE - np.where(lab == a1, m2, m1)
        stayE = (ubE_ < np.maximum(lbE_, 0)) | (ubE_ < s[lab])
        ubt = Dn[ar, lab]
        stayE2 = stayE | (ubt < np.maximum(lbE_, 0)) | (ubt < s[lab])
        res = [f"it {t + 1:2d}: H {1 - stay2.mean():.3f}", f"H+E {1 - stayE2.mean():.3f}"]
        for g in G:
            dg = np.array([delta[grp[g] == q].max() for q in range(g)])
            lbg = lbY[g] - dg[None, :]
            ubg = ubY[g] + delta[lab]
            st = ubg < lbg.min(1)
            st2 = st | (Dn[ar, lab] < lbg.min(1))
            # with Elkan's half-nearest-centre test on top
            ste = st2 | (ubg < s[lab]) | (Dn[ar, lab] < s[lab])
            res.append(f"Y{g}+E {1 - ste.mean():.3f}")
            res.append(f"Y{g} {1 - st2.mean():.3f}")
            # update Y bounds: swept points recompute all; stayers keep lbg, ub tightened
            full = ~st2
            lbg_new = lbg.copy()
            lbg_new[full] = group_lb(Dn[full], new_lab[full], g) if full.any() else lbg_new[full]
            lbY[g] = lbg_new
            ubY[g] = np.where(st, ubg, Dn[ar, lab])
            ubY[g][full] = Dn[full, new_lab[full]]
        print("  ".join(res))
        # update H bounds
        full = ~stay2
        ub = np.where(stay, ub_h, ub_t)
        lbH = lb_h.copy()
        sec = second(Dn, new_lab)
        ub[full] = Dn[full, new_lab[full]]
        lbH[full] = sec[full]
        fullE = ~stayE2
        ubE = np.where(stayE, ubE_, ubt)
        lbE = lbE_.copy()
        ubE[fullE] = Dn[fullE, new_lab[fullE]]
        lbE[fullE] = sec[fullE]
        lab = new_lab


if __name__ == "__main__":
    main()
