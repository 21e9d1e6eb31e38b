"""NumPy implementation of the sharded-Lloyd engine interface -- TEST
INFRASTRUCTURE ONLY (drives paper_1101_0395_b200.parallel.sharded_wsm on CPU
ranks under gloo). Exact FP64 reference assignment (kmeans.cpp:40-79, no FMA:
numpy ufuncs do not contract), exact integer moments and the exact-moment SSE,
i.e. the same contract as the device engine."""
import numpy as np
import torch


def d2(x, c):
    dr, dg, db = x[..., 0] - c[..., 0], x[..., 1] - c[..., 1], x[..., 2] - c[..., 2]
    return (dr * dr + dg * dg) + db * db


class NumpyShardEngine:
    def begin(self, colors, counts, P, init, K, term):
        self.col = np.asarray(colors, np.uint32)
        self.cnt = np.asarray(counts, np.int64)
        self.x = np.stack([(self.col >> 16) & 255, (self.col >> 8) & 255, self.col & 255], 1).astype(np.float64)
        self.P, self.K = int(P), int(K)
        self.c = np.asarray(init, np.float64).reshape(K, 3).copy()
        self.labels = np.zeros(len(self.col), np.int64)
        self.iter = 0
        self.sse = []
        self.eps, self.maxit, self.fixed = term.epsilon, term.max_iterations, term.fixed_iterations
        self.table = None

    def _moments(self):
        K = self.K
        m = np.zeros((K, 5), dtype=object)
        for k in range(K):
            sel = self.labels == k
            q = self.cnt[sel]
            xs = self.x[sel].astype(np.int64)
            m[k, 0] = int(q.sum())
            m[k, 1] = int((q * xs[:, 0]).sum())
            m[k, 2] = int((q * xs[:, 1]).sum())
            m[k, 3] = int((q * xs[:, 2]).sum())
            m[k, 4] = int((q * (xs * xs).sum(1)).sum())
        return m

    def _pack(self, ndc):
        m = self._moments()
        return torch.tensor([int(v) for v in m.reshape(-1)] + [int(ndc), 0], dtype=torch.int64)

    def assign(self):
        n, K = len(self.col), self.K
        ndc = 0
        if self.iter == 0:
            for i in range(n):
                self.labels[i] = int(np.argmin(d2(self.x[i], self.c)))  # first minimum = lowest index
            ndc = n * K
        else:
            dt, order = self.table
            for i in range(n):
                prev = self.labels[i]
                pd = d2(self.x[i], self.c[prev])
                cut = 4.0 * pd
                bd, best = pd, prev
                ndc += 1
                for j in range(1, K):
                    t = order[prev, j]
                    if dt[prev, t] >= cut:
                        break
                    d = d2(self.x[i], self.c[t])
                    ndc += 1
                    if d < bd:
                        bd, best = d, t
                self.labels[i] = best
        return self._pack(ndc)

    def moments(self):
        return self._pack(0)

    def finalize(self, glob):
        K = self.K
        g = [int(v) for v in glob.tolist()]
        mom = [g[5 * k: 5 * k + 5] for k in range(K)]
        if any(m[0] == 0 for m in mom):
            return 2, 0.0
        terms = []
        for k, (nk, sr, sg, sb, q) in enumerate(mom):
            nd = float(nk)
            self.c[k] = [float(sr) / nd, float(sg) / nd, float(sb) / nd]
            terms.append(float(nk * q - (sr * sr + sg * sg + sb * sb)) / nd)
        # the oracle's order: pairwise tree over the next power of two (cq_oracle.c tree_sum)
        st = 1
        while st < K:
            for i in range(0, K - st, 2 * st):
                terms[i] = terms[i] + terms[i + st]
            st *= 2
        sse = terms[0] / float(self.P)
        self.iter += 1
        self.sse.append(sse)
        it = self.iter
        if self.fixed > 0:
            done = it >= self.fixed
        else:
            done = sse == 0.0 or (it >= 2 and (self.sse[-2] - sse) / sse <= self.eps) or it >= self.maxit
        dt = np.array([[d2(self.c[i], self.c[j]) for j in range(K)] for i in range(K)])
        order = np.zeros((K, K), np.int64)
        for i in range(K):
            row = sorted(range(K), key=lambda j: (dt[i, j], j))
            row.remove(i)
            order[i] = [i] + row
        self.table = (dt, order)
        return (1 if done else 0), sse

    def sizes(self):
        return torch.tensor(np.bincount(self.labels, minlength=self.K), dtype=torch.int64)

    def donor(self, gs, fallback):
        n = len(self.col)
        if n == 0:
            return -2.0, None, 0, 0
        if fallback:
            gsn = gs.numpy()
            for i in range(n):
                if gsn[self.labels[i]] >= 2:
                    return 1.0, i, int(self.col[i]), int(self.labels[i])
            return -1.0, 0, int(self.col[0]), int(self.labels[0])
        w = self.cnt.astype(np.float64) * (1.0 / float(self.P))
        v = w * d2(self.x, self.c[self.labels])
        i = int(np.argmax(v))  # first maximum = lowest index
        return float(v[i]), i, int(self.col[i]), int(self.labels[i])

    def move(self, li, e, colour):
        if li is not None:
            self.labels[li] = e
        self.c[e] = [(colour >> 16) & 255, (colour >> 8) & 255, colour & 255]

    def end(self, limit, labels=True):
        return (self.c.copy(), self.labels.astype(np.uint32) if labels else None, np.array(self.sse), self.iter)
