"""Pinned synthetic inputs standing in for the paper's test images.

The reference measures on 8 photographs that are not in this
container; BASELINE.json names synthetic configurations instead. This module
pins one seeded generator (numpy PCG64) so the device path, the oracle and the
reference arm all see the same bytes:

  background  bilinear blend of 4 random corner colours
  per pixel   u ~ U[0,1): u < noise          -> uniform random 24-bit colour
                          u < noise + 0.6    -> Gaussian blob j ~ U{0..nblobs-1}:
                                                centre_j + sigma_j * N(0, I3)
                          otherwise          -> background
  rounding    channel_to_u8 (floor(v + 0.5), clamp; color.hpp:63-68)
  uniform     cfg5: independent uniform bytes
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def synth_image(width: int, height: int, seed: int, nblobs: int = 8, sigma=20.0,
                noise: float = 0.0, blob_frac: float = 0.6, uniform: bool = False) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if uniform:
        return rng.integers(0, 256, size=(height, width, 3), dtype=np.uint8)
    P = width * height
    corners = rng.random((4, 3)) * 255.0
    fx = (np.arange(width, dtype=np.float64) / max(width - 1, 1))[None, :, None]
    fy = (np.arange(height, dtype=np.float64) / max(height - 1, 1))[:, None, None]
    bg = ((1 - fx) * (1 - fy) * corners[0] + fx * (1 - fy) * corners[1] +
          (1 - fx) * fy * corners[2] + fx * fy * corners[3]).reshape(P, 3)
    centers = rng.random((nblobs, 3)) * 255.0
    if isinstance(sigma, (tuple, list)):
        sig = rng.uniform(sigma[0], sigma[1], nblobs)
    else:
        sig = np.full(nblobs, float(sigma))
    u = rng.random(P)
    j = rng.integers(0, nblobs, P)
    g = rng.standard_normal((P, 3))
    val = bg
    blob = (u >= noise) & (u < noise + blob_frac)
    val[blob] = centers[j[blob]] + sig[j[blob], None] * g[blob]
    nz = u < noise
    val[nz] = rng.integers(0, 256, size=(int(nz.sum()), 3)).astype(np.float64)
    out = np.clip(np.floor(val + 0.5), 0.0, 255.0).astype(np.uint8)
    return out.reshape(height, width, 3)


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    k: int
    init: str              # "mmx" | "kpp"
    seed: int
    nblobs: int = 8
    sigma: object = 20.0
    noise: float = 0.0
    uniform: bool = False
    fixed_iterations: int = 0
    images: int = 1        # batch size (cfg4)
    k_cycle: tuple = ()

    def image(self, i: int = 0) -> np.ndarray:
        if self.images > 1:
            nb = 8 + (self.seed + 7 * i) % 25  # 8..32 blobs per image
            return synth_image(self.width, self.height, self.seed + i, nblobs=nb,
                               sigma=self.sigma, noise=self.noise)
        return synth_image(self.width, self.height, self.seed, nblobs=self.nblobs,
                           sigma=self.sigma, noise=self.noise, uniform=self.uniform)

    def k_for(self, i: int = 0) -> int:
        return self.k_cycle[i % len(self.k_cycle)] if self.k_cycle else self.k


# BASELINE.json configs[0..4]
CONFIGS = {
    "cfg1": Config("cfg1", 512, 512, 32, "mmx", 101, nblobs=8, sigma=20.0),
    "cfg2": Config("cfg2", 512, 512, 256, "kpp", 202, nblobs=24, sigma=12.0, noise=0.02),
    "cfg3": Config("cfg3", 4096, 4096, 256, "mmx", 303, nblobs=64, sigma=(8.0, 30.0), noise=0.10),
    "cfg3k64": Config("cfg3k64", 4096, 4096, 64, "mmx", 303, nblobs=64, sigma=(8.0, 30.0), noise=0.10),
    "cfg4": Config("cfg4", 768, 512, 32, "mmx", 400, sigma=(8.0, 24.0), images=64,
                   k_cycle=(32, 64, 128, 256)),
    "cfg5": Config("cfg5", 8192, 8192, 256, "kpp", 505, uniform=True, fixed_iterations=20),
}
