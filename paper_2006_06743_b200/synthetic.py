"""Seeded synthetic stand-ins for BASELINE.json's five workload shapes.

The reference ships no generator for these shapes (its own generators,
proj/src/synthetic.cpp, make ball mixtures / theory scenarios), and the paper's
real datasets are not available here, so these seeded fp32 generators stand in
for them.  Choices the config text leaves open are pinned here and in
DESIGN.md (section "Workloads"):

  * cluster membership is drawn per row (categorical), so rows are already in
    random order (no ordering by cluster);
  * "uniform noise over the bounding box" = uniform over the box spanned by
    the cluster points (cfg3) or the stated range (cfg1 [0,1]^2, cfg4
    [0,100]^3, cfg5 [-50,50]^32);
  * cfg3 covariance = Q diag(lambda) Q^T, Q Haar-random orthogonal,
    lambda ~ U[0.01, 0.05];
  * cfg4 rings/arcs: radius ~ U[0.5, 2], random plane, arc extent ~ U[pi, 2 pi],
    radial + out-of-plane Gaussian thickness sigma = 0.05;
  * cfg5 cluster weights proportional to k^-1.1, k = 1..1000.

Data streams come from numpy's PCG64 keyed by (config seed, salt), never from
the reference's graph-sampling streams.  Generation is chunked over spawned
streams so the bytes do not depend on the thread count.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from dataclasses import dataclass

import numpy as np

_SALT = 0x534E4744  # "SNGD"
_CHUNK = 1 << 20


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    eps: float
    rate: float
    min_pts: int
    seed: int
    note: str

    @property
    def draws(self) -> int:
        import math
        return min(int(math.ceil(self.rate * float(self.n))), self.n - 1)

    @property
    def pairs(self) -> int:
        return self.n * self.draws


CONFIGS = {
    1: Workload("cfg1_blobs2d", 20_000, 2, 0.03, 0.1, 10, 1,
                "5 isotropic Gaussian blobs (sigma 0.05) + 5% uniform noise in [0,1]^2"),
    2: Workload("cfg2_mnistlike784", 70_000, 784, 4.5, 0.01, 10, 2,
                "10 Gaussian clusters in [0,1]^784, sigma 0.1, clipped to [0,1]"),
    3: Workload("cfg3_aniso16", 1_000_000, 16, 0.5, 0.001, 5, 3,
                "50 anisotropic Gaussian clusters in [-10,10]^16 + 2% noise"),
    4: Workload("cfg4_rings3d", 5_000_000, 3, 0.1, 0.0005, 4, 4,
                "200 noisy rings/arcs (r 0.5-2, sigma 0.05) in [0,100]^3 + 5% noise"),
    5: Workload("cfg5_zipf32", 20_000_000, 32, 1.2, 0.0002, 5, 5,
                "1000 Gaussian clusters (sigma 0.2) in [-50,50]^32, Zipf(1.1) sizes + 1% noise"),
}


def _threads() -> int:
    return max(1, min(16, os.cpu_count() or 1))


def _chunked(n: int, seed: int, fn) -> np.ndarray:
    """Run fn(rng, start, stop) over fixed 1M-row chunks with spawned streams."""
    ss = np.random.SeedSequence([seed, _SALT, 1])
    starts = list(range(0, n, _CHUNK))
    kids = ss.spawn(len(starts))
    parts = [None] * len(starts)

    def run(i):
        parts[i] = fn(np.random.Generator(np.random.PCG64(kids[i])), starts[i],
                      min(n, starts[i] + _CHUNK))

    with cf.ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(run, range(len(starts))))
    return np.concatenate(parts, axis=0) if parts else np.empty((0,), np.float32)


def _params_rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, _SALT, 0])))


def _gaussian_mixture(n, d, means, sigma, weights, noise_frac, noise_lo, noise_hi, seed,
                      clip=None, chols=None):
    """Categorical mixture of Gaussians + uniform noise, fp32, shuffled rows."""
    k = len(means)
    means = np.asarray(means, np.float32)

    def fn(rng, a, b):
        m = b - a
        is_noise = rng.random(m) < noise_frac
        comp = rng.choice(k, size=m, p=weights)
        z = rng.standard_normal((m, d), dtype=np.float32)
        if chols is not None:
            out = np.empty((m, d), np.float32)
            for c in range(k):
                idx = np.nonzero(comp == c)[0]
                if idx.size:
                    out[idx] = z[idx] @ chols[c].T + means[c]
        else:
            out = z * np.float32(sigma)
            out += means[comp]
        if noise_frac > 0:
            nn = int(is_noise.sum())
            if nn:
                lo = np.asarray(noise_lo, np.float32)
                hi = np.asarray(noise_hi, np.float32)
                out[is_noise] = lo + (hi - lo) * rng.random((nn, d), dtype=np.float32)
        if clip is not None:
            np.clip(out, clip[0], clip[1], out=out)
        return out

    return _chunked(n, seed, fn)


def generate(cfg: int | Workload, n: int | None = None) -> np.ndarray:
    """fp32 row-major points for config `cfg` (optionally with a different n)."""
    w = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    n = w.n if n is None else n
    pr = _params_rng(w.seed)
    d = w.d
    if w.name.startswith("cfg1"):
        means = pr.random((5, d))
        return _gaussian_mixture(n, d, means, 0.05, np.full(5, 0.2), 0.05, [0, 0], [1, 1], w.seed)
    if w.name.startswith("cfg2"):
        means = pr.random((10, d))
        return _gaussian_mixture(n, d, means, 0.1, np.full(10, 0.1), 0.0, 0, 1, w.seed,
                                 clip=(0.0, 1.0))
    if w.name.startswith("cfg3"):
        k = 50
        means = pr.uniform(-10, 10, (k, d))
        chols = []
        for _ in range(k):
            q, r = np.linalg.qr(pr.standard_normal((d, d)))
            q = q * np.sign(np.diag(r))
            lam = pr.uniform(0.01, 0.05, d)
            chols.append((q * np.sqrt(lam)).astype(np.float32))  # Q diag(sqrt(lam))
        # bounding box of the clusters (means +- 4 sigma_max)
        lo = means.min(0) - 4 * np.sqrt(0.05)
        hi = means.max(0) + 4 * np.sqrt(0.05)
        return _gaussian_mixture(n, d, means, None, np.full(k, 1.0 / k), 0.02, lo, hi, w.seed,
                                 chols=np.stack(chols))
    if w.name.startswith("cfg4"):
        k = 200
        centers = pr.uniform(0, 100, (k, 3))
        radius = pr.uniform(0.5, 2.0, k)
        theta0 = pr.uniform(0, 2 * np.pi, k)
        extent = pr.uniform(np.pi, 2 * np.pi, k)
        e1 = np.empty((k, 3))
        e2 = np.empty((k, 3))
        for c in range(k):
            q, r = np.linalg.qr(pr.standard_normal((3, 3)))
            q = q * np.sign(np.diag(r))
            e1[c], e2[c] = q[:, 0], q[:, 1]

        def fn(rng, a, b):
            m = b - a
            is_noise = rng.random(m) < 0.05
            comp = rng.integers(0, k, m)
            th = theta0[comp] + extent[comp] * rng.random(m)
            pts = (centers[comp] + radius[comp, None] *
                   (np.cos(th)[:, None] * e1[comp] + np.sin(th)[:, None] * e2[comp]))
            pts += 0.05 * rng.standard_normal((m, 3))
            nn = int(is_noise.sum())
            if nn:
                pts[is_noise] = rng.uniform(0, 100, (nn, 3))
            return pts.astype(np.float32)

        return _chunked(n, w.seed, fn)
    if w.name.startswith("cfg5"):
        k = 1000
        means = pr.uniform(-50, 50, (k, d))
        wts = np.arange(1, k + 1, dtype=np.float64) ** -1.1
        wts /= wts.sum()
        return _gaussian_mixture(n, d, means, 0.2, wts, 0.01, np.full(d, -50.0),
                                 np.full(d, 50.0), w.seed)
    raise KeyError(w.name)
