"""Seeded synthetic inputs for the five BASELINE.json configs.

This module holds NO arithmetic of the method: it only draws base vectors and
queries (Gaussian mixtures with the shapes, value distributions and list-size
skew that BASELINE.json's ``configs`` name).  It is the one module both the CUDA
path's tests/bench and the oracle's tests consume.  Recipe:

  CFG1  D=128  N=1e5  256 centres mu~N(0,4I), x = mu + N(0,I), labels uniform
  CFG2  D=960  N=1e6  1024 centres mu~N(0,4I), per-centre diag scales
                      s~U(0.5,2)^D, x = mu + s*N(0,I)
  CFG3  D=96   N=1e7  4096 centres mu~N(0,4I), x = mu + N(0,I), mixture weights
                      w_r ~ r^-1.1 over a seeded permutation (Zipf(1.1) list
                      sizes); every vector L2-normalised; k-means initialised
                      from the normalised generator centres
  CFG4  D=128  N=1e8  16384 centres |N(0,48^2)| (SIFT-like, non-negative),
                      x = rint(clip(mu + N(0,16^2 I), 0, 255)), stored fp32
  CFG5  D=96   N=1e9  65536 centres mu~N(0,4I), x = mu + N(0,I)

Queries come from the same mixture (a distinct seeded stream).  The paper's
public datasets (SIFT1M / Cohere10M / SIFT100M / SIFT1B) are not
available; these synthetic configs stand in for their shapes and scale.

Rows are generated in fixed chunks of ``CHUNK`` rows, each from its own
generator seeded by (data_seed, stream, chunk), so any contiguous id slice
(e.g. one GPU's shard) can be produced independently of the others.  The
values depend on the torch device the generator runs on (CPU vs CUDA streams
differ); a test that compares two implementations always feeds both the same
materialised tensor.
"""
from __future__ import annotations

import dataclasses
import math

import torch

CHUNK = 1 << 20


@dataclasses.dataclass(frozen=True)
class Spec:
    cfg: int
    D: int
    N: int
    ncent: int
    nlist: int
    nq: int
    nprobe: int
    k: int
    M: int
    kind: str  # "iso" | "aniso" | "zipf" | "uint8"
    data_seed: int
    build_seed: int = 42

    @property
    def W(self) -> int:
        return (self.D + 31) // 32


_BASE = {
    1: dict(D=128, N=100_000, ncent=256, nlist=256, nq=100, nprobe=16, k=10, M=100, kind="iso"),
    2: dict(D=960, N=1_000_000, ncent=1024, nlist=1024, nq=10_000, nprobe=64, k=100, M=1000, kind="aniso"),
    3: dict(D=96, N=10_000_000, ncent=4096, nlist=4096, nq=10_000, nprobe=64, k=10, M=200, kind="zipf"),
    4: dict(D=128, N=100_000_000, ncent=16384, nlist=16384, nq=10_000, nprobe=64, k=10, M=100, kind="uint8"),
    5: dict(D=96, N=1_000_000_000, ncent=65536, nlist=65536, nq=10_000, nprobe=128, k=10, M=100, kind="iso"),
}


def spec(cfg: int, **overrides) -> Spec:
    d = dict(_BASE[cfg])
    d.update(overrides)
    d.setdefault("data_seed", 1000 + cfg)
    return Spec(cfg=cfg, **d)


def _gen(device, *parts) -> torch.Generator:
    h = 1469598103934665603
    for p in parts:
        h = ((h ^ (int(p) & 0xFFFFFFFFFFFFFFFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    g = torch.Generator(device=device)
    g.manual_seed(h & 0x7FFFFFFFFFFFFFFF)
    return g


def centres(s: Spec, device="cpu"):
    """(mu [ncent, D], scales [ncent, D] or None, weights [ncent] or None)."""
    g = _gen(device, s.data_seed, 0)
    if s.kind == "uint8":
        mu = torch.randn(s.ncent, s.D, generator=g, device=device).abs_().mul_(48.0)
    else:
        mu = torch.randn(s.ncent, s.D, generator=g, device=device).mul_(2.0)
    scales = None
    if s.kind == "aniso":
        g1 = _gen(device, s.data_seed, 1)
        scales = torch.rand(s.ncent, s.D, generator=g1, device=device).mul_(1.5).add_(0.5)
    weights = None
    if s.kind == "zipf":
        g1 = _gen(device, s.data_seed, 1)
        perm = torch.randperm(s.ncent, generator=g1, device=device)
        r = torch.arange(1, s.ncent + 1, device=device, dtype=torch.float64)
        w = r.pow(-1.1)
        weights = torch.empty_like(w)
        weights[perm] = w
        weights = weights / weights.sum()
    return mu, scales, weights


def _draw(s: Spec, n: int, cen, g, device):
    mu, scales, weights = cen
    if weights is None:
        lab = torch.randint(0, s.ncent, (n,), generator=g, device=device)
    else:
        lab = torch.multinomial(weights, n, replacement=True, generator=g)
    if s.kind == "uint8":
        x = torch.randn(n, s.D, generator=g, device=device).mul_(16.0).add_(mu[lab])
        return x.clamp_(0.0, 255.0).round_()  # round-half-even
    x = torch.randn(n, s.D, generator=g, device=device)
    if scales is not None:
        x.mul_(scales[lab])
    x.add_(mu[lab])
    if s.kind == "zipf":
        x.div_(x.norm(dim=1, keepdim=True).clamp_min_(1e-30))
    return x


def base_rows(s: Spec, start: int, stop: int, device="cpu", cen=None, out=None) -> torch.Tensor:
    """Base vectors with global ids [start, stop) as fp32 [stop-start, D]."""
    cen = centres(s, device) if cen is None else cen
    if out is None:
        out = torch.empty(stop - start, s.D, dtype=torch.float32, device=device)
    c0 = start // CHUNK
    c1 = (stop + CHUNK - 1) // CHUNK
    for c in range(c0, c1):
        lo = c * CHUNK
        hi = min(lo + CHUNK, s.N)
        a = max(lo, start)
        b = min(hi, stop)
        if a >= b:
            continue
        g = _gen(device, s.data_seed, 3, c)
        x = _draw(s, hi - lo, cen, g, device)
        out[a - start:b - start] = x[a - lo:b - lo]
    return out


def base(s: Spec, device="cpu") -> torch.Tensor:
    return base_rows(s, 0, s.N, device)


def queries(s: Spec, device="cpu", cen=None) -> torch.Tensor:
    cen = centres(s, device) if cen is None else cen
    g = _gen(device, s.data_seed, 5)
    return _draw(s, s.nq, cen, g, device).contiguous()


def init_centroids(s: Spec, device="cpu"):
    """k-means initial centroids for CFG3 (normalised generator centres),
    None for the other configs (seeded sampled init)."""
    if s.kind != "zipf":
        return None
    mu, _, _ = centres(s, device)
    if mu.shape[0] != s.nlist:
        return None
    return (mu / mu.norm(dim=1, keepdim=True)).contiguous()


def shard_range(N: int, rank: int, world: int):
    """Contiguous id slice of rank `rank` (R#21)."""
    return (N * rank) // world, (N * (rank + 1)) // world


def isqrt_ceil(n: int) -> int:
    return int(math.ceil(math.sqrt(n)))
