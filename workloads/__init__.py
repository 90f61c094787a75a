"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO arithmetic of the method: it only draws the items and
queries that both the CUDA path and the CPU oracle consume.  Recipe (DESIGN.md
"Input recipe"): numpy ``Generator(PCG64)``; independent streams from
``SeedSequence(seed, spawn_key=...)`` for directions (one child per chunk of
``CHUNK`` rows, so chunked/threaded generation is order-stable), norms and
queries.  Items are ``g/||g||`` (g ~ N(0, I_d), fp64) scaled by a norm drawn
from the config's law, cast to fp32.  Queries are unit Gaussian directions.

The paper's datasets (Netflix, Yahoo!Music, ImageNet SIFT) are not
available; these synthetic stand-ins take their shapes (n, d) and long-tailed
2-norm laws from BASELINE.json.  No dataset record is reproduced.
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

CHUNK = 1 << 16


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    norm_law: str          # "lognormal:<sigma>" or "pareto:<alpha>" (1 + Pareto)
    code_bits: tuple       # SRP hash bits L_h per run
    num_parts: tuple       # m per run
    nq: int
    k: int
    budgets: tuple         # probe budgets as (num, den) fractions of n
    query_batch: int = 1024
    seed: int = 0
    extra_T: tuple = field(default_factory=tuple)  # absolute budgets (recall sweeps)

    def T(self, frac):
        num, den = frac
        return (num * self.n + den - 1) // den   # T = ceil(p * n), integer arithmetic (D13)

    def budget_list(self):
        return [self.T(b) for b in self.budgets]


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": Config("tiny", 10_000, 64, "lognormal:0.5", (32,), (8,), 100, 10, ((1, 100),)),
    # configs[1]: Netflix-shaped
    "c2": Config("c2", 17_770, 300, "lognormal:0.7", (64,), (32,), 1_000, 10,
                 ((5, 1000), (1, 100), (2, 100), (5, 100), (10, 100))),
    # configs[2]: Yahoo!Music-shaped, 64 partitions vs 1 (plain SIMPLE-LSH)
    "c3": Config("c3", 136_736, 300, "pareto:2.5", (64,), (64, 1), 10_000, 10,
                 ((1, 100),), extra_T=tuple([1 << i for i in range(18)] + [136_736])),
    # configs[3]: ImageNet-SIFT-shaped
    "c4": Config("c4", 2_340_373, 150, "lognormal:1.0", (32, 64), (128,), 10_000, 10,
                 ((1, 1000), (1, 100)), extra_T=tuple(1 << i for i in range(22))),
    # configs[4]: scale
    "scale": Config("scale", 16_777_216, 128, "lognormal:1.0", (128,), (256,), 65_536, 100,
                    ((1, 1000),), query_batch=4096),
}


def _seq(seed, *key):
    return np.random.SeedSequence(entropy=seed, spawn_key=tuple(key))


def _draw_norms(cfg: Config, n: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(_seq(cfg.seed, 1)))
    law, p = cfg.norm_law.split(":")
    p = float(p)
    if law == "lognormal":
        return rng.lognormal(mean=0.0, sigma=p, size=n)
    if law == "pareto":
        return 1.0 + rng.pareto(p, size=n)       # classical Pareto, x_m = 1
    raise ValueError(law)


def _unit_rows(rng, rows, d):
    g = rng.standard_normal((rows, d))            # fp64
    nrm = np.sqrt(np.einsum("ij,ij->i", g, g))
    nrm[nrm == 0.0] = 1.0
    return g / nrm[:, None]


def make_items(cfg: Config, n: int | None = None, threads: int = 8) -> np.ndarray:
    """Items X [n x d] fp32: unit Gaussian direction x norm from cfg.norm_law."""
    n = cfg.n if n is None else n
    norms = _draw_norms(cfg, cfg.n)[:n]
    X = np.empty((n, cfg.d), np.float32)
    nchunks = (n + CHUNK - 1) // CHUNK

    def work(c):
        r0 = c * CHUNK
        r1 = min(n, r0 + CHUNK)
        rng = np.random.Generator(np.random.PCG64(_seq(cfg.seed, 0, c)))
        u = _unit_rows(rng, CHUNK, cfg.d)[: r1 - r0]
        X[r0:r1] = (u * norms[r0:r1, None]).astype(np.float32)

    if nchunks == 1 or threads <= 1:
        for c in range(nchunks):
            work(c)
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(work, range(nchunks)))
    return X


def make_queries(cfg: Config, nq: int | None = None, shard: int = 0) -> np.ndarray:
    """Unit Gaussian queries Q [nq x d] fp32.  ``shard`` selects an independent
    stream (multi-GPU query sharding draws a distinct set per rank)."""
    nq = cfg.nq if nq is None else nq
    rng = np.random.Generator(np.random.PCG64(_seq(cfg.seed, 2, shard)))
    return _unit_rows(rng, nq, cfg.d).astype(np.float32)


def shard_range(total: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of ``total`` units for ``rank`` of ``world``."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi


def scaled(cfg: Config, n: int, nq: int) -> Config:
    """Same law/shape family at a reduced size (parity tests)."""
    from dataclasses import replace
    return replace(cfg, name=f"{cfg.name}@{n}", n=n, nq=nq)
