"""Synthetic shape sets of BASELINE.json's configs and the
per-shape roofline.

  C0  fp32 Dense N=K=768, M = 1..512 (FFMA validation mode)
  C1  BERT-base encoder, batch 32, GLUE-like sequence lengths 5..128, bf16:
      per T (M = 32*T): QKV (M,2304,768), out-proj (M,768,768),
      FFN1 (M,3072,768), FFN2 (M,768,3072); attention BMM over
      b = 32*12 = 384: scores (T,T,64) and context (T,64,K=T)
  C2  BERT-large attention BMM, b = 64*16 = 1024, T = 1..512
  C3  LLM Dense N=K=4096, M = batch*seq in 1..8192
  C4  10k-shape mixed Dense/BMM sweep (sharded across GPUs)

Inputs are synthetic (no datasets/checkpoints offline): U(-1, 1) cast to
the compute dtype, seeded per (config, shape).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .runtime import bmm_instance, dense_instance

HBM_ROOF_BPS = 8.0e12  # north_star: "HBM bytes at 8 TB/s"
CANONICAL_T = (5, 24, 43, 62, 81, 100, 119, 128)


@dataclass(frozen=True)
class Shape:
    kind: str        # "dense" | "bmm"
    name: str        # qkv | out | ffn1 | ffn2 | scores | context | dense | ...
    batch: int
    M: int
    N: int
    K: int
    b_layout: str    # "nk": B given as [N,K] (weights, K^T); "kn": B as [K,N] (V)
    dynamic: tuple = ("i",)
    in_bytes: int = 2
    out_bytes: int = 2

    @property
    def flops(self) -> int:
        return 2 * self.batch * self.M * self.N * self.K

    @property
    def bytes(self) -> int:
        """Algorithmic HBM bytes: inputs once + output once."""
        return self.in_bytes * self.batch * (self.M * self.K + self.K * self.N) + self.out_bytes * self.batch * self.M * self.N

    @property
    def bytes_padded(self) -> int:
        """Device bytes a ShapeSet allocates for this shape (rows padded to 8)."""
        r8 = lambda n: (n + 7) // 8 * 8  # noqa: E731
        ob = self.out_bytes * self.batch * self.M * (r8(self.N) if self.name == "scores" else self.N)
        ib = self.in_bytes * self.batch * (self.M * r8(self.K) + self.K * self.N)
        return ib + ob

    def t_roof(self, peak_flops: float) -> float:
        return max(self.flops / peak_flops, self.bytes / HBM_ROOF_BPS)

    def bound(self, peak_flops: float) -> str:
        return "tensor" if self.flops / peak_flops >= self.bytes / HBM_ROOF_BPS else "hbm"

    def instance(self):
        eb = self.in_bytes
        if self.kind == "dense":
            return dense_instance(self.M, self.N, self.K, elem_bytes=eb)
        return bmm_instance(self.batch, self.M, self.N, self.K, self.dynamic, elem_bytes=eb)


def glue_seq_lengths(n: int, seed: int = 0) -> list[int]:
    """GLUE-like sequence lengths: clipped log-normal, median ~38, sigma 0.55,
    clipped to [5, 128] (the paper's Fig. 1a has no numeric data)."""
    rng = np.random.default_rng(seed)
    t = np.exp(rng.normal(math.log(38.0), 0.55, size=n))
    return [int(v) for v in np.clip(np.rint(t), 5, 128)]


def bert_layer_shapes(T: int, batch: int = 32, hidden: int = 768, heads: int = 12, ffn: int = 3072) -> list[Shape]:
    M = batch * T
    hd = hidden // heads
    b = batch * heads
    return [
        Shape("dense", "qkv", 1, M, 3 * hidden, hidden, "nk"),
        Shape("dense", "out", 1, M, hidden, hidden, "nk"),
        Shape("dense", "ffn1", 1, M, ffn, hidden, "nk"),
        Shape("dense", "ffn2", 1, M, hidden, ffn, "nk"),
        Shape("bmm", "scores", b, T, T, hd, "nk", ("i", "j")),
        Shape("bmm", "context", b, T, hd, T, "kn", ("i", "k")),
    ]


def c1_shapes(n_draws: int = 24, seed: int = 0) -> list[Shape]:
    """BERT-base Dense+BMM over the 8 canonical T plus n_draws GLUE-like T."""
    ts = list(CANONICAL_T) + glue_seq_lengths(n_draws, seed)
    out: list[Shape] = []
    for T in ts:
        out += bert_layer_shapes(T)
    return out


def c0_shapes(ms=range(1, 513)) -> list[Shape]:
    return [Shape("dense", "dense", 1, m, 768, 768, "kn", ("i",), 4, 4) for m in ms]


def c2_shapes(ts=(1, 8, 64, 128, 257, 384, 512)) -> list[Shape]:
    out = []
    for T in ts:
        out.append(Shape("bmm", "scores", 1024, T, T, 64, "nk", ("i", "j")))
        out.append(Shape("bmm", "context", 1024, T, 64, T, "kn", ("i", "k")))
    return out


def c3_ms(seed: int = 0) -> list[int]:
    ms = set(range(1, 17))
    for p in range(5, 14):
        ms |= {2**p - 1, 2**p, 2**p + 1}
    rng = np.random.default_rng(seed)
    ms |= {int(v) for v in np.exp(rng.uniform(0, math.log(8192), 48)).round().clip(1, 8192)}
    return sorted(ms)


def c3_shapes(seed: int = 0) -> list[Shape]:
    return [Shape("dense", "llm", 1, m, 4096, 4096, "nk") for m in c3_ms(seed)]


def c4_shapes(n: int = 10_000, seed: int = 0) -> list[Shape]:
    rng = np.random.default_rng(seed)
    nk = [(768, 768), (2304, 768), (3072, 768), (768, 3072), (4096, 4096)]
    out = []
    for _ in range(n):
        if rng.random() < 0.5:
            N, K = nk[rng.integers(len(nk))]
            M = int(round(math.exp(rng.uniform(0, math.log(8192)))))
            out.append(Shape("dense", "dense", 1, max(1, M), N, K, "nk"))
        else:
            b = int(rng.choice([384, 1024]))
            T = int(rng.integers(1, 513))
            if rng.random() < 0.5:
                out.append(Shape("bmm", "scores", b, T, T, 64, "nk", ("i", "j")))
            else:
                out.append(Shape("bmm", "context", b, T, 64, T, "kn", ("i", "k")))
    return out


def shard_lpt(shapes: list[Shape], world: int, peak_flops: float) -> list[list[int]]:
    """Longest-processing-time assignment of shapes to ranks by roofline time
    (SURVEY §8e): shapes are independent, so no collective is needed."""
    order = sorted(range(len(shapes)), key=lambda i: -shapes[i].t_roof(peak_flops))
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(i)
        load[r] += shapes[i].t_roof(peak_flops)
    return [sorted(x) for x in out]
