"""The BASELINE.json configurations, their seeded inputs and algorithmic bytes.

Config ids follow SURVEY.md §8(a): D1 DOT fp32 2^24; G1 GEMV fp32 row-major
8192^2; R1 GER fp32 row-major 8192^2; G2/G3 GEMV fp64 col-major 2^20 x 256 and
256 x 2^20; G4 GEMV fp32 row-major 65536^2; D2 DOT fp32 2^32.  No public
dataset is involved — the reference itself only uses seeded synthetic data
(reference bench.hpp:68-71) — so inputs are the seeded SplitMix64 fills of
oracle/cabl_oracle.c (seed 42, streams x=1, y=2, A=3, c=4, C=5).

Algorithmic bytes (s = element bytes, G = GPUs):
  DOT  2 n s          GEMV  m n s + G n s + 2 m s          GER  2 m n s + m s + G n s
Flops follow the reference convention (reference bench.hpp:78-81): DOT 2n,
GEMV 2mn, GER 2mn.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

SEED = 42
STREAM_X, STREAM_Y, STREAM_A, STREAM_C, STREAM_CC = 1, 2, 3, 4, 5


@dataclass(frozen=True)
class Workload:
    id: str
    op: str          # dot | gemv-row | gemv-col | ger
    dtype: torch.dtype
    m: int           # rows (0 for dot)
    n: int           # cols / vector length
    dist: str        # uniform | normal
    shard: str       # how it splits over G GPUs: chunks | rows | none
    desc: str

    @property
    def s(self) -> int:
        return torch.tensor([], dtype=self.dtype).element_size()

    @property
    def dtype_name(self) -> str:
        return "f32" if self.dtype == torch.float32 else "f64"

    def alg_bytes(self, gpus: int = 1) -> int:
        s, m, n = self.s, self.m, self.n
        if self.op == "dot":
            return 2 * n * s
        if self.op.startswith("gemv"):
            return m * n * s + gpus * n * s + 2 * m * s
        return 2 * m * n * s + m * s + gpus * n * s

    def footprint_bytes(self) -> int:
        """Distinct bytes one step touches on one GPU (what has to fit in L2 for a
        back-to-back step to run out of L2): GER's C is read and written in place,
        so it counts once here and twice in alg_bytes."""
        s, m, n = self.s, self.m, self.n
        if self.op == "dot":
            return 2 * n * s
        return m * n * s + m * s + n * s

    def flops(self) -> int:
        return 2 * self.n if self.op == "dot" else 2 * self.m * self.n

    def shard_rows(self, rank: int, world: int) -> tuple[int, int]:
        """Balanced contiguous split of the shardable dimension."""
        total = self.n if self.op == "dot" else self.m
        q, r = divmod(total, world)
        b = rank * q + min(rank, r)
        return b, b + q + (1 if rank < r else 0)


WORKLOADS = {w.id: w for w in [
    Workload("D1", "dot", torch.float32, 0, 1 << 24, "uniform", "chunks",
             "DOT fp32 n=2^24, alpha0=0"),
    Workload("G1", "gemv-row", torch.float32, 8192, 8192, "uniform", "rows",
             "GEMV fp32 row-major 8192x8192"),
    Workload("R1", "ger", torch.float32, 8192, 8192, "uniform", "rows",
             "GER fp32 row-major 8192x8192"),
    Workload("G2", "gemv-col", torch.float64, 1 << 20, 256, "normal", "rows",
             "GEMV fp64 col-major 2^20x256 (tall-skinny)"),
    Workload("G3", "gemv-col", torch.float64, 256, 1 << 20, "normal", "none",
             "GEMV fp64 col-major 256x2^20 (short-wide)"),
    Workload("G4", "gemv-row", torch.float32, 65536, 65536, "uniform", "rows",
             "GEMV fp32 row-major 65536x65536 (16 GiB A)"),
    Workload("D2", "dot", torch.float32, 0, 1 << 32, "uniform", "chunks",
             "DOT fp32 n=2^32 (32 GiB)"),
]}
