"""The BASELINE.json configurations with this build's layout choice.

BASELINE.json fixes (d, k, κ, s, n, dtype); B_r (hence M = k/B_r, B_c = d/M) is part of
the definition of S and is chosen here (SURVEY §8a rule: B_r = 128/κ clamped to
[max(s, 8), 64] for production configs; B_r = 32 for the κ×s sweep; tiny as given).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

SEED = 1234


@dataclass(frozen=True)
class Config:
    name: str
    d: int
    k: int
    kappa: int
    s: int
    n: int
    dtype: str  # "f32" | "bf16"
    B_r: int
    seed: int = SEED

    @property
    def M(self) -> int:
        return self.k // self.B_r

    @property
    def B_c(self) -> int:
        return self.d // self.M

    @property
    def elem(self) -> int:
        return 4 if self.dtype == "f32" else 2

    def sketch_args(self):
        return dict(M=self.M, B_r=self.B_r, B_c=self.B_c, kappa=self.kappa, s=self.s, seed=self.seed)

    def roofline_bytes(self, n: int | None = None) -> int:
        """Algorithmic bytes: read A once, write fp32 Y once (BASELINE.json metric)."""
        n = self.n if n is None else n
        return self.d * n * self.elem + self.k * n * 4

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


TINY = Config("tiny", d=1024, k=256, kappa=2, s=2, n=16, dtype="f32", B_r=32)
LS = Config("ls", d=1 << 20, k=4096, kappa=4, s=4, n=512, dtype="f32", B_r=32)
GRAD = Config("grad", d=1 << 24, k=8192, kappa=8, s=2, n=4096, dtype="bf16", B_r=16)
# narrow inputs (per-example gradient batches, P:1841-1842 low-occupancy case): d large, n small
SMALLN = Config("smalln", d=1 << 24, k=8192, kappa=8, s=2, n=32, dtype="bf16", B_r=16)
# narrow-n experiments (profiles/r02_narrow_n.md): the smalln shape with fewer band entries per input row
SMALLN_K4 = Config("smalln_k4", d=1 << 24, k=8192, kappa=4, s=2, n=32, dtype="bf16", B_r=16)
SMALLN_K2 = Config("smalln_k2", d=1 << 24, k=8192, kappa=2, s=2, n=32, dtype="bf16", B_r=16)
SMALLN_K1 = Config("smalln_k1", d=1 << 24, k=8192, kappa=1, s=1, n=32, dtype="bf16", B_r=16)
SCALEOUT = Config("scaleout", d=1 << 26, k=16384, kappa=8, s=4, n=16384, dtype="bf16", B_r=16)


def sweep(kappa: int, s: int, dtype: str = "bf16") -> Config:
    return Config(f"sweep_k{kappa}_s{s}_{dtype}", d=1 << 22, k=4096, kappa=kappa, s=s, n=1024, dtype=dtype, B_r=32)


def sweep_tuned(kappa: int, s: int, dtype: str = "bf16") -> Config:
    """The same sweep point with B_r chosen per (κ, s) by the production layout rule
    B_r = 128/κ clamped to [max(s, 8), 64] (the paper tunes B_r per shape from a menu of
    templates): κ·B_r = 128 for κ ≥ 2, one band tile of the tcgen05 kernel."""
    B_r = min(64, max(max(s, 8), 128 // kappa))
    return Config(f"sweepT_k{kappa}_s{s}_{dtype}", d=1 << 22, k=4096, kappa=kappa, s=s, n=1024, dtype=dtype, B_r=B_r)


SWEEP = [sweep(k, s, dt) for dt in ("bf16", "f32") for k in (1, 2, 4, 8, 16) for s in (1, 2, 4, 8)]
SWEEP_TUNED = [sweep_tuned(k, s, dt) for dt in ("bf16", "f32") for k in (1, 2, 4, 8, 16) for s in (1, 2, 4, 8)]
# experiment shapes for the transposed layout: the sweep point κ=4 s=4 with short vectors (d = 2^17,
# 256 KiB per bf16 vector) and many of them, same bytes as the sweep
TPROBE = Config("tprobe", d=1 << 17, k=4096, kappa=4, s=4, n=32768, dtype="bf16", B_r=32)
TPROBE2 = Config("tprobe2", d=1 << 19, k=4096, kappa=4, s=4, n=8192, dtype="bf16", B_r=32)
CONFIGS = {c.name: c for c in [TINY, LS, GRAD, SMALLN, SMALLN_K4, SMALLN_K2, SMALLN_K1, SCALEOUT, TPROBE, TPROBE2] + SWEEP + SWEEP_TUNED}
