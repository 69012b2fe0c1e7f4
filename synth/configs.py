"""The five workload configurations of BASELINE.json (`configs[0..4]`).

Paper defaults: degree m=20, truncation p0=20, inherited extra subspace
nex = ceil(0.2 L)  (Appendix D.4 "Experimental Parameter
Configuration"). GRF details are not given by the paper (PAPER.md:759, 789,
807); the recipe below is the one SURVEY.md §8(d) fixes and DESIGN.md states.
"""
from dataclasses import dataclass, field, replace
import math


@dataclass(frozen=True)
class Config:
    name: str
    dim: int                 # 2 or 3
    nx: int                  # interior grid points per axis (ny = nz = nx)
    n_ops: int               # N, operators in the batch
    L: int                   # wanted eigenpairs
    family: str              # "diva" (-div(a grad u)), "lapv" (-Lap u + V u), "divac" (-div(a grad u) + c u),
                             # "vib" (thin plate: Lap(D Lap u) = lambda rho u, standard form)
    K: int                   # GRF modes per axis
    s: float                 # GRF spectral decay exponent: (1+|k|^2)^(-s)
    sigma: float | None      # target domain-RMS std of g (None: raw series)
    vscale: float = 1.0      # coefficient = vscale * exp(g)
    degree: int = 20         # Chebyshev filter degree m
    p0: int = 20             # truncation threshold
    tol: float = 1e-8        # relative residual ||Av - lv|| / ||Av||
    max_iter: int = 200
    chains: int = 8          # contiguous warm-start chains on an 8-GPU box

    @property
    def n(self) -> int:
        return self.nx ** self.dim

    @property
    def nex(self) -> int:
        return int(math.ceil(0.2 * self.L))

    @property
    def b(self) -> int:
        return self.L + self.nex

    @property
    def h(self) -> float:
        return 1.0 / (self.nx + 1)

    @property
    def fields(self) -> int:
        """F: number of parameter fields per operator used by the sort."""
        return 2 if self.family in ("divac", "vib") else 1

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: 2D -div(a grad u), 32x32, a=exp(GRF 8x8, 1/(1+k^2), sigma 0.5), 64 ops, L=16
    "C1": Config("C1", 2, 32, 64, 16, "diva", K=8, s=1.0, sigma=0.5),
    # configs[1]: 2D -Lap u + V u, 100x100, V=10 exp(GRF 16x16, decay 1/(1+k^2)^1.5), 1000 ops, L=100
    "C2": Config("C2", 2, 100, 1000, 100, "lapv", K=16, s=1.5, sigma=None, vscale=10.0),
    # configs[2]: 2D -div(a grad u) + c u, 200x200, a, c lognormal (12x12, sigma 0.7), 400 ops, L=200
    # max_iter 1000: over the full 400-operator queue a few operators converge slowly (cold or warm,
    # e.g. op 290: 415 iterations cold, 521 warm; test_gpu_bench_config.py full-queue test)
    "C3": Config("C3", 2, 200, 400, 200, "divac", K=12, s=1.0, sigma=0.7, max_iter=1000),
    # configs[3]: 3D -div(a grad u), 40^3, a=exp(GRF 6x6x6, sigma 0.5), 200 ops, L=100
    "C4": Config("C4", 3, 40, 200, 100, "diva", K=6, s=1.0, sigma=0.5),
    # configs[4]: 2D -Lap u + V u, 500x500, V lognormal (32x32), 64 ops, L=300
    "C5": Config("C5", 2, 500, 64, 300, "lapv", K=32, s=1.0, sigma=0.5, chains=1),
}

# SURVEY §8(f) f3, beyond BASELINE.json's five configs: the paper's fourth dataset, thin-plate
# vibration Lap(D Lap u) = lambda rho u, D and rho lognormal GRF fields
# ("derived using GRF"), n = 10^4 and L = 200, tol 1e-8 as the paper's smallest
# vibration comparison (caption P:942).
EXTRA_CONFIGS = {
    # max_iter 500: a cold start needs 100-250 outer iterations on this spectrum (beta / lambda_L ~ 2e3)
    "V1": Config("V1", 2, 100, 200, 200, "vib", K=8, s=1.0, sigma=0.3, max_iter=500, chains=8),
}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name] if name in CONFIGS else EXTRA_CONFIGS[name]
    return cfg.with_(**overrides) if overrides else cfg
