"""BASELINE.json's five configs as plain data.

Dependency-free on purpose: bench.py's reference arm loads this file by path
so that it never imports the product package (whose __init__ loads
libddsg_b200.so).  Choices BASELINE.json leaves open are fixed here and
recorded in DESIGN.md §6.
"""
from __future__ import annotations

from dataclasses import dataclass

ZERO_BOUNDARY, MODIFIED_LINEAR = 0, 1  # basis.hpp:22 (ddsg_boundary_mode)


@dataclass
class Config:
    name: str
    d: int
    m: int
    n_points: int
    kind: str  # "grid" or "hdmr"
    seed: int
    # plain grid
    max_level: int = 1
    eps_gamma: float = 0.0
    mode: int = ZERO_BOUNDARY
    target: str = ""
    # hdmr
    level_1d: int = 8
    level_2d: int = 5
    eps_1d: float = 0.0
    eps_2d: float = 0.0
    notes: str = ""


CONFIGS = {
    1: Config("config1_sg_d4_L5", d=4, m=1, n_points=65536, kind="grid", seed=1001, max_level=5,
              eps_gamma=0.0, mode=ZERO_BOUNDARY, target="wl_config1",
              notes="regular grid, hat basis, no boundary points"),
    2: Config("config2_sg_d10_L6", d=10, m=11, n_points=1 << 20, kind="grid", seed=1002, max_level=6,
              eps_gamma=0.0, mode=ZERO_BOUNDARY, target="wl_config2",
              notes="regular grid, hat basis, f_j = prod (1+0.1 j x_k)^0.3, j=0..10"),
    3: Config("config3_asg_d20", d=20, m=21, n_points=1 << 20, kind="grid", seed=1003, max_level=5,
              eps_gamma=1e-3, mode=MODIFIED_LINEAR, target="wl_config3",
              notes="adaptive, eps=1e-3, level capped at 5 (L=10 is infeasible, SURVEY.md finding 4)"),
    4: Config("config4_hdmr_d100", d=100, m=51, n_points=1 << 21, kind="hdmr", seed=1004, level_1d=8,
              level_2d=6, eps_1d=1e-6, eps_2d=1e-6, mode=MODIFIED_LINEAR, target="wl_config4",
              notes="100 1-d cuts (L=8) + 45 2-d cuts on dims 0-9 (L=6), eps_gamma=1e-6, center anchor"),
    5: Config("config5_hdmr_d300", d=300, m=151, n_points=1 << 22, kind="hdmr", seed=1005, level_1d=8,
              level_2d=5, eps_1d=1e-8, eps_2d=1e-8, mode=MODIFIED_LINEAR, target="wl_config5",
              notes="300 1-d cuts (L=8) + 300 seeded-random pair cuts (L=5), kinked policies, center anchor"),
}


