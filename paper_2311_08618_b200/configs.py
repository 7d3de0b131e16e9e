"""Synthetic problem generators for the BASELINE.json configurations.

Each config is a seeded point cloud + kernel + tree/admissibility recipe
(SURVEY.md §8d).  The reference publishes no data for these configurations;
every input here is synthetic and deterministic (numpy default_rng(seed)).

cfg1: 3D 1/r, n=2048 uniform in [0,1]^3, leaf 128, eta=1, eps=1e-8, k=n/2, eps_ev=1e-8
cfg2: 3D 1/r, n=65536 uniform in [0,1]^3, leaf 256, eps=1e-8
cfg3: 2D -log r, n=131072 jittered 512x256 lattice, leaf 256, eps_ev=1e-10
cfg4: 3D Yukawa on the unit sphere, n=262144, leaf 256
cfg5: tight-binding hopping on a helical tube, n=524288, leaf 512, isotropic Morton
"""

from dataclasses import dataclass

import numpy as np

from . import geometry as geo
from .cluster import build_tree, classify, strong


@dataclass(frozen=True)
class ProblemConfig:
    name: str
    n: int
    leaf: int
    eps: float
    eps_ev: float
    ks: tuple
    eta: float = 1.0


CONFIGS = {
    "cfg1": ProblemConfig("cfg1", 2048, 128, 1e-8, 1e-8, (1024,)),
    "cfg2": ProblemConfig("cfg2", 65536, 256, 1e-8, 1e-8, (1, 32768, 65536)),
    "cfg3": ProblemConfig("cfg3", 131072, 256, 1e-8, 1e-10, (65536,)),
    "cfg4": ProblemConfig("cfg4", 262144, 256, 1e-8, 1e-8, tuple(range(131041, 131105))),
    "cfg5": ProblemConfig("cfg5", 524288, 512, 1e-8, 1e-9, (262144, 262145)),
}


def uniform_cube(n, seed=0):
    return geo.PointCloud(np.random.default_rng(seed).uniform(0.0, 1.0, (n, 3)))


def jittered_lattice(nx, ny, seed=0, jitter=0.1):
    """Cell-centred nx x ny lattice in [0,1]^2 with per-axis U(-j h, j h) jitter."""
    rng = np.random.default_rng(seed)
    hx, hy = 1.0 / nx, 1.0 / ny
    gx, gy = np.meshgrid((np.arange(nx) + 0.5) * hx, (np.arange(ny) + 0.5) * hy, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel()], axis=1)
    pts[:, 0] += rng.uniform(-jitter * hx, jitter * hx, pts.shape[0])
    pts[:, 1] += rng.uniform(-jitter * hy, jitter * hy, pts.shape[0])
    return geo.PointCloud(pts)


def unit_sphere(n, seed=0):
    v = np.random.default_rng(seed).standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return geo.PointCloud(v)


def helical_tube(n, seed=0, radius=10.0, bond=1.42, jitter=0.01):
    """Armchair-like tube: rings of 2m atoms, m chosen so the radius is ~10 A."""
    rng = np.random.default_rng(seed)
    a = np.sqrt(3.0) * bond
    m = max(1, int(round(2 * np.pi * radius / a)))
    per_ring = 2 * m
    rings = -(-n // per_ring)
    k = np.arange(rings * per_ring)
    ring, slot = k // per_ring, k % per_ring
    theta = 2 * np.pi * (slot + 0.5 * (ring % 2)) / per_ring
    z = ring * (1.5 * bond / 2.0)
    pts = np.stack([radius * np.cos(theta), radius * np.sin(theta), z], axis=1)[:n]
    pts += rng.normal(0.0, jitter * bond, pts.shape)
    return geo.PointCloud(pts)


def config_cloud(name, seed=0, n=None):
    """Ordered point cloud of a config (n overrides the size for mini-configs)."""
    cfg = CONFIGS[name]
    n = cfg.n if n is None else n
    if name in ("cfg1", "cfg2"):
        cloud = uniform_cube(n, seed)
        iso = False
    elif name == "cfg3":
        ny = 1 << ((n.bit_length() - 1) // 2)
        cloud = jittered_lattice(n // ny, ny, seed)
        iso = False
    elif name == "cfg4":
        cloud = unit_sphere(n, seed)
        iso = False
    else:
        cloud = helical_tube(n, seed)
        iso = True
    return cloud.permuted(geo.sfc_order(cloud, isotropic=iso))


def config_kernel(name, cloud):
    if name in ("cfg1", "cfg2"):
        return geo.InverseDistanceKernel(cloud)
    if name == "cfg3":
        return geo.LogKernel(cloud)
    if name == "cfg4":
        return geo.YukawaKernel(cloud)
    return geo.HoppingKernel(cloud)


def config_problem(name, seed=0, n=None, leaf=None):
    """(cloud, kernel, tree, structure) for a config or a same-recipe mini-config."""
    cfg = CONFIGS[name]
    cloud = config_cloud(name, seed, n)
    tree = build_tree(cloud, cfg.leaf if leaf is None else leaf)
    st = classify(tree, strong(cfg.eta))
    return cloud, config_kernel(name, cloud), tree, st
