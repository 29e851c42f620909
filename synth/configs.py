"""The five BASELINE.json configurations as seeded synthetic inputs.

Stand-ins for the paper's 125/216-particle Janus simulations,
which are not available: dense lattices with jitter (R21) and random sequential
packings (R24).  Draw order per config, rng = numpy default_rng(20260000 + c):
  (1) positions (jitter [Np,3] uniform on [-J, J], or the RSA proposal sequence)
  (2) Janus axes [Np,3] N(0,1), normalised
  (3) external forces F_nc [Np,3] N(0,1)            (R23; torques zero)
then, from fresh generators seeded per purpose (so they do not depend on Nc/N):
  (4) c5 layer densities f, q [N,3] N(0,1)            seed 20260000 + c + 1000
  (5) MVP test vectors lambda ~ U(0,1)^Nc             seed 20260000 + c + 2000 + k
"""
import numpy as np

CONFIGS = {
    1: dict(name="c1", kind="lattice", n=2, spacing=2.05, jitter=0.02, p=8, p_lo=None,
            solve="mono", radius=1.0, mu=1.0, delta=0.1, slip_B=1.0),
    2: dict(name="c2", kind="lattice", n=3, spacing=2.03, jitter=0.015, p=12, p_lo=6,
            solve="both", radius=1.0, mu=1.0, delta=0.1, slip_B=1.0),
    3: dict(name="c3", kind="rsa", np=64, phi=0.30, min_gap=0.005, p=16, p_lo=8,
            solve="bi", radius=1.0, mu=1.0, delta=0.1, slip_B=1.0),
    4: dict(name="c4", kind="lattice", n=6, spacing=2.02, jitter=0.01, p=16, p_lo=8,
            solve="bi", radius=1.0, mu=1.0, delta=0.1, slip_B=1.0),
    5: dict(name="c5", kind="rsa", np=216, phi=0.35, min_gap=0.005, p=24, p_lo=None,
            solve="layer", radius=1.0, mu=1.0, delta=0.1, slip_B=1.0),
}


def _lattice(rng, n, spacing, jitter):
    idx = np.array([(i, j, k) for i in range(n) for j in range(n) for k in range(n)], dtype=np.float64)
    base = (idx - 0.5 * (n - 1)) * spacing
    return base + rng.uniform(-jitter, jitter, size=base.shape)


def _rsa(rng, np_, phi, min_gap, a, max_attempts=10_000_000):
    L = (np_ * (4.0 / 3.0) * np.pi * a ** 3 / phi) ** (1.0 / 3.0)
    out = np.zeros((np_, 3))
    k = 0
    for _ in range(max_attempts):
        c = rng.uniform(0.0, L, size=3)
        if k:
            d = np.sqrt(((out[:k] - c) ** 2).sum(axis=1))
            if (d - 2.0 * a < min_gap).any():
                continue
        out[k] = c
        k += 1
        if k == np_:
            return out
    raise RuntimeError("RSA packing failed after %d attempts" % max_attempts)


def make_config(c):
    """Returns dict(cfg..., centers [Np,3], axes [Np,3], F_nc [Np,3])."""
    cfg = dict(CONFIGS[c])
    rng = np.random.default_rng(20260000 + c)
    if cfg["kind"] == "lattice":
        centers = _lattice(rng, cfg["n"], cfg["spacing"], cfg["jitter"])
    else:
        centers = _rsa(rng, cfg["np"], cfg["phi"], cfg["min_gap"], cfg["radius"])
    npart = centers.shape[0]
    axes = rng.standard_normal((npart, 3))
    axes /= np.linalg.norm(axes, axis=1, keepdims=True)
    F_nc = rng.standard_normal((npart, 3))
    cfg.update(centers=centers, axes=axes, F_nc=F_nc, np=npart, seed=20260000 + c)
    return cfg


def layer_densities(c, N):
    """(f, q) [N,3] each, N(0,1), for the layer-apply workload."""
    rng = np.random.default_rng(20260000 + c + 1000)
    f = rng.standard_normal((N, 3))
    q = rng.standard_normal((N, 3))
    return f, q


def lambda_test(c, nc, k=0):
    """k-th seeded MVP test vector, U(0,1)^nc."""
    rng = np.random.default_rng(20260000 + c + 2000 + k)
    return rng.uniform(0.0, 1.0, size=nc)


def ft_test(c, npart):
    """Seeded force/torque test vector [Np,6] N(0,1) for mobility parity."""
    rng = np.random.default_rng(20260000 + c + 3000)
    return rng.standard_normal((npart, 6))
