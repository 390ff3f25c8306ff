"""The five BASELINE.json workloads as seeded synthetic inputs.

The paper's Ariane 5 meshes are proprietary and absent; these
configs stand in with the shapes BASELINE.json states: FP64 Euler, gamma 1.4,
unit cube, transmissive boundaries (kernels.cpp:154-156), Sod / blast initial
states, graded + jittered hex meshes treated as unstructured. Decisions the
configs leave open are fixed here once:

* CFL: 0.5 for config 1 (stated); 0.25 for the 3D blast configs 2-5 (none
  stated; the reference default 0.9 exceeds the ~1/3 3D Rusanov limit,
  SURVEY.md Appendix B.3).
* dt_cap = 1e30 (never binds: Euler wave speeds are > 0).
* Config 2 levels come from a centre-fine grading tuned to ~10/30/60 % of
  cells in tau = 0/1/2 at iteration 0 (jitter alone cannot produce them).
* Config 3/4: geometric stretch from one corner / one wall.
* Config 5: synthetic levels from a seeded smooth size field, smoothed to the
  |dtau| <= 1 fixpoint, injected through the run_iteration-with-plan entry
  with dt = min_c dt_max_c / 2^tau_c.

``scale`` shrinks a config's resolution (same shape, fewer cells) for
CPU-oracle parity tests and smoke runs.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import meshgen

GAMMA = 1.4


def euler_conserved(rho, p, gamma=GAMMA):
    rho = np.asarray(rho, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    w = np.zeros((rho.size, 5))
    w[:, 0] = rho
    w[:, 4] = p / (gamma - 1.0)
    return w


@dataclass
class Config:
    name: str
    n: tuple
    grading: str
    grading_args: tuple
    jitter: float
    permute: bool
    init: str
    init_args: dict
    theta_max: int
    cfl: float
    iterations: int
    seed: int
    dt_cap: float = 1e30
    synthetic_levels: float | None = None  # tau=0 fraction for config 5
    tiles: int = 1  # weak-scaling copies of the unit-cube config along x
    periodic: tuple = ()  # axes with periodic boundaries (meshgen.make_periodic)
    extra: dict = field(default_factory=dict)

    @property
    def n_cells(self):
        return int(np.prod(self.n))

    @property
    def n_faces(self):
        nx, ny, nz = self.n
        return int((nx + 1) * ny * nz + nx * (ny + 1) * nz + nx * ny * (nz + 1))

    def nodes(self):
        axes = []
        for d, n in enumerate(self.n):
            if d == 0 and self.tiles > 1:  # tiles copies of the x grading over [0, tiles]
                one = self._axis(0, n // self.tiles)
                axes.append(np.concatenate([one[:-1] + t for t in range(self.tiles)] + [[float(self.tiles)]]))
                continue
            axes.append(self._axis(d, n))
        return axes

    def _axis(self, d, n):
        g, a = self.grading, self.grading_args
        if g == "uniform":
            return meshgen.uniform_nodes(n)
        if g == "centre":
            return meshgen.centre_graded_nodes(n, *a)
        if g == "corner":
            return meshgen.geometric_nodes(n, a[0])
        if g == "wall_z":
            return meshgen.geometric_nodes(n, a[0]) if d == 2 else meshgen.uniform_nodes(n)
        raise ValueError(g)

    def mesh(self, window=None, lib=None):
        """The config's mesh; `window` = (i0, i1, j0, j1, k0, k1) gives only
        those cells (bitwise the full mesh's cells there, cut sides
        transmissive): bounded samples and slabs. `lib`: the library whose
        generator runs (default the product's; the CPU checkers pass the
        oracle library so a CPU-only process never maps the product)."""
        if window is not None and self.permute:
            raise ValueError("mesh: windows of permuted configs are not supported")
        x, y, z = self.nodes()
        m = meshgen.hex_mesh(x, y, z, jitter=self.jitter, seed=self.seed, permute=self.permute,
                             window=window, lib=lib)
        return meshgen.make_periodic(m, self.periodic) if self.periodic else m

    def initial_state(self, mesh):
        c = mesh["cen"]
        a = self.init_args
        if self.init == "sod":
            left = c[:, 0] < 0.5
            rho = np.where(left, 1.0, 0.125)
            p = np.where(left, 1.0, 0.1)
        else:  # blast (one per tile)
            inside = np.zeros(len(c), dtype=bool)
            for t in range(self.tiles):
                ctr = np.asarray(a["centre"], dtype=np.float64) + np.array([t, 0.0, 0.0])
                inside |= ((c - ctr) ** 2).sum(axis=1) < a["radius"] ** 2
            rho = np.where(inside, a["rho_in"], 1.0)
            p = np.where(inside, a["p_in"], 1.0)
        return euler_conserved(rho, p)

    def options(self):
        from .api import SolverOptions
        return SolverOptions(theta_max=self.theta_max, cfl=self.cfl, dt_cap=self.dt_cap)

    def levels(self, mesh):
        """Config 5: seeded synthetic level field, smoothed (tau in original ids)."""
        rng = np.random.default_rng(self.seed)
        c = mesh["cen"]
        s = np.zeros(len(c))
        for _ in range(6):
            ctr = rng.uniform(0.1, 0.9, 3)
            sig = rng.uniform(0.08, 0.25)
            s += rng.uniform(0.5, 1.0) * np.exp(-((c - ctr) ** 2).sum(axis=1) / (2 * sig * sig))
        s = -s  # small "size" where the bumps are
        f0 = self.synthetic_levels
        qs = np.quantile(s, [f0, f0 + (1 - f0) / 3, f0 + 2 * (1 - f0) / 3])
        tau = np.minimum(np.searchsorted(qs, s, side="right"), self.theta_max).astype(np.int32)
        return smooth_to_fixpoint(mesh, tau)

    def tiled(self, n):
        """Weak-scaling workload: n copies of this config side by side along x
        (domain [0, n] x [0, 1]^2, one blast per copy): every slab rank of an
        n-GPU run owns one copy's worth of cells and work."""
        import copy
        c = copy.deepcopy(self)
        if n > 1:
            c.tiles = n
            c.n = (self.n[0] * n, self.n[1], self.n[2])
            c.name = f"{self.name}-x{n}"
        return c

    def scaled(self, factor):
        """Same config at resolution n / factor (for CPU parity runs)."""
        import copy
        c = copy.deepcopy(self)
        c.n = tuple(max(4, int(round(v / factor))) for v in self.n)
        if c.grading == "corner":
            c.grading_args = (self.grading_args[0] ** factor,)
        if c.grading == "wall_z":
            c.grading_args = (self.grading_args[0] ** factor,)
        c.name = f"{self.name}/{factor}"
        return c


def smooth_to_fixpoint(mesh, tau):
    """Jacobi tau <- min(tau, 1 + min over face neighbours) to the fixpoint
    (levels.cpp:33-51), on the host for synthetic level maps."""
    tau = np.asarray(tau, dtype=np.int32).copy()
    fl, fr = mesh["fl"], mesh["fr"]
    inner = fr >= 0
    a, b = fl[inner], fr[inner]
    while True:
        bound = tau.copy()
        np.minimum.at(bound, a, tau[b] + 1)
        np.minimum.at(bound, b, tau[a] + 1)
        if np.array_equal(bound, tau):
            return tau
        tau = bound


BLAST2 = dict(centre=(0.5, 0.5, 0.5), radius=0.1, p_in=10.0, rho_in=2.0)
BLAST3 = dict(centre=(0.0, 0.0, 0.0), radius=0.1, p_in=20.0, rho_in=3.0)
BLAST4 = dict(centre=(0.5, 0.5, 0.0), radius=0.1, p_in=50.0, rho_in=3.0)
BLAST5 = dict(centre=(0.5, 0.5, 0.5), radius=0.15, p_in=10.0, rho_in=2.0)

CONFIGS = {
    1: Config("cfg1-sod-64^3", (64, 64, 64), "uniform", (), 0.0, True, "sod", {}, 0, 0.5, 200, 1001),
    2: Config("cfg2-blast-100^3-3lvl", (100, 100, 100), "centre", (1.06, 0.04), 0.15, True, "blast",
              BLAST2, 2, 0.25, 50, 1002),
    3: Config("cfg3-corner-200^3-4lvl", (200, 200, 200), "corner", (1.02,), 0.10, False, "blast",
              BLAST3, 3, 0.25, 20, 1003),
    4: Config("cfg4-wall-431^3-5lvl", (431, 431, 431), "wall_z", (1.01,), 0.10, False, "blast",
              BLAST4, 4, 0.25, 10, 1004),
    5: Config("cfg5-synthetic-252^3", (252, 252, 252), "uniform", (), 0.10, False, "blast",
              BLAST5, 3, 0.25, 10, 1005, synthetic_levels=0.10),
}


def get(i, scale=1):
    c = CONFIGS[int(i)]
    return c if scale == 1 else c.scaled(scale)


def periodic_blast():
    """Test workload (not a BASELINE config): a 10x8x6 hex mesh graded in z,
    periodic in x and y, with a blast straddling the x-periodic boundary --
    exercises partner faces in the Euler path."""
    return Config("periodic-blast", (10, 8, 6), "wall_z", (1.15,), 0.0, True, "blast",
                  dict(centre=(0.95, 0.5, 0.3), radius=0.2, rho_in=2.0, p_in=10.0), 2, 0.25, 4, 77,
                  periodic=(0, 1))
