"""Seeded synthetic instance generator shared by the oracle tests, the CUDA path and bench.py.

This module holds PROBLEM DATA only -- grids, control tables, coefficient tables, the Dirichlet
kind mask (free / target / obstacle) and the boundary-subset table Gamma_p -- and none of the
method's arithmetic (no scheme, no interpolation, no argmin, no labelling).  Both sides of the
parity tests (``oracle/`` and ``paper_1502_01629_b200``) consume the arrays built here.

Citations: ``P:<line>`` = PAPER.md (arXiv 1502.01629 LaTeX source), ``S:<line>`` = SPEC.md,
configs C1..C5 = BASELINE.json ``configs[0..4]``.

* Problem statement, Eq. (HJB2): dynamics f(x,a), diffusion columns sigma_k(x), running
  cost l(x), Dirichlet data g.  Here f(x,a) = c(x) * a + d(x) (speed c, drift d).
* Control set A discretised by N_A points "by direct comparison" P:376-377; A = unit circle,
  a_k = (cos 2 pi k / N_A, sin 2 pi k / N_A), k = 0.. from (1,0) counter-clockwise.
* Dirichlet set: a target ball with V = 0 and (C4) obstacle discs with V = 1/lambda.  Target
  membership is the integer lattice rule di^2 + dj^2 <= (r/dx)^2 + 1e-9 (reading R7).
* Boundary split Gamma_p: target nodes are split into N_P angular sectors about
  the target centre, sector = floor(N_P * theta / 2 pi), theta = atan2(dj, di) in [0, 2 pi)
  (reading R17).  Tabulated here so both sides read the same integers.
* Grid: n nodes per axis on [lo, hi]^2, node (i, j) at (lo + i dx, lo + j dx), linear index
  j * n + i (x fastest).

Random numbers (C3 Fourier modes, C4 obstacle discs) come from ``numpy.random.Generator(PCG64)``
with the seeds fixed in DESIGN.md (1502 for C3, 1629 for C4).
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

COEF_CONST, COEF_ROW, COEF_COL, COEF_FIELD = 0, 1, 2, 3
KIND_FREE, KIND_TARGET, KIND_OBSTACLE = 0, 1, 2


@dataclasses.dataclass
class Coef:
    """A coefficient of the problem: constant, per-row (depends on x2 only), per-column
    (depends on x1 only) or a full n*n field (row-major, x fastest)."""
    kind: int = COEF_CONST
    value: float = 0.0
    data: Optional[np.ndarray] = None

    @staticmethod
    def const(v: float) -> "Coef":
        return Coef(COEF_CONST, float(v), None)

    @staticmethod
    def row(values: np.ndarray) -> "Coef":
        return Coef(COEF_ROW, 0.0, np.ascontiguousarray(values, dtype=np.float64))

    @staticmethod
    def field(values: np.ndarray) -> "Coef":
        return Coef(COEF_FIELD, 0.0, np.ascontiguousarray(values, dtype=np.float64).reshape(-1))

    def at(self, i: int, j: int, n: int) -> float:
        if self.kind == COEF_CONST:
            return self.value
        if self.kind == COEF_ROW:
            return float(self.data[j])
        if self.kind == COEF_COL:
            return float(self.data[i])
        return float(self.data[j * n + i])

    def max_abs(self) -> float:
        if self.kind == COEF_CONST:
            return abs(self.value)
        return float(np.max(np.abs(self.data))) if self.data.size else 0.0


@dataclasses.dataclass
class Instance:
    """One discretised problem on one grid (fine or coarse)."""
    name: str
    n: int
    lo: float
    hi: float
    dx: float
    h: float
    lam: float
    controls: np.ndarray            # (N_A, 2) float64
    speed: Coef                     # c(x)
    drift: tuple                    # (d1(x), d2(x))
    p: int                          # number of noise columns sigma_k (0, 1, 2)
    sigma: tuple                    # ((s00, s01), (s10, s11)): sigma[k][component]
    cost: Coef                      # l(x)
    kind: np.ndarray                # (n*n,) uint8: 0 free, 1 target, 2 obstacle
    sector: np.ndarray              # (n*n,) int32: Gamma_p id of target nodes, -1 elsewhere
    diffusion_scale: int = 0        # 0: sqrt(h p) (north star), 1: sqrt(h)
    n_patches: int = 1
    static_blocks: tuple = (1, 1)   # (px, py) for the static equal-square decomposition
    coarse: Optional["Instance"] = None
    tol: float = 1e-9               # fine-grid sup-norm tolerance
    tol_coarse: float = 1e-12
    precision: int = 64
    meta: dict = dataclasses.field(default_factory=dict)
    # general nonlinear terms (readings R32, R33)
    sigma_mode: int = 0             # 1: one noise column along the control, sigma(x,a) = s(x) a,
                                    #    s = sigma[0][0] (p = 1)
    cost_ctrl: Optional[np.ndarray] = None   # (N_A,) additive per-control cost m(a_k)

    @property
    def n_controls(self) -> int:
        return int(self.controls.shape[0])

    @property
    def beta(self) -> float:
        return 1.0 / (1.0 + self.lam * self.h)

    def x(self, i) -> np.ndarray:
        return self.lo + np.asarray(i, dtype=np.float64) * self.dx

    def free_count(self) -> int:
        return int(np.count_nonzero(self.kind == KIND_FREE))

    def fingerprint(self) -> str:
        """SHA-256 over every array and scalar that defines the instance."""
        hsh = hashlib.sha256()
        for v in (self.n, self.lo, self.hi, self.dx, self.h, self.lam, self.p,
                  self.diffusion_scale, self.n_patches):
            hsh.update(repr(v).encode())
        hsh.update(self.controls.tobytes())
        for c in (self.speed, self.drift[0], self.drift[1], self.cost,
                  self.sigma[0][0], self.sigma[0][1], self.sigma[1][0], self.sigma[1][1]):
            hsh.update(repr((c.kind, c.value)).encode())
            if c.data is not None:
                hsh.update(c.data.tobytes())
        hsh.update(self.kind.tobytes())
        hsh.update(self.sector.tobytes())
        if self.sigma_mode:
            hsh.update(b"sigma_mode=%d" % self.sigma_mode)
        if self.cost_ctrl is not None:
            hsh.update(np.ascontiguousarray(self.cost_ctrl, dtype=np.float64).tobytes())
        if self.coarse is not None:
            hsh.update(self.coarse.fingerprint().encode())
        return hsh.hexdigest()


# --------------------------------------------------------------------------------------------
# building blocks
# --------------------------------------------------------------------------------------------

def unit_circle_controls(n_a: int) -> np.ndarray:
    """a_k = (cos 2 pi k/N_A, sin 2 pi k/N_A), k = 0..N_A-1."""
    if n_a < 1:
        raise ValueError("N_A must be >= 1")
    k = np.arange(n_a, dtype=np.float64)
    ang = 2.0 * math.pi * k / n_a
    c = np.cos(ang)
    s = np.sin(ang)
    # exact cardinal directions (cos(pi/2) is 6e-17 in fp64): keep the table symmetric
    c[np.abs(c) < 1e-15] = 0.0
    s[np.abs(s) < 1e-15] = 0.0
    return np.ascontiguousarray(np.stack([c, s], axis=1))


def grid_params(n: int, lo: float, hi: float):
    if n < 3:
        raise ValueError("n must be >= 3 (S:48)")
    if not hi > lo:
        raise ValueError("hi must exceed lo")
    dx = (hi - lo) / (n - 1)
    return dx


def ball_target(n: int, lo: float, dx: float, centre, radius: float) -> np.ndarray:
    """Boolean (n*n) mask of target nodes: integer lattice rule about the centre node,
    di^2 + dj^2 <= (r/dx)^2 + 1e-9 (inclusive)."""
    ic = int(round((centre[0] - lo) / dx))
    jc = int(round((centre[1] - lo) / dx))
    rr = (radius / dx) ** 2 + 1e-9
    ii = np.arange(n)
    di2 = (ii - ic) ** 2
    dj2 = (ii - jc) ** 2
    mask = (dj2[:, None] + di2[None, :]) <= rr
    return mask.reshape(-1), (ic, jc)


def sector_table(n: int, mask: np.ndarray, centre_idx, n_patches: int) -> np.ndarray:
    """Gamma_p: sector id of each target node (angular split about the target centre)."""
    sec = np.full(n * n, -1, dtype=np.int32)
    idx = np.nonzero(mask)[0]
    j = idx // n
    i = idx % n
    th = np.arctan2((j - centre_idx[1]).astype(np.float64), (i - centre_idx[0]).astype(np.float64))
    th = np.where(th < 0.0, th + 2.0 * math.pi, th)
    s = np.floor(n_patches * th / (2.0 * math.pi)).astype(np.int64)
    s = np.clip(s, 0, n_patches - 1)
    sec[idx] = s.astype(np.int32)
    return sec


def make_instance(name: str, n: int, lo: float, hi: float, *, n_a: int, lam: float,
                  speed: Coef = None, drift=None, p: int = 0, sigma=None, cost: Coef = None,
                  kind: np.ndarray, sector: np.ndarray = None, h: float = None,
                  diffusion_scale: int = 0, **kw) -> Instance:
    dx = grid_params(n, lo, hi)
    z = Coef.const(0.0)
    inst = Instance(
        name=name, n=n, lo=float(lo), hi=float(hi), dx=dx, h=dx if h is None else float(h),
        lam=float(lam), controls=unit_circle_controls(n_a),
        speed=speed if speed is not None else Coef.const(1.0),
        drift=tuple(drift) if drift is not None else (z, z),
        p=int(p), sigma=sigma if sigma is not None else ((z, z), (z, z)),
        cost=cost if cost is not None else Coef.const(1.0),
        kind=np.ascontiguousarray(kind, dtype=np.uint8).reshape(-1),
        sector=(np.ascontiguousarray(sector, dtype=np.int32).reshape(-1) if sector is not None
                else np.where(np.asarray(kind).reshape(-1) == KIND_TARGET, 0, -1).astype(np.int32)),
        diffusion_scale=diffusion_scale, **kw)
    return inst


# --------------------------------------------------------------------------------------------
# BASELINE.json configs C1..C5 (and the same physics on other grid sizes)
# --------------------------------------------------------------------------------------------

FULL_N = {"C1": 51, "C2": 401, "C3": 2049, "C4": 4097, "C5": 8193}
FULL_NC = {"C1": None, "C2": 51, "C3": 129, "C4": 257, "C5": 513}
COARSE_RATIO = {"C2": 8, "C3": 16, "C4": 16, "C5": 16}


def _fourier_speed_modes():
    """C3: 8 Fourier modes, omega ~ U[1,4], theta ~ U[0,2pi), phi ~ U[0,2pi), PCG64(1502),
    drawn in the order (omega, theta, phi) per mode (reading R23)."""
    rng = np.random.Generator(np.random.PCG64(1502))
    modes = []
    for _ in range(8):
        om = rng.uniform(1.0, 4.0)
        th = rng.uniform(0.0, 2.0 * math.pi)
        ph = rng.uniform(0.0, 2.0 * math.pi)
        modes.append((om, th, ph))
    return modes


def c3_speed_field(n: int, lo: float, dx: float) -> np.ndarray:
    x = lo + np.arange(n) * dx
    X1, X2 = np.meshgrid(x, x, indexing="xy")   # X1[j, i] = x_i, X2[j, i] = x_j
    m = np.zeros_like(X1)
    for om, th, ph in _fourier_speed_modes():
        m += np.cos(om * (math.cos(th) * X1 + math.sin(th) * X2) + ph)
    m /= math.sqrt(8.0)
    return np.clip(1.0 + 0.5 * m, 0.25, 1.75)


C4_TARGET = (1.5, 1.5)
C4_TARGET_R = 0.05


def c4_obstacle_discs():
    """C4: 20 discs, PCG64(1629); per disc cx, cy ~ U[-2,2] then r ~ U[0.05,0.2]; redraw when
    the disc comes within r + 0.05 + 2 dx_fine of the target centre (reading R24, dx_fine of
    the full 4097 grid so every grid size sees the same discs)."""
    rng = np.random.Generator(np.random.PCG64(1629))
    dx_full = 4.0 / (FULL_N["C4"] - 1)
    discs = []
    while len(discs) < 20:
        cx = rng.uniform(-2.0, 2.0)
        cy = rng.uniform(-2.0, 2.0)
        r = rng.uniform(0.05, 0.2)
        if math.hypot(cx - C4_TARGET[0], cy - C4_TARGET[1]) < r + C4_TARGET_R + 2.0 * dx_full:
            continue
        discs.append((cx, cy, r))
    return discs


def _config_instance(cfg: str, n: int, n_coarse: Optional[int], *, coarse_level=False) -> Instance:
    z = Coef.const(0.0)
    if cfg in ("C1", "C2"):
        lo, hi = -1.0, 1.0
        n_a = 16 if cfg == "C1" else 32
        s = 0.05 if cfg == "C1" else 0.02
        lam = 1.0
        centre, rad = (0.0, 0.0), 0.1
        dx = grid_params(n, lo, hi)
        tmask, cidx = ball_target(n, lo, dx, centre, rad)
        kind = np.where(tmask, KIND_TARGET, KIND_FREE).astype(np.uint8)
        npatch = 1 if cfg == "C1" else 16
        p = 0 if coarse_level else 2
        sig = ((Coef.const(s), z), (z, Coef.const(s)))
        inst = make_instance(cfg, n, lo, hi, n_a=n_a, lam=lam, p=p, sigma=sig, kind=kind,
                             sector=sector_table(n, tmask, cidx, npatch),
                             n_patches=npatch, static_blocks=(1, 1) if cfg == "C1" else (4, 4))
    elif cfg == "C3":
        lo, hi = -2.0, 2.0
        dx = grid_params(n, lo, hi)
        tmask, cidx = ball_target(n, lo, dx, (0.0, 0.0), 0.05)
        kind = np.where(tmask, KIND_TARGET, KIND_FREE).astype(np.uint8)
        s = 0.01
        sig = ((Coef.const(s), z), (z, Coef.const(s)))
        inst = make_instance(cfg, n, lo, hi, n_a=32, lam=1.0,
                             speed=Coef.field(c3_speed_field(n, lo, dx)),
                             p=0 if coarse_level else 2, sigma=sig, kind=kind,
                             sector=sector_table(n, tmask, cidx, 64), n_patches=64,
                             static_blocks=(8, 8))
    elif cfg == "C4":
        lo, hi = -2.0, 2.0
        dx = grid_params(n, lo, hi)
        tmask, cidx = ball_target(n, lo, dx, C4_TARGET, C4_TARGET_R)
        x = lo + np.arange(n) * dx
        X1, X2 = np.meshgrid(x, x, indexing="xy")
        obst = np.zeros((n, n), dtype=bool)
        for cx, cy, r in c4_obstacle_discs():
            obst |= ((X1 - cx) ** 2 + (X2 - cy) ** 2) <= r * r
        obst = obst.reshape(-1) & ~tmask
        kind = np.where(tmask, KIND_TARGET, np.where(obst, KIND_OBSTACLE, KIND_FREE)).astype(np.uint8)
        # sigma_1(x) = 0.02 * (x2, 0): one noise column, per-row table (degenerate on x2 = 0)
        sig = ((Coef.row(0.02 * x), z), (z, z))
        inst = make_instance(cfg, n, lo, hi, n_a=48, lam=1.0, p=0 if coarse_level else 1,
                             sigma=sig, kind=kind, sector=sector_table(n, tmask, cidx, 128),
                             n_patches=128, static_blocks=(16, 8))
    elif cfg == "C5":
        lo, hi = -2.0, 2.0
        dx = grid_params(n, lo, hi)
        tmask, cidx = ball_target(n, lo, dx, (0.0, 0.0), 0.02)
        kind = np.where(tmask, KIND_TARGET, KIND_FREE).astype(np.uint8)
        x = lo + np.arange(n) * dx
        d1 = 0.5 * np.sin(math.pi * x)                       # Zermelo current (0.5 sin(pi x2), 0)
        s = 0.005
        sig = ((Coef.const(s), z), (z, Coef.const(s)))
        inst = make_instance(cfg, n, lo, hi, n_a=64, lam=0.5, drift=(Coef.row(d1), z),
                             p=0 if coarse_level else 2, sigma=sig, kind=kind,
                             sector=sector_table(n, tmask, cidx, 256), n_patches=256,
                             static_blocks=(16, 16))
    else:
        raise KeyError(cfg)
    inst.meta["config"] = cfg
    if coarse_level:
        inst.name = cfg + "-coarse"
        return inst
    inst.precision = 64 if cfg == "C1" else 32
    # R12: fp32 runs stop at a verified residual < 1e-7; at C5 a residual of 1e-6 still leaves
    # 8e-5 max|V| of error (amplification up to 1/(1-beta) = 4097), 1e-7 leaves 6e-6 max|V|
    inst.tol = 1e-9 if cfg == "C1" else 1e-7
    if n_coarse is not None:
        if (n - 1) % (n_coarse - 1) != 0:
            raise ValueError("coarse grid must nest in the fine grid")
        inst.coarse = _config_instance(cfg, n_coarse, None, coarse_level=True)
    return inst


def make_config(cfg: str, n: Optional[int] = None, n_coarse: Optional[int] = None) -> Instance:
    """Instance for BASELINE config ``cfg`` (C1..C5).  ``n`` overrides the fine grid size (same
    physics and domain, used for parity-sized runs); ``n_coarse`` defaults to keep the config's
    coarse/fine ratio (8 for C2, 16 for C3-C5) with at least 9 coarse nodes."""
    n_full = FULL_N[cfg]
    n = n_full if n is None else int(n)
    if n_coarse is None and FULL_NC[cfg] is not None:
        if n == n_full:
            n_coarse = FULL_NC[cfg]
        else:
            r = COARSE_RATIO[cfg]
            while r > 1 and ((n - 1) % r != 0 or (n - 1) // r < 8):
                r //= 2
            n_coarse = (n - 1) // r + 1
    inst = _config_instance(cfg, n, n_coarse)
    inst.name = cfg if n == n_full else f"{cfg}@{n}"
    return inst


def halfplane_instance(n: int = 21, n_a: int = 16, lam: float = 1.0, sigma: float = 0.0,
                       edge_cells: int = 2) -> Instance:
    """Target = half-plane {x1 <= x0} (columns i < edge_cells), sigma = s I, f = a, h = dx on
    [0, 1]^2.  Used by pins P4 (exact geometric series), P5 (1-D reduction) and P17."""
    lo, hi = 0.0, 1.0
    kind = np.zeros((n, n), dtype=np.uint8)
    kind[:, :edge_cells] = KIND_TARGET
    z = Coef.const(0.0)
    p = 2 if sigma > 0 else 0
    sig = ((Coef.const(sigma), z), (z, Coef.const(sigma)))
    return make_instance("halfplane", n, lo, hi, n_a=n_a, lam=lam, p=p, sigma=sig, kind=kind)


def exit_instance(n: int, *, problem: str = "eikonal", eps: float = 0.0, h_ratio: float = 0.5,
                  n_a: int = 16) -> Instance:
    """The paper's exit-time setup: Omega = [-1,1]^2, g = 0 on the boundary (kind =
    target on the boundary ring), l = 1, no discount (lambda = 0), sigma = sqrt(2 eps) I
    with the paper's sqrt(h) scaling (diffusion_scale=1), h = h_ratio * dx.
    ``problem``: 'eikonal' (f = a), 'advection' (f = -b with b = (1,0), reading R25)."""
    lo, hi = -1.0, 1.0
    kind = np.zeros((n, n), dtype=np.uint8)
    kind[0, :] = kind[-1, :] = kind[:, 0] = kind[:, -1] = KIND_TARGET
    dx = grid_params(n, lo, hi)
    z = Coef.const(0.0)
    s = math.sqrt(2.0 * eps)
    p = 2 if eps > 0 else 0
    sig = ((Coef.const(s), z), (z, Coef.const(s)))
    if problem == "eikonal":
        speed, drift = Coef.const(1.0), (z, z)
    elif problem == "advection":
        speed, drift = Coef.const(0.0), (Coef.const(-1.0), z)
    else:
        raise KeyError(problem)
    return make_instance(f"exit-{problem}", n, lo, hi, n_a=n_a, lam=0.0, speed=speed,
                         drift=drift, p=p, sigma=sig, kind=kind, h=h_ratio * dx,
                         diffusion_scale=1)


def boundary_side_sectors(n: int, mask: np.ndarray, n_patches: int) -> np.ndarray:
    """Gamma_p for a boundary-ring Dirichlet set (exit problems): angular sectors about the box
    centre rotated by pi/4, so that n_patches = 4 gives the four sides of the square (P:1107,
    reading R34); corner nodes belong to the side counter-clockwise of them."""
    sec = np.full(n * n, -1, dtype=np.int32)
    idx = np.nonzero(mask)[0]
    c = 0.5 * (n - 1)
    th = np.arctan2(idx // n - c, idx % n - c) + 0.25 * math.pi
    th = np.mod(th, 2.0 * math.pi)
    sec[idx] = np.minimum(np.floor(n_patches * th / (2.0 * math.pi)).astype(np.int64), n_patches - 1)
    return sec


def general_instance(n: int, *, cost: int = 3, sigma: int = 3, eps: float = 0.1,
                     lam: float = 0.0, h_ratio: float = 0.5, n_a: int = 16,
                     n_coarse: Optional[int] = None, n_patches: int = 4,
                     coarse_level: bool = False) -> Instance:
    """The paper's general nonlinear test on the exit-time setup of P:878-885
    (Omega = [-1,1]^2, g = 0 on the boundary ring, 16 controls on the unit circle, sqrt(h)
    scaling, h = h_ratio dx; lam = 0: no discount as in the paper):
        f(x,a) = c(x) a,  c(x) = 1 + max{x2, max{x1, 0}}                         Eq. (nonomog)
        d_eps(x) = sqrt(2 eps) chi_{x2 >= 0}(x)
        sigma_1 = 0,  sigma_2(x) = d_eps(x) I_2,  sigma_3(x,a) = d_eps(x) a      Eq. (s123)
        l_1 = 1,  l_2(x) = 1 + |x1 x2|,  l_3(x,a) = 1 + |x1 x2| + |a1 / (2 + a2)|  Eq. (l123)
    ``cost`` / ``sigma`` select i, j in 1..3.  m(a) = |a1/(2+a2)| is tabulated per control (problem
    data, fp64)."""
    if cost not in (1, 2, 3) or sigma not in (1, 2, 3):
        raise ValueError("cost and sigma select l_1..l_3 and sigma_1..sigma_3")
    lo, hi = -1.0, 1.0
    dx = grid_params(n, lo, hi)
    x = lo + np.arange(n) * dx
    X1, X2 = np.meshgrid(x, x, indexing="xy")          # [j, i]: X1 varies along i (x fastest)
    kind = np.zeros((n, n), dtype=np.uint8)
    kind[0, :] = kind[-1, :] = kind[:, 0] = kind[:, -1] = KIND_TARGET
    speed = Coef.field(1.0 + np.maximum(X2, np.maximum(X1, 0.0)))
    d = Coef.row(np.where(x >= 0.0, math.sqrt(2.0 * eps), 0.0))
    z = Coef.const(0.0)
    p, sig, smode = 0, ((z, z), (z, z)), 0
    if sigma == 2 and not coarse_level:
        p, sig = 2, ((d, z), (z, d))
    elif sigma == 3 and not coarse_level:
        p, sig, smode = 1, ((d, z), (z, z)), 1
    lc = Coef.const(1.0) if cost == 1 else Coef.field(1.0 + np.abs(X1 * X2))
    ctrl = unit_circle_controls(n_a)
    cc = np.abs(ctrl[:, 0] / (2.0 + ctrl[:, 1])) if cost == 3 else None
    mask = kind.reshape(-1) == KIND_TARGET
    inst = make_instance(f"general-l{cost}s{sigma}", n, lo, hi, n_a=n_a, lam=lam, speed=speed,
                         p=p, sigma=sig, cost=lc, kind=kind, h=h_ratio * dx, diffusion_scale=1,
                         sigma_mode=smode, cost_ctrl=cc,
                         sector=boundary_side_sectors(n, mask, n_patches), n_patches=n_patches,
                         static_blocks=(2, 2))
    inst.meta.update(cost=cost, sigma=sigma, eps=eps)
    if coarse_level:
        inst.name += "-coarse"
    elif n_coarse is not None:
        if (n - 1) % (n_coarse - 1) != 0:
            raise ValueError("coarse grid must nest in the fine grid")
        # the coarse solve is the sigma = 0 problem on G_c with the same h / dx ratio
        inst.coarse = general_instance(n_coarse, cost=cost, sigma=sigma, eps=eps, lam=lam,
                                       h_ratio=h_ratio, n_a=n_a, n_patches=n_patches,
                                       coarse_level=True)
    return inst


PAPER_FMINMAX = {"eikonal": (1.0, 1.0), "zermelo": (1.0 / 6.0, 1.5)}


def paper_time_step(dx: float, eps: float, f_min: float, f_max: float) -> float:
    """The paper's time step h = alpha dx / f_min: alpha = 1/(1 + Upsilon) when the upwind
    diffusion ball condition 2 eps / f_min < dx / (1 + Upsilon) holds, otherwise
    0.99 alpha_hi of Eq. (upper-alpha) so that h f_max + sqrt(2 eps h) < dx is kept (
    DESIGN.md readings R36, R37).  Parameter choice only (problem data), no scheme arithmetic."""
    ups = f_max / f_min
    if eps <= 0.0 or (2.0 * eps / f_min) < (dx / (1.0 + ups)) * (1.0 - 1e-12):
        alpha = 1.0 / (1.0 + ups)
    else:
        om = f_min / (2.0 * eps)
        alpha = 0.99 * (1.0 / ups - (math.sqrt(1.0 + 4.0 * om * dx * ups) - 1.0) / (2.0 * om * dx * ups * ups))
    return alpha * dx / f_min


def paper_instance(problem: str, cells: int, eps: float, *, coarse_cells: Optional[int] = 50,
                   eta: float = 1.0, theta: float = 0.25 * math.pi, n_a: int = 16,
                   coarse_level: bool = False) -> Instance:
    """The workloads of the paper's performance comparison (Tables 1 and 2):
    Omega = [-1,1]^2 with ``cells`` cells per axis (the tables' "100^2 ... 800^2", dx = 2/cells,
    reading Q26/R26), exit problem g = 0 on the boundary (lambda = 0), l = 1, 16 controls on the
    unit circle, sigma = sqrt(2 eps) I with the paper's sqrt(h) scaling, h from
    paper_time_step, boundary split into the four sides of the square, static
    decomposition = four squares, coarse grid of 50^2 cells.
      eikonal  (problem B, c = 1):  f(x,a) = a
      zermelo  (problem C):         f(x,a) = (R_theta x/|x| + eta a / 2) / (1 + |x|^2)
               theta = pi/4 and x/|x| := 0 at x = 0 (reading R35)."""
    if problem not in PAPER_FMINMAX:
        raise KeyError(problem)
    lo, hi = -1.0, 1.0
    n = cells + 1
    dx = grid_params(n, lo, hi)
    fmin, fmax = PAPER_FMINMAX[problem]
    h = paper_time_step(dx, eps, fmin, fmax)
    x = lo + np.arange(n) * dx
    X1, X2 = np.meshgrid(x, x, indexing="xy")
    kind = np.zeros((n, n), dtype=np.uint8)
    kind[0, :] = kind[-1, :] = kind[:, 0] = kind[:, -1] = KIND_TARGET
    z = Coef.const(0.0)
    if problem == "eikonal":
        speed, drift = Coef.const(1.0), (z, z)
    else:
        r2 = X1 * X1 + X2 * X2
        r = np.sqrt(r2)
        inv = np.where(r > 0.0, 1.0 / np.where(r > 0.0, r, 1.0), 0.0) / (1.0 + r2)
        ct, st = math.cos(theta), math.sin(theta)
        speed = Coef.field(0.5 * eta / (1.0 + r2))
        drift = (Coef.field((ct * X1 - st * X2) * inv), Coef.field((st * X1 + ct * X2) * inv))
    s = math.sqrt(2.0 * eps)
    p = 2 if (eps > 0.0 and not coarse_level) else 0
    sig = ((Coef.const(s), z), (z, Coef.const(s)))
    mask = kind.reshape(-1) == KIND_TARGET
    inst = make_instance(f"paper-{problem}-{cells}", n, lo, hi, n_a=n_a, lam=0.0, speed=speed,
                         drift=drift, p=p, sigma=sig, kind=kind, h=h, diffusion_scale=1,
                         sector=boundary_side_sectors(n, mask, 4), n_patches=4,
                         static_blocks=(2, 2))
    inst.meta.update(problem=problem, eps=eps, cells=cells, f_min=fmin, f_max=fmax)
    if coarse_level:
        inst.name += "-coarse"
    elif coarse_cells is not None:
        if cells % coarse_cells != 0:
            raise ValueError("coarse grid must nest in the fine grid")
        # same h/dx ratio on G_c (the coarse problem is the sigma = 0 problem there)
        c = paper_instance(problem, coarse_cells, 0.0, coarse_cells=None, eta=eta, theta=theta,
                           n_a=n_a, coarse_level=True)
        c.h = h * (c.dx / dx)
        inst.coarse = c
    return inst


def random_instance(n: int, seed: int, *, n_a: int = 8, p: int = 2, lam: float = 1.0,
                    field_speed: bool = True, obstacles: bool = True) -> Instance:
    """Small random instance (for brute force / schedule-independence pins): random positive
    speed field, random constant drift, random diffusion, a few random target/obstacle nodes."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lo, hi = 0.0, 1.0
    kind = np.zeros(n * n, dtype=np.uint8)
    kind[rng.choice(n * n, size=max(1, n * n // 20), replace=False)] = KIND_TARGET
    if obstacles:
        cand = np.nonzero(kind == KIND_FREE)[0]
        kind[rng.choice(cand, size=max(1, n * n // 30), replace=False)] = KIND_OBSTACLE
    dx = grid_params(n, lo, hi)
    speed = Coef.field(rng.uniform(0.5, 1.5, size=n * n)) if field_speed else Coef.const(1.0)
    drift = (Coef.const(rng.uniform(-0.3, 0.3)), Coef.const(rng.uniform(-0.3, 0.3)))
    s = 0.3 * math.sqrt(dx)
    z = Coef.const(0.0)
    sig = ((Coef.const(s), Coef.const(0.3 * s)), (Coef.const(-0.2 * s), Coef.const(s)))
    return make_instance(f"random{n}-{seed}", n, lo, hi, n_a=n_a, lam=lam, speed=speed,
                         drift=drift, p=p, sigma=sig, kind=kind)


def reach_cells(inst: Instance) -> float:
    """Upper bound on |foot - x_i| in cells: (h max|f| + s max|sigma_k|)/dx (reading R4)."""
    amax = float(np.max(np.hypot(inst.controls[:, 0], inst.controls[:, 1])))
    fmax = inst.speed.max_abs() * amax + math.hypot(inst.drift[0].max_abs(), inst.drift[1].max_abs())
    if inst.p == 0:
        smax = 0.0
    else:
        sc = math.sqrt(inst.h * inst.p) if inst.diffusion_scale == 0 else math.sqrt(inst.h)
        if inst.sigma_mode == 1:
            smax = sc * inst.sigma[0][0].max_abs() * amax
        else:
            smax = sc * max(math.hypot(inst.sigma[k][0].max_abs(), inst.sigma[k][1].max_abs())
                            for k in range(inst.p))
    return (inst.h * fmax + smax) / inst.dx
