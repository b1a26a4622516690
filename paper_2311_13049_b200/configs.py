"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference has no public dataset; these generators pin every input the
configs leave open and are shared by the tests, the golden
fixture script and bench.py, so every checker sees identical arrays.  Each takes
a size so reduced-size parity cases use the same construction.

  C1  1D [-32,32), N=4096, u0=exp(-x^2), Q=20+80(1+tanh(x/2))/2, M=8, tau=1e-3, 100 steps
  C2  2D [-16,16)^2, 1024^2, u0=exp(-(x^2+y^2)/0.5), Q two-layer along y (20 for y>0,
      100 for y<0, tanh width 1), M=16, tau=5e-4, 200 steps
  C3  3D [-8,8)^3, 256^3, Ricker(nu0=2) at the origin (the reference's initial Ricker pulse,
      seismic.cpp:70-83; it has no time-dependent source), Q=10+190*sigmoid(g),
      g = 32 random Fourier modes (|k_i|_inf <= 4, a_i~N(0,1), phase~U[0,2pi)) drawn from
      numpy PCG64 seed 0, M=16, tau=1e-3, 100 steps
  C4  3D [-16,16)^3, 512^3, u0=exp(-r^2/0.5), Q = 15/60/200 layers along z (axis 2) with
      tanh transitions of width 1 at z=-16/3, +16/3, blended with a Q=8 sphere of radius 3
      at the origin by b=(1-tanh(r-3))/2, M=32, tau=5e-4, 50 steps
  C5  64 fields on [-16,16)^2, 512^2: u = periodic Gaussian filter (sigma = 4 cells) of N(0,1),
      s = 1 + 0.45 g/max|g| with g = 16 random modes (|k|_inf <= 4), field f seeded PCG64(f);
      M in {4, 8, 16, 32, 64}; apply only
All media: c0 = 1, omega0 = 1, gamma = arctan(1/Q)/pi.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


def gamma_from_q(Q):
    return np.arctan(1.0 / Q) / np.pi


def _coords(lo, hi, J):
    return [lo[m] + np.arange(J[m]) * ((hi[m] - lo[m]) / J[m]) for m in range(len(J))]


def _mesh(lo, hi, J):
    return np.meshgrid(*_coords(lo, hi, J), indexing="ij")


@dataclass
class SeismicConfig:
    name: str
    lo: tuple
    hi: tuple
    J: tuple
    M: int
    tau: float
    steps: int
    phi: np.ndarray
    gamma: np.ndarray
    c0: np.ndarray
    omega0: float = 1.0
    psi: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.psi is None:
            self.psi = np.zeros(self.J)

    @property
    def N(self):
        return int(np.prod(self.J))

    @property
    def N_half(self):
        return int(np.prod(self.J[:-1])) * (self.J[-1] // 2 + 1)


def c1(n: int = 4096) -> SeismicConfig:
    lo, hi, J = (-32.0,), (32.0,), (n,)
    (x,) = _coords(lo, hi, J)
    Q = 20.0 + 80.0 * (1.0 + np.tanh(x / 2.0)) / 2.0
    return SeismicConfig("C1", lo, hi, J, 8, 1e-3, 100, np.exp(-x**2), gamma_from_q(Q), np.ones(J))


def c2(n: int = 1024) -> SeismicConfig:
    lo, hi, J = (-16.0, -16.0), (16.0, 16.0), (n, n)
    X, Y = _mesh(lo, hi, J)
    Q = 100.0 + (20.0 - 100.0) * (1.0 + np.tanh(Y / 1.0)) / 2.0
    return SeismicConfig("C2", lo, hi, J, 16, 5e-4, 200, np.exp(-(X**2 + Y**2) / 0.5), gamma_from_q(Q),
                         np.ones(J))


def random_modes(rng, nmodes, kmax, d):
    ks = []
    while len(ks) < nmodes:
        k = rng.integers(-kmax, kmax + 1, size=d)
        if np.any(k != 0):
            ks.append(k)
    amps = rng.standard_normal(nmodes)
    phases = rng.uniform(0.0, 2.0 * np.pi, size=nmodes)
    return np.array(ks), amps, phases


def mode_sum(lo, hi, J, ks, amps, phases):
    Xs = _mesh(lo, hi, J)
    g = np.zeros(J)
    for k, a, ph in zip(ks, amps, phases):
        arg = np.zeros(J)
        for m in range(len(J)):
            arg = arg + 2.0 * np.pi * k[m] * (Xs[m] - lo[m]) / (hi[m] - lo[m])
        g += a * np.cos(arg + ph)
    return g


def ricker(lo, hi, J, nu0, xc):
    """ricker_initial (seismic.cpp:70-83)."""
    Xs = _mesh(lo, hi, J)
    a = np.pi * np.pi * nu0 * nu0
    r2 = np.zeros(J)
    for m in range(len(J)):
        r2 = r2 + (Xs[m] - xc[m]) ** 2
    return (1.0 - 2.0 * a * r2) * np.exp(-a * r2)


def c3(n: int = 256, L: float = 8.0) -> SeismicConfig:
    lo, hi, J = (-L,) * 3, (L,) * 3, (n,) * 3
    rng = np.random.default_rng(0)
    ks, amps, phases = random_modes(rng, 32, 4, 3)
    g = mode_sum(lo, hi, J, ks, amps, phases)
    Q = 10.0 + 190.0 / (1.0 + np.exp(-g))
    return SeismicConfig("C3", lo, hi, J, 16, 1e-3, 100, ricker(lo, hi, J, 2.0, (0.0, 0.0, 0.0)),
                         gamma_from_q(Q), np.ones(J))


def c4(n: int = 512, L: float = 16.0) -> SeismicConfig:
    lo, hi, J = (-L,) * 3, (L,) * 3, (n,) * 3
    X, Y, Z = _mesh(lo, hi, J)
    r = np.sqrt(X**2 + Y**2 + Z**2)
    zb = L / 3.0
    Ql = 15.0 + (60.0 - 15.0) * 0.5 * (1.0 + np.tanh((Z + zb) / 1.0)) + (200.0 - 60.0) * 0.5 * (
        1.0 + np.tanh((Z - zb) / 1.0))
    b = 0.5 * (1.0 - np.tanh((r - 3.0) / 1.0))
    Q = Ql * (1.0 - b) + 8.0 * b
    return SeismicConfig("C4", lo, hi, J, 32, 5e-4, 50, np.exp(-r**2 / 0.5), gamma_from_q(Q), np.ones(J))


@dataclass
class ApplyField:
    lo: tuple
    hi: tuple
    J: tuple
    u: np.ndarray
    s: np.ndarray


def c5_field(f: int, n: int = 512, sigma_cells: float = 4.0) -> ApplyField:
    lo, hi, J = (-16.0, -16.0), (16.0, 16.0), (n, n)
    rng = np.random.default_rng(f)
    w = rng.standard_normal(J)
    k0 = np.fft.fftfreq(n)  # cycles per cell
    K2 = k0[:, None] ** 2 + k0[None, :] ** 2
    u = np.real(np.fft.ifft2(np.fft.fft2(w) * np.exp(-2.0 * np.pi**2 * sigma_cells**2 * K2)))
    ks, amps, phases = random_modes(rng, 16, 4, 2)
    g = mode_sum(lo, hi, J, ks, amps, phases)
    s = 1.0 + 0.45 * g / np.max(np.abs(g))
    return ApplyField(lo, hi, J, np.ascontiguousarray(u), np.ascontiguousarray(s))


C5_M = (4, 8, 16, 32, 64)
C5_FIELDS = 64


def s1_profile(lo, hi, J):
    """1 + 0.3 sin(pi x / 8) (test_flap.cpp:20-25)."""
    X = _mesh(lo, hi, J)[0]
    return 1.0 + 0.3 * np.sin(np.pi * X / 8.0)


def orders(cfg: SeismicConfig):
    """Orders of the two seismic operators (seismic.cpp:37-38)."""
    return 1.0 + cfg.gamma, 0.5 + cfg.gamma


def bytes_per_apply(N: int, N_half: int, M: int, table_model: bool = True) -> int:
    """Algorithmic HBM bytes of one apply (SURVEY.md §8(d) table-streaming model):
    8N (u) + 8N (Lu) + 8MN ((s-s0)^m) + 8(M+1)N_h (w_m).  With on-chip regeneration of
    the deviation powers (dev_m = dev_{m-1} dev_1, bit-identical) the 8MN term becomes 8N."""
    dev = 8 * M * N if table_model else 8 * N
    return 8 * N + 8 * N + dev + 8 * (M + 1) * N_half


def bytes_per_apply_pass_model(N: int, N_half: int, M: int, table_model: bool = True) -> int:
    """SURVEY.md §8(d) 3D pass model (one plane pass + transpose + one pencil pass per
    transform, intermediates in HBM): 8N + 3*16 N_h + (M+1)(16+8+16+16) N_h + 8MN + 8N;
    the 8MN deviation-table term becomes 8N when the powers are regenerated on chip."""
    dev = 8 * M * N if table_model else 8 * N
    return 8 * N + 3 * 16 * N_half + (M + 1) * (16 + 8 + 16 + 16) * N_half + dev + 8 * N


def bytes_per_seismic_step(N: int, N_half: int, M: int, table_model: bool = True) -> int:
    """B_step = 2 B_apply - 8N + 72N (shared forward transform, update
    reading cur, prev, L1, L2, L2prev, c, eta, tau_c and writing next)."""
    return 2 * bytes_per_apply(N, N_half, M, table_model) - 8 * N + 72 * N
