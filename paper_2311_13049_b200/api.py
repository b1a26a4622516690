"""Reference-shaped host API over the C-ABI (see package docstring).

Names, argument meaning and error behaviour follow fracwave's C++ API:
Grid (grid.hpp:20-59), OrderField (orderfield.hpp:13-29), build_expansion /
apply_matrix_free / apply_perturbation (flap.hpp:14-41), SeismicMedium /
build_medium / SeismicStepper (seismic.hpp:13-55), Stepper TSFP2
(stepping.hpp:72-104).  Fields are numpy float64 arrays of the grid's shape
(row-major, axis 0 slowest, as the reference's Field).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ArgumentError, DimOutOfRange, EmptyInterval, GridMismatch, OddSize, check, load_library

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a, n: Optional[int] = None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and a.size != n:
        raise GridMismatch(f"field length {a.size} does not match grid point count {n}")
    return a


class Context:
    """One CUDA device + stream (fw_ctx)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        check(lib.fw_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def sync(self):
        check(load_library().fw_ctx_sync(self._h))

    @property
    def stream(self) -> int:
        return int(load_library().fw_ctx_stream(self._h) or 0)

    def launches(self) -> int:
        return int(load_library().fw_ctx_launches(self._h))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_ctx_destroy(self._h)
                self._h = None
        except Exception:
            pass


_default: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


class Grid:
    """Periodic tensor-product grid (grid.cpp:35-58 validation)."""

    def __init__(self, bounds: Sequence[Sequence[float]], sizes: Sequence[int]):
        if len(bounds) != len(sizes):
            raise DimOutOfRange("bounds and sizes length mismatch")
        d = len(bounds)
        if d < 1 or d > 3:
            raise DimOutOfRange(f"dimension must be 1, 2 or 3, got {d}")
        for m, (J, (a, b)) in enumerate(zip(sizes, bounds)):
            if J < 4 or J % 2 != 0:
                raise OddSize(f"axis {m}: point count {J} must be even and >= 4")
            if not (b > a):
                raise EmptyInterval(f"axis {m}: empty interval")
        self.dim = d
        self.sizes = tuple(int(J) for J in sizes)
        self.lo = tuple(float(a) for a, _ in bounds)
        self.hi = tuple(float(b) for _, b in bounds)

    @property
    def shape(self):
        return self.sizes

    def total(self) -> int:
        return int(np.prod(self.sizes))

    def size(self, axis: int) -> int:
        return self.sizes[axis]

    def step(self, axis: int) -> float:
        return (self.hi[axis] - self.lo[axis]) / self.sizes[axis]

    def same_as(self, other: "Grid") -> bool:
        return self.sizes == other.sizes and self.lo == other.lo and self.hi == other.hi

    def coords(self):
        """Per-axis coordinate vectors a + j h (Grid::point, grid.cpp:107-116)."""
        return [self.lo[m] + np.arange(self.sizes[m]) * self.step(m) for m in range(self.dim)]

    def mesh(self):
        return np.meshgrid(*self.coords(), indexing="ij")

    def _carrays(self):
        J = (C.c_int * 3)(*(list(self.sizes) + [1] * (3 - self.dim)))
        lo = (C.c_double * 3)(*(list(self.lo) + [0.0] * (3 - self.dim)))
        hi = (C.c_double * 3)(*(list(self.hi) + [1.0] * (3 - self.dim)))
        return J, lo, hi


def build_grid(bounds, sizes) -> Grid:
    return Grid(bounds, sizes)


class OrderField:
    """Sampled s(x) with optional s0 override.  Validation (range, deviation) is
    performed when the operator is built, exactly as orderfield.cpp:10-36."""

    def __init__(self, grid: Grid, values, s0_override: Optional[float] = None):
        self.grid = grid
        self.values = _f64(values, grid.total()).reshape(grid.shape)
        self.s0_override = s0_override


class ExpansionOperator:
    """Device-resident M-term operator (fw_op)."""

    def __init__(self, handle, grid: Grid, ctx: Context, order: Optional[OrderField] = None):
        self._h = handle
        self.grid = grid
        self.ctx = ctx
        self.order = order
        info = _capi.OpInfo()
        check(load_library().fw_op_info(handle, C.byref(info)))
        self.M = info.M
        self.constant_order = bool(info.constant_order)
        self.s0 = info.s0
        self.smin, self.smax = info.smin, info.smax
        self.N, self.N_half = info.N, info.N_half
        self.device_bytes = info.device_bytes
        self.slab = None  # (P, rank) for build_slab_expansion operators

    @property
    def handle(self):
        return self._h

    @property
    def persistent(self) -> bool:
        """True when applies run on the single-launch persistent 2D kernel (fw_op_path)."""
        return load_library().fw_op_path(self._h) == 1

    @classmethod
    def from_tables(cls, grid: Grid, M: int, s0: float, constant_order: bool, base_symbol,
                    log_weights, deviation_powers, ctx: Optional[Context] = None):
        """Upload a host ExpansionOperator's tables (flap.hpp:14-22)."""
        ctx = ctx or default_context()
        N = grid.total()
        base = _f64(base_symbol, N)
        lw = [_f64(r, N) for r in log_weights]
        dv = [_f64(r, N) for r in deviation_powers]
        lwp = (_dp * max(M, 1))(*[_ptr(r) for r in lw])
        dvp = (_dp * max(M, 1))(*[_ptr(r) for r in dv])
        J, lo, hi = grid._carrays()
        h = C.c_void_p()
        check(load_library().fw_op_create_from_tables(ctx.handle, grid.dim, J, lo, hi, int(M), float(s0),
                                                      int(bool(constant_order)), _ptr(base), lwp, dvp,
                                                      C.byref(h)))
        return cls(h, grid, ctx)

    def apply(self, u, m_first: int = 0, residue: bool = False):
        u = _f64(u, self.N)
        out = np.empty(self.grid.shape, dtype=np.float64)
        res = C.c_double(0.0)
        check(load_library().fw_apply(self._h, _ptr(u), _ptr(out), int(m_first),
                                      C.byref(res) if residue else None))
        return (out, res.value) if residue else out

    def apply_device(self, u_ptr: int, out_ptr: int, m_first: int = 0, residue_ptr: int = 0):
        """Device pointers (e.g. torch.Tensor.data_ptr()), enqueued on the context stream."""
        check(load_library().fw_apply_device(self._h, C.c_void_p(u_ptr), C.c_void_p(out_ptr), int(m_first),
                                             C.c_void_p(residue_ptr) if residue_ptr else None))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_op_destroy(self._h)
                self._h = None
        except Exception:
            pass


def build_expansion(order: OrderField, M: int, ctx: Optional[Context] = None) -> ExpansionOperator:
    """build_expansion (flap.cpp:96-135): NegativeM / OrderOutOfRange / DeviationTooLarge."""
    ctx = ctx or default_context()
    g = order.grid
    J, lo, hi = g._carrays()
    s0 = C.c_double(order.s0_override) if order.s0_override is not None else None
    h = C.c_void_p()
    check(load_library().fw_op_create(ctx.handle, g.dim, J, lo, hi, _ptr(order.values),
                                      C.byref(s0) if s0 is not None else None, int(M), C.byref(h)))
    return ExpansionOperator(h, g, ctx, order)


def build_slab_expansion(order: OrderField, M: int, P: int, rank: int,
                         ctx: Optional[Context] = None) -> ExpansionOperator:
    """One rank's tables of a slab-decomposed 3D operator (fw_op_create_slab): w_m on the rank's
    spectral columns, s - s0 on its planes; s0 and validation from the global order values."""
    ctx = ctx or default_context()
    g = order.grid
    if g.dim != 3:
        raise ArgumentError("slab decomposition is three-dimensional")
    J, lo, hi = g._carrays()
    s0 = C.c_double(order.s0_override) if order.s0_override is not None else None
    h = C.c_void_p()
    check(load_library().fw_op_create_slab(ctx.handle, J, lo, hi, _ptr(order.values),
                                           C.byref(s0) if s0 is not None else None, int(M), int(P), int(rank),
                                           C.byref(h)))
    op = ExpansionOperator(h, g, ctx, order)
    op.slab = (int(P), int(rank))
    return op


def nccl_unique_id() -> bytes:
    """An NCCL unique id for SlabSeismicStepperC (made on rank 0, handed to every rank by the host)."""
    buf = C.create_string_buffer(128)
    check(load_library().fw_nccl_unique_id(buf))
    return buf.raw


class SlabSeismicStepperC:
    """The slab-decomposed SeismicStepper of the C-ABI (fw_slab_seis_*: the stepping logic in C++,
    one process per GPU, NCCL-bootstrapped IPC transposes, stream-ordered barriers) -- what a C/C++
    host of the reference drives; gamma, c0, phi, psi are the GLOBAL fields."""

    def __init__(self, grid: Grid, gamma, c0, omega0: float, M: int, phi, psi, tau: float, P: int = 1,
                 rank: int = 0, nccl_id: Optional[bytes] = None, blowup_factor: float = 1e8,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.grid, self.P, self.rank = grid, int(P), int(rank)
        N = grid.total()
        J, lo, hi = grid._carrays()
        self._keep = [_f64(a, N) for a in (gamma, c0, phi, psi)]
        h = C.c_void_p()
        check(load_library().fw_slab_seis_create(self.ctx.handle, nccl_id, int(P), int(rank), J, lo, hi,
                                                 *[_ptr(a) for a in self._keep[:2]], float(omega0), int(M),
                                                 *[_ptr(a) for a in self._keep[2:]], float(tau),
                                                 float(blowup_factor), C.byref(h)))
        self._h = h
        self.slab_shape = (grid.sizes[0] // self.P,) + tuple(grid.sizes[1:])

    def advance(self, steps: int):
        check(load_library().fw_slab_seis_step(self._h, int(steps)))

    def step(self):
        self.advance(1)

    def state(self):
        """(cur, prev, L2prev) of this rank's planes and n."""
        cur, prev, ap = (np.empty(self.slab_shape) for _ in range(3))
        n = C.c_long(0)
        check(load_library().fw_slab_seis_get(self._h, _ptr(cur), _ptr(prev), _ptr(ap), C.byref(n)))
        return cur, prev, ap, n.value

    def n(self) -> int:
        n = C.c_long(0)
        check(load_library().fw_slab_seis_get(self._h, None, None, None, C.byref(n)))
        return n.value

    @property
    def table_bytes(self) -> int:
        b = C.c_size_t(0)
        check(load_library().fw_slab_seis_info(self._h, C.byref(b), None, None))
        return b.value

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_slab_seis_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _check_field(op: ExpansionOperator, u):
    if hasattr(u, "grid") and not u.grid.same_as(op.grid):
        raise GridMismatch("field defined on a different grid than the operator")
    arr = np.asarray(u, dtype=np.float64)
    if arr.size != op.N:
        raise GridMismatch("field defined on a different grid than the operator")
    return arr


def apply_matrix_free(op: ExpansionOperator, u, residue: bool = False):
    """flap.cpp:151-154 — returns L u (and the imaginary residue when asked)."""
    return op.apply(_check_field(op, u), 0, residue)


def apply_matrix_free_serial(op: ExpansionOperator, u, residue: bool = False):
    """flap.cpp:156-159 — the device reduction order is fixed (ascending m), so the
    serial and parallel entry points are the same computation."""
    return op.apply(_check_field(op, u), 0, residue)


def apply_perturbation(op: ExpansionOperator, u, residue: bool = False):
    """flap.cpp:161-168 — terms m = 1..M (exact zeros for a constant order)."""
    return op.apply(_check_field(op, u), 1, residue)



def apply_batch_device(ops, u_ptrs, out_ptrs):
    """``apply_matrix_free`` of many independent fields at once (configs[4]: 64 fields
    of one grid, each with its own order field).  Device pointers; enqueued on the
    operators' (common) context stream.  Fields sharing grid and M run as ONE batched
    pipeline (one launch per stage for all fields, fw_apply_batch_device)."""
    n = len(ops)
    if len(u_ptrs) != n or len(out_ptrs) != n:
        raise ValueError("ops, u_ptrs and out_ptrs must have the same length")
    H = C.c_void_p * max(n, 1)
    check(load_library().fw_apply_batch_device(H(*[o._h for o in ops]), n, H(*[C.c_void_p(p) for p in u_ptrs]),
                                               H(*[C.c_void_p(p) for p in out_ptrs])))


def apply_batch(ops, fields):
    """Host-buffer variant of :func:`apply_batch_device`: returns the list of results."""
    import torch

    us = [torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda() for f in fields]
    outs = [torch.empty_like(u) for u in us]
    apply_batch_device(ops, [u.data_ptr() for u in us], [o.data_ptr() for o in outs])
    if ops:
        ops[0].ctx.sync()
    return [o.cpu().numpy() for o in outs]

class SeismicMedium:
    """Inputs of derive_medium (seismic.cpp:11-44); the coefficient fields and the
    two operators are built on the device by SeismicStepper."""

    def __init__(self, grid: Grid, gamma, c0, omega0: float, M: int):
        self.grid = grid
        self.gamma = _f64(gamma, grid.total()).reshape(grid.shape)
        c0 = np.broadcast_to(np.asarray(c0, dtype=np.float64), grid.shape)
        self.c0 = np.ascontiguousarray(c0)
        self.omega0 = float(omega0)
        self.M = int(M)
        bad = ~((self.gamma >= 0.0) & (self.gamma < 0.5))
        if bad.any():
            from ._capi import GammaOutOfRange
            raise GammaOutOfRange(f"gamma = {self.gamma[bad].flat[0]} outside [0, 0.5)")


def ricker_initial(nu0: float, xc, grid: Grid) -> np.ndarray:
    """ricker_initial (seismic.cpp:70-83): (1 - 2 a r^2) exp(-a r^2), a = pi^2 nu0^2, on the
    reference's grid points (grid.cpp:107-116); bit-identical to the reference (fw_ricker_initial)."""
    xc = _f64(xc)
    if xc.size < grid.dim:
        raise ArgumentError("xc needs one coordinate per grid axis")
    J, lo, hi = grid._carrays()
    out = np.empty(grid.shape)
    check(load_library().fw_ricker_initial(grid.dim, J, lo, hi, float(nu0), _ptr(xc), _ptr(out)))
    return out


def build_medium(grid: Grid, gamma, c0, omega0: float, M: int) -> SeismicMedium:
    return SeismicMedium(grid, gamma, c0, omega0, M)


class SeismicStepper:
    """Explicit two-level viscoacoustic stepper (seismic.cpp:85-142), state resident
    on the device, both operator applies and the update fused per step."""

    def __init__(self, medium: SeismicMedium, phi, psi, tau: float, blowup_factor: float = 1e8,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.medium = medium
        g = medium.grid
        self.grid = g
        N = g.total()
        phi = _f64(phi, N)
        psi = _f64(psi, N)
        J, lo, hi = g._carrays()
        h = C.c_void_p()
        check(load_library().fw_seis_create(self.ctx.handle, g.dim, J, lo, hi, _ptr(medium.gamma),
                                            _ptr(medium.c0), medium.omega0, medium.M, _ptr(phi), _ptr(psi),
                                            float(tau), float(blowup_factor), C.byref(h)))
        self._h = h
        self.tau = float(tau)

    def step(self):
        check(load_library().fw_seis_step(self._h, 1))

    def advance(self, steps: int):
        check(load_library().fw_seis_step(self._h, int(steps)))

    def enqueue(self, steps: int):
        check(load_library().fw_seis_enqueue(self._h, int(steps)))

    def advance_to(self, t_final: float):
        target = int(round(t_final / self.tau))  # std::lround (seismic.cpp:140)
        k = target - self.n()
        if k > 0:
            self.advance(k)

    def current(self):
        out = np.empty(self.grid.shape)
        check(load_library().fw_seis_get(self._h, _ptr(out), None, None, None))
        return out

    def state(self):
        """(cur, prev, atten_prev, n)"""
        cur, prev, ap = (np.empty(self.grid.shape) for _ in range(3))
        n = C.c_long(0)
        check(load_library().fw_seis_get(self._h, _ptr(cur), _ptr(prev), _ptr(ap), C.byref(n)))
        return cur, prev, ap, n.value

    def set_current(self, cur):
        cur = _f64(cur, self.grid.total())
        check(load_library().fw_seis_set_current(self._h, _ptr(cur)))

    def step_io(self, cur_in=None, cur_out=None, steps: int = 1):
        """Host-owned wavefield exchange in one call (fw_seis_step_io): the current field is
        overwritten from cur_in (if given), `steps` steps run, the new current field lands in
        cur_out (a float64 array of the grid's size, if given).  BlowupDetected as step()."""
        pin = None if cur_in is None else _f64(cur_in, self.grid.total())
        if cur_out is not None and (cur_out.dtype != np.float64 or not cur_out.flags.c_contiguous
                                    or cur_out.size != self.grid.total()):
            raise ValueError("cur_out must be a C-contiguous float64 array of the grid's size")
        check(load_library().fw_seis_step_io(self._h, None if pin is None else _ptr(pin), int(steps),
                                             None if cur_out is None else _ptr(cur_out)))
        return cur_out

    def step_io_async(self, cur_in=None, cur_out=None, steps: int = 1):
        """The enqueue half of step_io (fw_seis_step_io_async): upload, `steps` steps and download
        go onto this stepper's context stream and the call returns at once; `wait()` completes
        it.  Both arrays must be C-contiguous float64 of the grid's size and stay alive (pinned
        for overlap) until wait().  Steppers on different contexts overlap each other."""
        for a in (cur_in, cur_out):
            if a is not None and (a.dtype != np.float64 or not a.flags.c_contiguous
                                  or a.size != self.grid.total()):
                raise ValueError("host fields must be C-contiguous float64 arrays of the grid's size")
        check(load_library().fw_seis_step_io_async(self._h, None if cur_in is None else _ptr(cur_in), int(steps),
                                                   None if cur_out is None else _ptr(cur_out)))

    def wait(self):
        """Completes step_io_async (fw_seis_wait): one host synchronisation and the blow-up
        check; BlowupDetected as step(), with the pending cur_out holding the pre-step state."""
        check(load_library().fw_seis_wait(self._h))

    def n(self) -> int:
        n = C.c_long(0)
        check(load_library().fw_seis_get(self._h, None, None, None, C.byref(n)))
        return n.value

    def time(self) -> float:
        return self.n() * self.tau

    def coefficients(self):
        c, eta, tc = (np.empty(self.grid.shape) for _ in range(3))
        check(load_library().fw_seis_medium(self._h, _ptr(c), _ptr(eta), _ptr(tc)))
        return c, eta, tc

    @property
    def persistent(self) -> bool:
        """True when every step runs on the single-launch persistent 2D kernel."""
        d, a = C.c_void_p(), C.c_void_p()
        check(load_library().fw_seis_ops(self._h, C.byref(d), C.byref(a)))
        return load_library().fw_op_path(d) == 1 and load_library().fw_op_path(a) == 1

    def operators(self):
        d, a = C.c_void_p(), C.c_void_p()
        check(load_library().fw_seis_ops(self._h, C.byref(d), C.byref(a)))
        info = []
        for h in (d, a):
            i = _capi.OpInfo()
            check(load_library().fw_op_info(h, C.byref(i)))
            info.append(i)
        return info

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_seis_destroy(self._h)
                self._h = None
        except Exception:
            pass


class TSFP2Stepper:
    """Strang time splitting (stepping.cpp:119-138, 266-304) for
    u_tt = -kappa (-Delta)^{s(x)} u + f(u), f in {none, cubic}."""

    def __init__(self, order: OrderField, M: int, kappa: float, phi, psi, tau: float, f: str = "none",
                 ctx: Optional[Context] = None, blowup_factor: float = 1e8):
        self.ctx = ctx or default_context()
        g = order.grid
        self.grid = g
        N = g.total()
        J, lo, hi = g._carrays()
        h = C.c_void_p()
        check(load_library().fw_tsfp2_create(self.ctx.handle, g.dim, J, lo, hi, _ptr(order.values), int(M),
                                             float(kappa), 1 if f == "cubic" else 0, _ptr(_f64(phi, N)),
                                             _ptr(_f64(psi, N)), float(tau), float(blowup_factor), C.byref(h)))
        self._h = h
        self.tau = float(tau)

    def advance(self, steps: int):
        check(load_library().fw_tsfp2_step(self._h, int(steps)))

    def step(self):
        self.advance(1)

    def current(self):
        return self.state()[0]

    def velocity(self):
        return self.state()[1]

    def state(self):
        u, v = np.empty(self.grid.shape), np.empty(self.grid.shape)
        check(load_library().fw_tsfp2_get(self._h, _ptr(u), _ptr(v), None))
        return u, v

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_tsfp2_destroy(self._h)
                self._h = None
        except Exception:
            pass


@dataclass
class WaveProblem:
    """u_tt = -kappa (-Delta)^{s(x)} u + f(u) (stepping.hpp:30-37); f in {"none", "cubic"}
    (the reference's expression-valued f is out of scope)."""
    order: OrderField
    phi: object
    psi: object
    kappa: float = 1.0
    f: str = "none"
    M: int = 15


@dataclass
class StepperConfig:
    """stepping.hpp:39-48 (use_dense is not offered: the dense operator is out of scope)."""
    method: str = "TSFP2"  # "LFFP", "CNFP" or "TSFP2"
    tau: float = 1e-3
    picard_tol: float = 1e-12
    picard_max_iters: int = 200
    inner_cg_tol: float = 1e-14
    cg_max_iters: int = 500
    blowup_factor: float = 1e8


class Stepper:
    """The reference's Stepper (stepping.hpp:72-104) with the Laplacian seam served by
    the device apply.  LFFP / CNFP keep both levels, and CNFP every Picard / CG vector,
    on the device (fw_wave_*); TSFP2 delegates to TSFP2Stepper (fw_tsfp2_*).  LFFP and
    TSFP2 are bit-identical to the reference; CNFP agrees to the CG tolerance (its
    dot products are deterministic tree sums, not the reference's serial sums)."""

    _METHODS = {"LFFP": 0, "CNFP": 1}

    def __init__(self, problem: WaveProblem, config: StepperConfig, ctx: Optional[Context] = None):
        if problem.f not in ("none", "cubic"):
            raise ArgumentError(f"f must be 'none' or 'cubic', not {problem.f!r}")
        self.ctx = ctx or default_context()
        self.config = config
        g = problem.order.grid
        self.grid = g
        self.method = config.method.upper()
        if self.method == "TSFP2":
            self._ts = TSFP2Stepper(problem.order, problem.M, problem.kappa, problem.phi, problem.psi, config.tau,
                                    f=problem.f, ctx=self.ctx, blowup_factor=config.blowup_factor)
            return
        if self.method not in self._METHODS:
            raise ArgumentError(f"unknown method {config.method!r}")
        self._ts = None
        N = g.total()
        J, lo, hi = g._carrays()
        h = C.c_void_p()
        check(load_library().fw_wave_create(
            self.ctx.handle, self._METHODS[self.method], g.dim, J, lo, hi, _ptr(problem.order.values),
            int(problem.M), float(problem.kappa), 1 if problem.f == "cubic" else 0, _ptr(_f64(problem.phi, N)),
            _ptr(_f64(problem.psi, N)), float(config.tau), float(config.picard_tol), int(config.picard_max_iters),
            float(config.inner_cg_tol), int(config.cg_max_iters), float(config.blowup_factor), C.byref(h)))
        self._h = h

    def advance(self, steps: int):
        if self._ts is not None:
            self._ts.advance(steps)
            return
        check(load_library().fw_wave_step(self._h, int(steps)))

    def step(self):
        self.advance(1)

    def advance_to(self, t_final: float):
        target = int(round(t_final / self.config.tau))  # std::lround (stepping.cpp:165-168)
        if target > self.n():
            self.advance(target - self.n())

    def _get(self):
        cur, prev = np.empty(self.grid.shape), np.empty(self.grid.shape)
        n, pt = C.c_long(), C.c_long()
        check(load_library().fw_wave_get(self._h, _ptr(cur), _ptr(prev), C.byref(n), C.byref(pt)))
        return cur, prev, n.value, pt.value

    def current(self):
        return self._ts.current() if self._ts is not None else self._get()[0]

    def previous(self):
        """u^{n-1} (two-level methods)."""
        return self._get()[1]

    def velocity(self):
        if self._ts is None:
            raise ArgumentError("velocity() is TSFP2 only")
        return self._ts.velocity()

    def n(self) -> int:
        n, pt = C.c_long(), C.c_long()
        if self._ts is not None:
            check(load_library().fw_tsfp2_get(self._ts._h, None, None, C.byref(n)))
        else:
            check(load_library().fw_wave_get(self._h, None, None, C.byref(n), C.byref(pt)))
        return n.value

    def time(self) -> float:
        return self.n() * self.config.tau

    def total_picard_iterations(self) -> int:
        if self._ts is not None:
            return 0
        n, pt = C.c_long(), C.c_long()
        check(load_library().fw_wave_get(self._h, None, None, C.byref(n), C.byref(pt)))
        return pt.value

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_wave_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _cplx(a, n: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if a.size != n:
        raise GridMismatch("spectrum length does not match grid point count")
    return a


def grid_dft(grid: Grid, data, sign: int, ctx: Optional[Context] = None) -> np.ndarray:
    """Grid::dft (grid.cpp:134-137): unnormalised C2C of a complex array on the grid's shape,
    sign -1 (FFTW_FORWARD) / +1 (FFTW_BACKWARD); returns the transformed array (the input is
    not modified)."""
    ctx = ctx or default_context()
    x = _cplx(data, grid.total()).reshape(grid.shape).copy()
    J, _, _ = grid._carrays()
    check(load_library().fw_grid_dft(ctx.handle, grid.dim, J, x.view(np.float64).ctypes.data_as(_dp), int(sign)))
    return x


def forward(grid: Grid, u, ctx: Optional[Context] = None) -> np.ndarray:
    """Grid::forward (grid.cpp:171-179): the full spectrum DFT(u) / N."""
    ctx = ctx or default_context()
    u = _f64(u, grid.total())
    spec = np.empty(grid.shape, dtype=np.complex128)
    J, _, _ = grid._carrays()
    check(load_library().fw_grid_forward(ctx.handle, grid.dim, J, _ptr(u), spec.view(np.float64).ctypes.data_as(_dp)))
    return spec


def inverse(grid: Grid, spec, residue: bool = False, ctx: Optional[Context] = None):
    """Grid::inverse (grid.cpp:181-197): Re IDFT(spec) [and max |Im|]."""
    ctx = ctx or default_context()
    sp = _cplx(spec, grid.total())
    out = np.empty(grid.shape)
    res = C.c_double(0.0)
    J, _, _ = grid._carrays()
    check(load_library().fw_grid_inverse(ctx.handle, grid.dim, J, sp.view(np.float64).ctypes.data_as(_dp), _ptr(out),
                                         C.byref(res)))
    return (out, res.value) if residue else out


def apply_constant_order(grid: Grid, u, s: float, residue: bool = False, ctx: Optional[Context] = None):
    """apply_constant_order (flap.cpp:137-149): (-Delta)^s of a real field (returns a field) or of a
    full complex spectrum (returns the spectrum times |mu|^{2s}); s in (0, 2) else OrderOutOfRange."""
    ctx = ctx or default_context()
    J, lo, hi = grid._carrays()
    if np.iscomplexobj(u):
        sp = _cplx(u, grid.total())
        out = np.empty(grid.shape, dtype=np.complex128)
        check(load_library().fw_apply_constant_order_spectrum(ctx.handle, grid.dim, J, lo, hi,
                                                              sp.view(np.float64).ctypes.data_as(_dp), float(s),
                                                              out.view(np.float64).ctypes.data_as(_dp)))
        return out
    uu = _f64(u, grid.total())
    out = np.empty(grid.shape)
    res = C.c_double(0.0)
    check(load_library().fw_apply_constant_order(ctx.handle, grid.dim, J, lo, hi, _ptr(uu), float(s), _ptr(out),
                                                 C.byref(res)))
    return (out, res.value) if residue else out


DEFAULT_MEMORY_BUDGET = 8 << 30  # kDefaultMemoryBudget (flap.hpp:48)


class DenseOperator:
    """assemble_dense (flap.cpp:170-230): the N x N spatial matrix of (-Delta)^{s(x)}, assembled and
    kept on the device (fw_dense_*); the reference's verification oracle."""

    def __init__(self, order: OrderField, memory_budget: int = DEFAULT_MEMORY_BUDGET, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.grid, self.order = order.grid, order
        J, lo, hi = order.grid._carrays()
        h = C.c_void_p()
        check(load_library().fw_dense_create(self.ctx.handle, order.grid.dim, J, lo, hi, _ptr(order.values),
                                             int(memory_budget), C.byref(h)))
        self._h = h

    @property
    def entries(self) -> np.ndarray:
        N = self.grid.total()
        a = np.empty((N, N))
        check(load_library().fw_dense_entries(self._h, _ptr(a)))
        return a

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().fw_dense_destroy(self._h)
                self._h = None
        except Exception:
            pass


def assemble_dense(order: OrderField, memory_budget: int = DEFAULT_MEMORY_BUDGET,
                   ctx: Optional[Context] = None) -> DenseOperator:
    return DenseOperator(order, memory_budget, ctx)


def apply_dense(op: DenseOperator, u) -> np.ndarray:
    """apply_dense (flap.cpp:233-243)."""
    u = _f64(u, op.grid.total())
    out = np.empty(op.grid.shape)
    check(load_library().fw_dense_apply(op._h, _ptr(u), _ptr(out)))
    return out


def apply_toeplitz(order: OrderField, u, ctx: Optional[Context] = None) -> np.ndarray:
    """apply_toeplitz (flap.cpp:245-285): constant order, 1D; NotConstantOrder / DimUnsupported."""
    ctx = ctx or default_context()
    g = order.grid
    J, lo, hi = g._carrays()
    uu = _f64(u, g.total())
    out = np.empty(g.shape)
    check(load_library().fw_apply_toeplitz(ctx.handle, g.dim, J, lo, hi, _ptr(order.values), _ptr(uu), _ptr(out)))
    return out


def truncation_indicator(M: int, mu_abs: float, s0: float) -> float:
    """truncation_indicator (flap.cpp:287-294); NonpositiveFrequency unless |mu| > 0."""
    out = C.c_double(0.0)
    check(load_library().fw_truncation_indicator(int(M), float(mu_abs), float(s0), C.byref(out)))
    return out.value


def rfftn(x, ctx: Optional[Context] = None):
    """Canonical forward real transform on the device (unscaled half spectrum)."""
    ctx = ctx or default_context()
    x = _f64(x)
    shape = x.shape
    J = (C.c_int * 3)(*(list(shape) + [1] * (3 - len(shape))))
    H = np.empty(shape[:-1] + (shape[-1] // 2 + 1,), dtype=np.complex128)
    check(load_library().fw_rfftn(ctx.handle, len(shape), J, _ptr(x), H.view(np.float64).ctypes.data_as(_dp)))
    return H


def irfftn(H, shape, ctx: Optional[Context] = None):
    """Canonical unnormalized C2R on the device."""
    ctx = ctx or default_context()
    H = np.ascontiguousarray(H, dtype=np.complex128)
    J = (C.c_int * 3)(*(list(shape) + [1] * (3 - len(shape))))
    x = np.empty(tuple(shape))
    check(load_library().fw_irfftn(ctx.handle, len(shape), J, H.view(np.float64).ctypes.data_as(_dp), _ptr(x)))
    return x
