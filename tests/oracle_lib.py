"""Test-side ctypes bindings to the CPU oracles (TEST INFRASTRUCTURE ONLY).

Two checkers live under ``oracle/``:

* ``oracle/build/liboracle.so`` -- the plain-C restatement of the reference hot
  path (``oracle/fw_oracle.c``), rebuildable anywhere with gcc (``make -C oracle``).
* ``oracle/_ref/libfracwave_ref.so`` -- the reference itself: the unmodified
  sources of ``/root/reference/proj/src`` compiled against the FFTW-API shim
  (``oracle/fwshim``).  Built in the development container (where
  ``/root/reference`` exists) and shipped to the GPU box as a prebuilt file.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
RESTATEMENT_SO = os.path.join(ORACLE_DIR, "build", "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libfracwave_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _opt_double(v):
    return None if v is None else C.byref(C.c_double(float(v)))


# --------------------------------------------------------------------------
# C restatement


_restatement = None


def restatement():
    """Load (building if needed) oracle/build/liboracle.so."""
    global _restatement
    if _restatement is not None:
        return _restatement
    if not os.path.exists(RESTATEMENT_SO):
        subprocess.run(["make", "-C", ORACLE_DIR, "restatement"], check=True,
                       stdout=subprocess.DEVNULL)
    lib = C.CDLL(RESTATEMENT_SO)
    lib.fwo_last_error.restype = C.c_char_p
    lib.fwo_apply.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_void_p, C.c_int, C.c_int, _dp, _dp,
                              C.POINTER(C.c_double)]
    lib.fwo_mu2.argtypes = [C.c_int, _ip, _dp, _dp, _dp]
    lib.fwo_constant_order.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_double, _dp]
    lib.fwo_medium.argtypes = [C.c_int, _ip, _dp, _dp, C.c_double, _dp, _dp, _dp]
    lib.fwo_seismic.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp,
                                C.c_double, C.c_double, C.c_int, _dp, _dp, _dp,
                                C.POINTER(C.c_long)]
    lib.fwo_tsfp2.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp,
                              C.c_double, C.c_int, _dp, _dp]
    lib.fwo_rfftn.argtypes = [C.c_int, _ip, _dp, _dp]
    lib.fwo_irfftn.argtypes = [C.c_int, _ip, _dp, _dp]
    lib.fwo_order_stats.argtypes = [_dp, C.c_size_t, C.c_void_p, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int)]
    _restatement = lib
    return lib


def _chk(lib, rc, err_fn):
    if rc != 0:
        raise OracleError(rc, err_fn().decode(errors="replace"))


def port_apply(J, lo, hi, s, u, M, m_first=0, s0=None):
    """fwo_apply: apply_matrix_free (m_first=0) / apply_perturbation (m_first=1)."""
    lib = restatement()
    J = _i32(J)
    out = np.empty(int(np.prod(J)), dtype=np.float64)
    res = C.c_double(0.0)
    rc = lib.fwo_apply(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), _opt_double(s0), int(M),
                       int(m_first), _f64(u).ravel(), out, C.byref(res))
    _chk(lib, rc, lib.fwo_last_error)
    return out.reshape(tuple(J)), res.value


def port_mu2(J, lo, hi):
    lib = restatement()
    J = _i32(J)
    out = np.empty(int(np.prod(J)), dtype=np.float64)
    _chk(lib, lib.fwo_mu2(len(J), J, _f64(lo), _f64(hi), out), lib.fwo_last_error)
    return out.reshape(tuple(J))


def port_order_stats(s, s0=None):
    lib = restatement()
    s = _f64(s).ravel()
    z, mn, mx, c = C.c_double(), C.c_double(), C.c_double(), C.c_int()
    _chk(lib, lib.fwo_order_stats(s, s.size, _opt_double(s0), C.byref(z), C.byref(mn),
                                  C.byref(mx), C.byref(c)), lib.fwo_last_error)
    return z.value, mn.value, mx.value, bool(c.value)


def port_constant_order(J, lo, hi, u, s):
    lib = restatement()
    J = _i32(J)
    out = np.empty(int(np.prod(J)), dtype=np.float64)
    _chk(lib, lib.fwo_constant_order(len(J), J, _f64(lo), _f64(hi), _f64(u).ravel(), float(s), out),
         lib.fwo_last_error)
    return out.reshape(tuple(J))


def port_medium(J, gamma, c0, omega0):
    lib = restatement()
    J = _i32(J)
    N = int(np.prod(J))
    c, eta, tc = (np.empty(N) for _ in range(3))
    _chk(lib, lib.fwo_medium(len(J), J, _f64(gamma).ravel(), _f64(c0).ravel(), float(omega0), c,
                             eta, tc), lib.fwo_last_error)
    return c.reshape(tuple(J)), eta.reshape(tuple(J)), tc.reshape(tuple(J))


def port_seismic(J, lo, hi, gamma, c0, omega0, M, phi, psi, tau, nsteps, blowup_factor=1e8,
                 allow_blowup=False):
    """Returns (cur, prev, atten_prev, n) [+ rc when allow_blowup: on BlowupDetected (rc 7) the
    state is the one before the offending step and n is the offending step]."""
    lib = restatement()
    J = _i32(J)
    N = int(np.prod(J))
    cur, prev, ap = (np.empty(N) for _ in range(3))
    n = C.c_long(0)
    rc = lib.fwo_seismic(len(J), J, _f64(lo), _f64(hi), _f64(gamma).ravel(), _f64(c0).ravel(),
                         float(omega0), int(M), _f64(phi).ravel(), _f64(psi).ravel(), float(tau),
                         float(blowup_factor), int(nsteps), cur, prev, ap, C.byref(n))
    shp = tuple(J)
    if allow_blowup and rc == 7:
        return cur.reshape(shp), prev.reshape(shp), ap.reshape(shp), n.value, rc
    _chk(lib, rc, lib.fwo_last_error)
    if allow_blowup:
        return cur.reshape(shp), prev.reshape(shp), ap.reshape(shp), n.value, rc
    return cur.reshape(shp), prev.reshape(shp), ap.reshape(shp), n.value


def port_tsfp2(J, lo, hi, s, M, kappa, cubic, phi, psi, tau, nsteps):
    lib = restatement()
    J = _i32(J)
    N = int(np.prod(J))
    u, v = np.empty(N), np.empty(N)
    rc = lib.fwo_tsfp2(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), int(M), float(kappa),
                       int(bool(cubic)), _f64(phi).ravel(), _f64(psi).ravel(), float(tau),
                       int(nsteps), u, v)
    _chk(lib, rc, lib.fwo_last_error)
    return u.reshape(tuple(J)), v.reshape(tuple(J))


def port_rfftn(x):
    lib = restatement()
    J = _i32(x.shape)
    nh = int(np.prod(J[:-1])) * (int(J[-1]) // 2 + 1)
    H = np.empty(2 * nh)
    _chk(lib, lib.fwo_rfftn(len(J), J, _f64(x).ravel(), H), lib.fwo_last_error)
    return H.view(np.complex128).reshape(tuple(J[:-1]) + (int(J[-1]) // 2 + 1,))


def port_irfftn(H, J):
    lib = restatement()
    J = _i32(J)
    x = np.empty(int(np.prod(J)))
    Hc = np.ascontiguousarray(H, dtype=np.complex128).view(np.float64).ravel()
    _chk(lib, lib.fwo_irfftn(len(J), J, Hc, x), lib.fwo_last_error)
    return x.reshape(tuple(J))


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref)


_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def reference():
    global _ref
    if _ref is not None:
        return _ref
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(REF_SO)
    lib = C.CDLL(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_apply.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_void_p, C.c_int, C.c_int, _dp, _dp,
                              C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.ref_tables.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
    lib.ref_constant_order.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_double, _dp]
    lib.ref_forward.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp]
    lib.ref_ricker.argtypes = [C.c_int, _ip, _dp, _dp, C.c_double, _dp, _dp]
    lib.ref_truncation_indicator.argtypes = [C.c_int, C.c_double, C.c_double, C.POINTER(C.c_double)]
    lib.ref_dense.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_void_p, C.c_void_p]
    lib.ref_toeplitz.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp, _dp]
    lib.ref_medium.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp,
                               _dp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.ref_seismic.argtypes = [C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp,
                                C.c_double, C.c_double, C.c_int, _dp, C.POINTER(C.c_long)]
    lib.ref_tsfp2.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp,
                              C.c_double, C.c_int, _dp, _dp]
    lib.ref_lffp.argtypes = [C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_double, _dp, _dp,
                             C.c_double, C.c_int, _dp]
    lib.ref_wave.argtypes = [C.c_int, C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp,
                             C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int, _dp,
                             C.POINTER(C.c_long), C.POINTER(C.c_long)]
    _ref = lib
    return lib


def ref_apply(J, lo, hi, s, u, M, mode=0, s0=None):
    """mode 0 apply_matrix_free, 1 apply_matrix_free_serial, 2 apply_perturbation.
    Returns (out, imag_residue, s0, constant_order)."""
    lib = reference()
    J = _i32(J)
    out = np.empty(int(np.prod(J)))
    res, z, c = C.c_double(), C.c_double(), C.c_int()
    rc = lib.ref_apply(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), _opt_double(s0), int(M),
                       int(mode), _f64(u).ravel(), out, C.byref(res), C.byref(z), C.byref(c))
    _chk(lib, rc, lib.ref_last_error)
    return out.reshape(tuple(J)), res.value, z.value, bool(c.value)


def ref_tables(J, lo, hi, s, M):
    lib = reference()
    J = _i32(J)
    N = int(np.prod(J))
    mu2, base = np.empty(N), np.empty(N)
    lw, dev = np.empty(max(M, 1) * N), np.empty(max(M, 1) * N)
    z = C.c_double()
    _chk(lib, lib.ref_tables(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), int(M),
                             mu2.ctypes.data, base.ctypes.data, lw.ctypes.data, dev.ctypes.data,
                             C.byref(z)), lib.ref_last_error)
    return mu2, base, lw[: M * N].reshape(M, N), dev[: M * N].reshape(M, N), z.value


def ref_constant_order(J, lo, hi, u, s):
    lib = reference()
    J = _i32(J)
    out = np.empty(int(np.prod(J)))
    _chk(lib, lib.ref_constant_order(len(J), J, _f64(lo), _f64(hi), _f64(u).ravel(), float(s), out),
         lib.ref_last_error)
    return out.reshape(tuple(J))


def ref_forward(J, lo, hi, u):
    lib = reference()
    J = _i32(J)
    out = np.empty(2 * int(np.prod(J)))
    _chk(lib, lib.ref_forward(len(J), J, _f64(lo), _f64(hi), _f64(u).ravel(), out),
         lib.ref_last_error)
    return out.view(np.complex128).reshape(tuple(J))


def ref_truncation_indicator(M, mu_abs, s0):
    lib = reference()
    out = C.c_double()
    _chk(lib, lib.ref_truncation_indicator(int(M), float(mu_abs), float(s0), C.byref(out)), lib.ref_last_error)
    return out.value


def ref_dense(J, lo, hi, s, u, entries=False):
    """assemble_dense + apply_dense of the reference: (A u[, entries])."""
    lib = reference()
    J = _i32(J)
    N = int(np.prod(J))
    out = np.empty(N)
    ent = np.empty(N * N) if entries else None
    _chk(lib, lib.ref_dense(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), _f64(u).ravel(),
                            ent.ctypes.data_as(_dp) if entries else None, out.ctypes.data_as(_dp)), lib.ref_last_error)
    return (out.reshape(tuple(J)), ent.reshape(N, N)) if entries else out.reshape(tuple(J))


def ref_toeplitz(J, lo, hi, s, u):
    lib = reference()
    J = _i32(J)
    out = np.empty(int(np.prod(J)))
    _chk(lib, lib.ref_toeplitz(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), _f64(u).ravel(), out),
         lib.ref_last_error)
    return out.reshape(tuple(J))


def ref_ricker(J, lo, hi, nu0, xc):
    """ricker_initial (seismic.cpp:70-83) of the reference."""
    lib = reference()
    J = _i32(J)
    out = np.empty(int(np.prod(J)))
    _chk(lib, lib.ref_ricker(len(J), J, _f64(lo), _f64(hi), float(nu0), _f64(xc), out), lib.ref_last_error)
    return out.reshape(tuple(J))


def ref_medium(J, lo, hi, gamma, c0, omega0, M):
    lib = reference()
    J = _i32(J)
    N = int(np.prod(J))
    c, eta, tc = (np.empty(N) for _ in range(3))
    z1, z2 = C.c_double(), C.c_double()
    _chk(lib, lib.ref_medium(len(J), J, _f64(lo), _f64(hi), _f64(gamma).ravel(), _f64(c0).ravel(),
                             float(omega0), int(M), c, eta, tc, C.byref(z1), C.byref(z2)),
         lib.ref_last_error)
    shp = tuple(J)
    return c.reshape(shp), eta.reshape(shp), tc.reshape(shp), z1.value, z2.value


def ref_seismic(J, lo, hi, gamma, c0, omega0, M, phi, psi, tau, nsteps, blowup_factor=1e8,
                allow_blowup=False):
    """Returns (cur, n) [+ rc].  Raises OracleError(code 7) on BlowupDetected unless allow_blowup."""
    lib = reference()
    J = _i32(J)
    cur = np.empty(int(np.prod(J)))
    n = C.c_long(0)
    rc = lib.ref_seismic(len(J), J, _f64(lo), _f64(hi), _f64(gamma).ravel(), _f64(c0).ravel(),
                         float(omega0), int(M), _f64(phi).ravel(), _f64(psi).ravel(), float(tau),
                         float(blowup_factor), int(nsteps), cur, C.byref(n))
    if allow_blowup and rc == 7:
        return cur.reshape(tuple(J)), n.value, rc
    _chk(lib, rc, lib.ref_last_error)
    return (cur.reshape(tuple(J)), n.value, rc) if allow_blowup else (cur.reshape(tuple(J)), n.value)


def ref_tsfp2(J, lo, hi, s, M, kappa, cubic, phi, psi, tau, nsteps):
    lib = reference()
    J = _i32(J)
    N = int(np.prod(J))
    u, v = np.empty(N), np.empty(N)
    _chk(lib, lib.ref_tsfp2(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), int(M), float(kappa),
                            int(bool(cubic)), _f64(phi).ravel(), _f64(psi).ravel(), float(tau),
                            int(nsteps), u, v), lib.ref_last_error)
    return u.reshape(tuple(J)), v.reshape(tuple(J))


def ref_lffp(J, lo, hi, s, M, kappa, phi, psi, tau, nsteps):
    lib = reference()
    J = _i32(J)
    u = np.empty(int(np.prod(J)))
    _chk(lib, lib.ref_lffp(len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), int(M), float(kappa),
                           _f64(phi).ravel(), _f64(psi).ravel(), float(tau), int(nsteps), u),
         lib.ref_last_error)
    return u.reshape(tuple(J))


def ref_wave(method, J, lo, hi, s, M, kappa, cubic, phi, psi, tau, nsteps, picard_tol=1e-12,
             picard_max_iters=200, inner_cg_tol=1e-14, cg_max_iters=500, blowup_factor=1e8,
             allow_error=False):
    """Stepper with Method::LFFP ("LFFP") / CNFP ("CNFP") / TSFP2 ("TSFP2") (stepping.cpp:119-138,
    170-304).
    Returns (current, n, total_picard_iterations[, rc])."""
    lib = reference()
    J = _i32(J)
    cur = np.empty(int(np.prod(J)))
    n, pt = C.c_long(), C.c_long()
    rc = lib.ref_wave({"LFFP": 0, "CNFP": 1, "TSFP2": 2}[method], len(J), J, _f64(lo), _f64(hi), _f64(s).ravel(), int(M),
                      float(kappa), int(bool(cubic)), _f64(phi).ravel(), _f64(psi).ravel(), float(tau),
                      float(picard_tol), int(picard_max_iters), float(inner_cg_tol), int(cg_max_iters),
                      float(blowup_factor), int(nsteps), cur, C.byref(n), C.byref(pt))
    if allow_error:
        return cur.reshape(tuple(J)), n.value, pt.value, rc
    _chk(lib, rc, lib.ref_last_error)
    return cur.reshape(tuple(J)), n.value, pt.value
