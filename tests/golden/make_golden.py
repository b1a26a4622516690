"""Generate the golden fixtures in tests/golden/ by running THE REFERENCE ITSELF
(oracle/_ref/libfracwave_ref.so: the unmodified /root/reference/proj sources built
against the FFTW-API shim) on the seeded synthetic inputs of
paper_2311_13049_b200.configs.  Every array (inputs and outputs) is written with
the reference's own write_snapshot (harness.cpp:541-557) as FWS1; manifest.json
records parameters, sha256 and scalar outputs.

Run in the development container (needs /root/reference to build oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as O  # noqa: E402
from paper_2311_13049_b200 import configs as cfgs  # noqa: E402

lib = O.reference()
lib.ref_write_snapshot.argtypes = [C.c_int, O._ip, O._dp, O._dp, O._dp, C.c_double, C.c_char_p]

manifest = {"generator": "tests/golden/make_golden.py", "oracle": "oracle/_ref (reference sources + fwshim)",
            "cases": {}}


def snap(name, arr, lo, hi, t=0.0):
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    J = O._i32(arr.shape)
    path = os.path.join(HERE, name + ".fws1")
    rc = lib.ref_write_snapshot(arr.ndim, J, O._f64(lo), O._f64(hi), arr.ravel(), float(t), path.encode())
    if rc:
        raise RuntimeError(lib.ref_last_error())
    with open(path, "rb") as f:
        return {"file": name + ".fws1", "sha256": hashlib.sha256(f.read()).hexdigest()}


def apply_case(key, lo, hi, s, u, M, extra=None):
    J = u.shape
    out, res, s0, const = O.ref_apply(J, lo, hi, s, u, M, mode=0)
    pert, pres, _, _ = O.ref_apply(J, lo, hi, s, u, M, mode=2)
    c = {"kind": "apply", "J": list(J), "lo": list(lo), "hi": list(hi), "M": M, "s0": s0,
         "constant_order": const, "imag_residue": res, "imag_residue_pert": pres,
         "files": {"u": snap(key + "_u", u, lo, hi), "s": snap(key + "_s", s, lo, hi),
                   "out": snap(key + "_out", out, lo, hi), "pert": snap(key + "_pert", pert, lo, hi)}}
    if extra:
        c.update(extra)
    manifest["cases"][key] = c


def seismic_case(key, cfg, steps, extra=None):
    J, lo, hi = cfg.J, cfg.lo, cfg.hi
    o1, o2 = cfgs.orders(cfg)
    c, eta, tc, s0d, s0a = O.ref_medium(J, lo, hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    l1, r1, _, _ = O.ref_apply(J, lo, hi, o1, cfg.phi, cfg.M)
    l2, r2, _, _ = O.ref_apply(J, lo, hi, o2, cfg.phi, cfg.M)
    cur, n = O.ref_seismic(J, lo, hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M, cfg.phi, cfg.psi, cfg.tau, steps)
    case = {"kind": "seismic", "J": list(J), "lo": list(lo), "hi": list(hi), "M": cfg.M, "tau": cfg.tau,
            "steps": steps, "n": n, "omega0": cfg.omega0, "s0_disp": s0d, "s0_atten": s0a,
            "files": {"phi": snap(key + "_phi", cfg.phi, lo, hi), "gamma": snap(key + "_gamma", cfg.gamma, lo, hi),
                      "c": snap(key + "_c", c, lo, hi), "eta": snap(key + "_eta", eta, lo, hi),
                      "tau_coef": snap(key + "_tc", tc, lo, hi),
                      "apply_disp": snap(key + "_l1", l1, lo, hi), "apply_atten": snap(key + "_l2", l2, lo, hi),
                      "cur": snap(key + "_cur", cur, lo, hi, n * cfg.tau)}}
    if extra:
        case.update(extra)
    manifest["cases"][key] = case


# C1 at full size (the reference's own CPU-runnable config)
seismic_case("c1", cfgs.c1(), 100, {"config": "BASELINE configs[0]"})
# reduced-size C2 / C3 / C4 media (same construction, smaller grids)
seismic_case("c2_64", cfgs.c2(64), 20, {"config": "configs[1] construction at 64^2"})
c3s = cfgs.c3(16)
seismic_case("c3_16", c3s, 5, {"config": "configs[2] construction at 16^3"})
c4s = cfgs.c4(16)
seismic_case("c4_16", c4s, 3, {"config": "configs[3] construction at 16^3"})
# reference unit-test style cases (test_flap.cpp:179-186, 205-234): s1 profile, white N(0,1) input
rng = np.random.default_rng(17)
lo, hi = (-32.0,), (32.0,)
apply_case("s1_256", lo, hi, cfgs.s1_profile(lo, hi, (256,)), rng.standard_normal(256), 15)
lo2, hi2 = (-8.0, -8.0), (8.0, 8.0)
X, Y = np.meshgrid(*[lo2[m] + np.arange(32) * 0.5 for m in range(2)], indexing="ij")
apply_case("s2d_32", lo2, hi2, 1.0 - 0.4 * np.cos(np.pi * X / 4.0) * np.cos(np.pi * Y / 4.0),
           rng.standard_normal((32, 32)), 20)
apply_case("const_128", lo, hi, np.full(128, 1.3), rng.standard_normal(128), 15)
# C5 construction at 64^2, two M values
f = cfgs.c5_field(3, n=64)
apply_case("c5_64_M8", f.lo, f.hi, f.s, f.u, 8)
apply_case("c5_64_M32", f.lo, f.hi, f.s, f.u, 32)
# TSFP2 (stepping.cpp:266-304), 1D s1 profile with the cubic nonlinearity (acceptance.cpp:108-122)
lo3, hi3 = (-16.0,), (16.0,)
J3 = (256,)
x = lo3[0] + np.arange(256) * (32.0 / 256)
s3 = cfgs.s1_profile(lo3, hi3, J3)
phi3 = np.exp(-x**2)
u, v = O.ref_tsfp2(J3, lo3, hi3, s3, 15, 1.0, 1, phi3, np.zeros(J3), 1e-3, 20)
manifest["cases"]["tsfp2_256"] = {
    "kind": "tsfp2", "J": list(J3), "lo": list(lo3), "hi": list(hi3), "M": 15, "kappa": 1.0, "f": "cubic",
    "tau": 1e-3, "steps": 20,
    "files": {"s": snap("tsfp2_256_s", s3, lo3, hi3), "phi": snap("tsfp2_256_phi", phi3, lo3, hi3),
              "u": snap("tsfp2_256_u", u, lo3, hi3), "v": snap("tsfp2_256_v", v, lo3, hi3)}}

# LFFP / CNFP (stepping.cpp:170-264) through the reference's Stepper: 1D s1 profile (f none and
# cubic, the CNFP cubic case runs Picard) and a 2D variable order
def wave_case(key, method, lo, hi, s, M, kappa, cubic, phi, tau, steps):
    J = phi.shape
    cur, n, pt = O.ref_wave(method, J, lo, hi, s, M, kappa, cubic, phi, np.zeros(J), tau, steps)
    manifest["cases"][key] = {
        "kind": "wave", "method": method, "J": list(J), "lo": list(lo), "hi": list(hi), "M": M, "kappa": kappa,
        "f": "cubic" if cubic else "none", "tau": tau, "steps": steps, "n": n, "picard_total": pt,
        "files": {"s": snap(key + "_s", s, lo, hi), "phi": snap(key + "_phi", phi, lo, hi),
                  "cur": snap(key + "_cur", cur, lo, hi, n * tau)}}


wave_case("lffp_256", "LFFP", lo3, hi3, s3, 15, 1.0, 0, phi3, 1e-3, 30)
wave_case("lffp_cubic_256", "LFFP", lo3, hi3, s3, 15, 1.0, 1, phi3, 1e-3, 30)
wave_case("cnfp_256", "CNFP", lo3, hi3, s3, 15, 1.0, 0, phi3, 1e-2, 10)
wave_case("cnfp_cubic_256", "CNFP", lo3, hi3, s3, 15, 1.0, 1, phi3, 1e-2, 8)
X2, Y2 = np.meshgrid(*[-8.0 + np.arange(64) * 0.25 for _ in range(2)], indexing="ij")
s_2d = 1.0 - 0.4 * np.cos(np.pi * X2 / 4.0) * np.cos(np.pi * Y2 / 4.0)
phi_2d = np.exp(-(X2**2 + Y2**2))
wave_case("lffp_2d_64", "LFFP", (-8.0, -8.0), (8.0, 8.0), s_2d, 12, 1.0, 0, phi_2d, 2e-3, 25)
wave_case("cnfp_2d_64", "CNFP", (-8.0, -8.0), (8.0, 8.0), s_2d, 12, 1.0, 0, phi_2d, 1e-2, 6)

with open(os.path.join(HERE, "manifest.json"), "w") as fh:
    json.dump(manifest, fh, indent=1, sort_keys=True)
print("wrote", len(manifest["cases"]), "cases")
