"""Pins the CPU oracles before anything is compared against them (CPU only).

1. The reference's own known-answer / property suites pass on the shim-built
   reference (test_grid.cpp:33-98 FFT KATs, Parseval, conjugate symmetry;
   test_flap.cpp; test_seismic.cpp; test_stepping.cpp TSFP2; acceptance 1, 2, 5, 9).
2. The canonical FFT agrees with numpy's pocketfft to the fp64 floor.
3. The C restatement (oracle/fw_oracle.c) reproduces the reference bit for bit,
   both on the committed golden fixtures and on fresh seeded cases.
"""
import hashlib
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as O
from conftest import GOLDEN, ROOT, load_golden
from paper_2311_13049_b200 import configs as cfgs

REF_TESTS = "/root/reference/proj/tests"
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


# ---------------------------------------------------------------------------- 1


@pytest.mark.skipif(not (os.path.exists(os.path.join(ROOT, "oracle/_ref/unit_tests"))
                         and os.path.isdir(REF_TESTS)), reason="reference unit suites need /root/reference")
@pytest.mark.parametrize("suite", ["grid", "flap", "seismic", "orderfield", "stepping"])
def test_reference_unit_suites_pass_on_shim(suite):
    r = subprocess.run([os.path.join(ROOT, "oracle/_ref/unit_tests"), f"-ts={suite}"], cwd=REF_TESTS,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "0 failed" in r.stdout


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle/_ref/acceptance")), reason="no acceptance binary")
@pytest.mark.parametrize("criterion", [1, 2, 5, 9])
def test_reference_acceptance_on_shim(criterion, tmp_path):
    r = subprocess.run([os.path.join(ROOT, "oracle/_ref/acceptance"), "--criterion", str(criterion)],
                       cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout[-3000:]


# ---------------------------------------------------------------------------- 2


@pytest.mark.parametrize("shape", [(4,), (16,), (4096,), (8, 4), (64, 32), (16, 8, 32), (4, 4, 4)])
def test_canonical_fft_matches_pocketfft(shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    H = O.port_rfftn(x)
    ref = np.fft.rfftn(x)
    assert rel_l2(H, ref) < 1e-15 * max(1.0, np.log2(x.size))
    back = O.port_irfftn(H, shape) / x.size
    assert rel_l2(back, x) < 1e-15 * max(1.0, np.log2(x.size))


def test_canonical_fft_pure_modes():
    """test_grid.cpp:73-94 known answers, on the canonical transform directly."""
    J = 16
    x = np.cos(3.0 * np.arange(J) * (2 * np.pi / J))
    H = O.port_rfftn(x) / J
    assert abs(H[3].real - 0.5) < 1e-15
    H[3] = 0.0
    assert np.max(np.abs(H)) < 1e-15
    H = O.port_rfftn(np.full(J, 3.25)) / J
    assert H[0].real == 3.25 and np.max(np.abs(H[1:])) == 0.0


@needs_ref
def test_shim_forward_is_hermitian_and_matches_numpy():
    J, lo, hi = (8, 16), (-1.0, 0.0), (1.0, 4.0)
    u = np.random.default_rng(5).standard_normal(J)
    spec = O.ref_forward(J, lo, hi, u)
    assert rel_l2(spec, np.fft.fftn(u) / u.size) < 1e-15
    # exact conjugate symmetry X[-k] == conj(X[k]) (the property the C2R path relies on)
    neg = spec[(-np.arange(8)) % 8][:, (-np.arange(16)) % 16]
    assert np.array_equal(neg, np.conj(spec))


# ---------------------------------------------------------------------------- 3


def test_golden_fixture_integrity(manifest):
    for key, case in manifest["cases"].items():
        for f in case["files"].values():
            with open(os.path.join(GOLDEN, f["file"]), "rb") as fh:
                assert hashlib.sha256(fh.read()).hexdigest() == f["sha256"], (key, f["file"])


def test_restatement_reproduces_golden_applies(manifest):
    for key, c in manifest["cases"].items():
        if c["kind"] != "apply":
            continue
        u, s = load_golden(c, "u"), load_golden(c, "s")
        out, res = O.port_apply(c["J"], c["lo"], c["hi"], s, u, c["M"])
        assert np.array_equal(out, load_golden(c, "out")), key
        assert res == c["imag_residue"], key
        pert, _ = O.port_apply(c["J"], c["lo"], c["hi"], s, u, c["M"], m_first=1)
        assert np.array_equal(pert, load_golden(c, "pert")), key


def test_restatement_reproduces_golden_seismic(manifest):
    for key, c in manifest["cases"].items():
        if c["kind"] != "seismic":
            continue
        phi, gamma = load_golden(c, "phi"), load_golden(c, "gamma")
        J = tuple(c["J"])
        cc, eta, tc = O.port_medium(J, gamma, np.ones(J), c["omega0"])
        assert np.array_equal(cc, load_golden(c, "c")) and np.array_equal(eta, load_golden(c, "eta"))
        assert np.array_equal(tc, load_golden(c, "tau_coef"))
        l1, _ = O.port_apply(J, c["lo"], c["hi"], 1.0 + gamma, phi, c["M"])
        assert np.array_equal(l1, load_golden(c, "apply_disp")), key
        cur, _, _, n = O.port_seismic(J, c["lo"], c["hi"], gamma, np.ones(J), c["omega0"], c["M"], phi,
                                      np.zeros(J), c["tau"], c["steps"])
        assert n == c["n"]
        assert np.array_equal(cur, load_golden(c, "cur")), key


def test_restatement_reproduces_golden_tsfp2(manifest):
    c = manifest["cases"]["tsfp2_256"]
    s, phi = load_golden(c, "s"), load_golden(c, "phi")
    u, v = O.port_tsfp2(c["J"], c["lo"], c["hi"], s, c["M"], c["kappa"], 1, phi, np.zeros(c["J"]), c["tau"],
                        c["steps"])
    assert np.array_equal(u, load_golden(c, "u")) and np.array_equal(v, load_golden(c, "v"))


def _port_lffp(J, lo, hi, s, M, kappa, cubic, phi, tau, steps):
    """LFFP (stepping.cpp:88-104, 170-181) on the C restatement's apply; the elementwise
    updates in numpy with the reference's evaluation order (IEEE, no contraction)."""
    def L(u):
        return O.port_apply(J, lo, hi, s, u, M)[0].reshape(np.shape(u))

    def f(u):
        return u * u * u if cubic else np.zeros_like(u)

    half_t2 = 0.5 * tau * tau
    prev = np.array(phi, dtype=np.float64)
    cur = prev + tau * np.zeros_like(prev) + half_t2 * (-kappa * L(prev) + f(prev))
    t2 = tau * tau
    for _ in range(steps):
        nxt = 2.0 * cur - prev + t2 * (-kappa * L(cur) + f(cur))
        prev, cur = cur, nxt
    return cur


@pytest.mark.parametrize("key", ["lffp_256", "lffp_cubic_256", "lffp_2d_64"])
def test_restatement_reproduces_golden_lffp(manifest, key):
    """The restatement's apply + the reference's LFFP update reproduce the reference's
    Stepper(Method::LFFP) bit for bit (the CNFP fixtures pin the device CG to tolerance)."""
    c = manifest["cases"][key]
    cur = _port_lffp(tuple(c["J"]), c["lo"], c["hi"], load_golden(c, "s"), c["M"], c["kappa"], c["f"] == "cubic",
                     load_golden(c, "phi"), c["tau"], c["steps"])
    assert np.array_equal(cur, load_golden(c, "cur")), key


@needs_ref
def test_reference_wave_reproduces_golden(manifest):
    for key in ("lffp_256", "cnfp_256", "cnfp_cubic_256"):
        c = manifest["cases"][key]
        cur, n, pt = O.ref_wave(c["method"], c["J"], c["lo"], c["hi"], load_golden(c, "s"), c["M"], c["kappa"],
                                c["f"] == "cubic", load_golden(c, "phi"), np.zeros(c["J"]), c["tau"], c["steps"])
        assert n == c["n"] and pt == c["picard_total"] and np.array_equal(cur, load_golden(c, "cur")), key


@needs_ref
@pytest.mark.parametrize("J,lo,hi,M,m_first,s0", [
    ((64,), (-32.0,), (32.0,), 0, 0, None),
    ((128,), (-32.0,), (32.0,), 15, 0, None),
    ((128,), (-32.0,), (32.0,), 15, 1, None),
    ((128,), (-32.0,), (32.0,), 7, 0, 1.05),
    ((16, 32), (-8.0, -4.0), (8.0, 4.0), 9, 0, None),
    ((8, 8, 16), (0.0, 0.0, 0.0), (1.0, 2.0, 3.0), 5, 1, None),
])
def test_restatement_bitwise_vs_reference(J, lo, hi, M, m_first, s0):
    rng = np.random.default_rng(M + len(J))
    s = cfgs.s1_profile(lo, hi, J) if lo[0] < 0 else 1.0 + 0.2 * rng.uniform(-1, 1, J)
    u = rng.standard_normal(J)
    ref, rres, _, _ = O.ref_apply(J, lo, hi, s, u, M, mode=2 if m_first else 0, s0=s0)
    got, gres = O.port_apply(J, lo, hi, s, u, M, m_first=m_first, s0=s0)
    assert np.array_equal(ref, got)
    assert rres == gres


@needs_ref
@pytest.mark.parametrize("case,code", [
    (dict(M=-1), 3),                              # NegativeM
    (dict(s=2.5), 4),                             # OrderOutOfRange
    (dict(s=None, wide=True), 5),                 # DeviationTooLarge
])
def test_error_codes_match_reference(case, code):
    J, lo, hi = (32,), (-8.0,), (8.0,)
    s = np.full(J, case.get("s") or 1.0)
    if case.get("wide"):
        s = np.linspace(0.05, 1.95, 32)
        s0 = 0.05
    else:
        s0 = None
    u = np.ones(J)
    M = case.get("M", 4)
    with pytest.raises(O.OracleError) as e1:
        O.ref_apply(J, lo, hi, s, u, M, s0=s0)
    with pytest.raises(O.OracleError) as e2:
        O.port_apply(J, lo, hi, s, u, M, s0=s0)
    assert e1.value.code == e2.value.code == code


def test_fp64_noise_floor_vs_independent_fft():
    """Independent numpy (pocketfft C2C) restatement of flap.cpp:38-135 vs the oracle
    on C1: agreement at the fp64 noise floor, not bitwise."""
    import math

    cfg = cfgs.c1()
    s = 1.0 + cfg.gamma
    J, lo, hi = cfg.J, cfg.lo, cfg.hi
    got, _ = O.port_apply(J, lo, hi, s, cfg.phi, cfg.M)
    mu2 = O.port_mu2(J, lo, hi)
    s0 = O.port_order_stats(s)[0]
    uh = np.fft.fftn(cfg.phi) / cfg.N
    out = np.zeros(J)
    pos = mu2 > 0
    base = np.where(pos, np.power(np.where(pos, mu2, 1.0), s0), 0.0)
    L = np.where(pos, np.log(np.where(pos, mu2, 1.0)), 0.0)
    for m in range(cfg.M + 1):
        out += (s - s0) ** m * np.real(np.fft.ifftn(base * L**m / math.factorial(m) * uh)) * cfg.N
    assert rel_l2(got, out) < 5e-12
