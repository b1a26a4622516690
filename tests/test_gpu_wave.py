"""GPU parity of the two-level integrators behind the reference's Laplacian seam
(SURVEY.md §8(f) row 3): Stepper with Method::LFFP / CNFP (stepping.cpp:88-104,
119-138, 170-264) with the state, the Picard iterates and the CG vectors in HBM and
the operator served by the hot-path apply.

Tolerances: LFFP is bit-identical to the reference (every elementwise expression
keeps the reference's order; the apply is bit-identical).  CNFP's dot products are
deterministic tree sums on the device, not the reference's serial sums, so the CG
iterates differ at rounding level; the solves converge to inner_cg_tol = 1e-14, and
the state after the configured steps is asserted to relative L2 <= 1e-10
(STEP_TOL of the north star), with identical step and Picard counts.
"""
import numpy as np
import pytest

import oracle_lib as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-10
WAVE_CASES = ["lffp_256", "lffp_cubic_256", "lffp_2d_64", "cnfp_256", "cnfp_cubic_256", "cnfp_2d_64"]


def fw():
    import paper_2311_13049_b200 as m

    return m


def rel_l2(a, b):
    nb = np.linalg.norm(np.ravel(b))
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / (nb if nb > 0 else 1.0))


def stepper(J, lo, hi, s, M, kappa, f, phi, psi, method, tau, **cfg):
    m = fw()
    grid = m.Grid(list(zip(lo, hi)), J)
    prob = m.WaveProblem(m.OrderField(grid, s), phi, psi, kappa=kappa, f=f, M=M)
    return m.Stepper(prob, m.StepperConfig(method=method, tau=tau, **cfg))


@pytest.mark.parametrize("key", WAVE_CASES)
def test_golden_wave(manifest, key):
    """Committed fixtures written by the reference's own Stepper (tests/golden/make_golden.py)."""
    c = manifest["cases"][key]
    J = tuple(c["J"])
    st = stepper(J, c["lo"], c["hi"], load_golden(c, "s"), c["M"], c["kappa"], c["f"], load_golden(c, "phi"),
                 np.zeros(J), c["method"], c["tau"])
    assert st.n() == 1  # Taylor start: cur = u^1
    st.advance(c["steps"])
    cur = st.current()
    ref = load_golden(c, "cur")
    assert st.n() == c["n"]
    assert st.total_picard_iterations() == c["picard_total"]
    if c["method"] == "LFFP":
        assert np.array_equal(cur, ref), (key, rel_l2(cur, ref))
    else:
        assert rel_l2(cur, ref) <= STEP_TOL, (key, rel_l2(cur, ref))


def test_lffp_persistent_2d_bitwise_vs_reference():
    """LFFP on the persistent-kernel grid (1024^2, M = 16): a few steps through the
    device apply, bitwise against the reference Stepper."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    J, lo, hi = (1024, 1024), (-16.0, -16.0), (16.0, 16.0)
    X, Y = np.meshgrid(*[lo[m] + np.arange(J[m]) * (32.0 / J[m]) for m in range(2)], indexing="ij")
    s = 1.2 + 0.2 * np.tanh(Y)
    phi = np.exp(-(X**2 + Y**2) / 0.5)
    ref, n_r, _ = O.ref_wave("LFFP", J, lo, hi, s, 16, 1.0, 0, phi, np.zeros(J), 5e-4, 3)
    st = stepper(J, lo, hi, s, 16, 1.0, "none", phi, np.zeros(J), "LFFP", 5e-4)
    st.advance(3)
    assert st.n() == n_r
    cur = st.current()
    assert np.array_equal(cur, ref), rel_l2(cur, ref)


def test_lffp_blowup_in_a_batch_keeps_pre_step_levels():
    """A too-large step blows up in the middle of one advance(): the device freezes the
    later updates, the host reports BlowupDetected with the reference's n (incremented
    before the check, stepping.cpp:178-179) and the levels before the offending step."""
    m = fw()
    J, lo, hi = (256,), (-16.0,), (16.0,)
    x = lo[0] + np.arange(256) * (32.0 / 256)
    s = 1.5 + 0.3 * np.tanh(x)
    phi = np.exp(-x**2)
    tau = 0.9
    if O.ref_available():
        cur_r, n_r, _, rc = O.ref_wave("LFFP", J, lo, hi, s, 8, 1.0, 0, phi, np.zeros(J), tau, 400,
                                       allow_error=True)
        assert rc == 7
    st = stepper(J, lo, hi, s, 8, 1.0, "none", phi, np.zeros(J), "LFFP", tau)
    with pytest.raises(m.BlowupDetected):
        st.advance(400)
    n_b = st.n()
    assert 1 < n_b < 400
    if O.ref_available():
        assert n_b == n_r
        assert np.array_equal(st.current(), cur_r)
    # the state is usable: stepping again from the pre-blow-up levels blows up again
    with pytest.raises(m.BlowupDetected):
        st.advance(400)


def test_cnfp_errors_match_reference():
    """CgStagnated (cg_max_iters too small) and PicardDiverged (one Picard sweep) are
    raised as by the reference; the state and n are unchanged."""
    m = fw()
    J, lo, hi = (128,), (-8.0,), (8.0,)
    x = lo[0] + np.arange(128) * (16.0 / 128)
    s = 1.4 + 0.2 * np.sin(x)
    phi = np.exp(-x**2)
    # CG capped at one iteration with a tight tolerance
    st = stepper(J, lo, hi, s, 8, 1.0, "none", phi, np.zeros(J), "CNFP", 5e-2, cg_max_iters=1)
    before = st.current()
    with pytest.raises(m.CgStagnated):
        st.step()
    assert st.n() == 1 and np.array_equal(st.current(), before)
    if O.ref_available():
        _, n_r, _, rc = O.ref_wave("CNFP", J, lo, hi, s, 8, 1.0, 0, phi, np.zeros(J), 5e-2, 1, cg_max_iters=1,
                                   allow_error=True)
        assert rc == 16 and n_r == 1
    # one Picard sweep cannot meet picard_tol for the cubic problem
    st = stepper(J, lo, hi, s, 8, 1.0, "cubic", phi, np.zeros(J), "CNFP", 5e-2, picard_max_iters=1)
    with pytest.raises(m.PicardDiverged):
        st.step()
    assert st.n() == 1 and st.total_picard_iterations() == 1
    if O.ref_available():
        _, n_r, pt_r, rc = O.ref_wave("CNFP", J, lo, hi, s, 8, 1.0, 1, phi, np.zeros(J), 5e-2, 1,
                                      picard_max_iters=1, allow_error=True)
        assert rc == 15 and n_r == 1 and pt_r == 1


def test_stepper_facade_tsfp2_matches_golden(manifest):
    """Stepper(method = TSFP2) is the TSFP2 stepper (bitwise, golden fixture)."""
    c = manifest["cases"]["tsfp2_256"]
    J = tuple(c["J"])
    st = stepper(J, c["lo"], c["hi"], load_golden(c, "s"), c["M"], c["kappa"], c["f"], load_golden(c, "phi"),
                 np.zeros(J), "TSFP2", c["tau"])
    st.advance(c["steps"])
    assert st.n() == c["steps"]
    assert np.array_equal(st.current(), load_golden(c, "u"))
    assert np.array_equal(st.velocity(), load_golden(c, "v"))


@pytest.mark.parametrize("blowup_factor", [2.0, 5.0])
def test_tsfp2_blowup_in_a_batch_matches_reference(blowup_factor):
    """TSFP2 (stepping.cpp:266-304) blowing up inside one multi-step advance(): the device
    leaves (u, v) at the offending step, n() is that step and u the state right after it,
    as after the reference's throw; the StepperConfig blow-up factor is honoured."""
    m = fw()
    J, lo, hi = (256,), (-16.0,), (16.0,)
    x = lo[0] + np.arange(256) * (32.0 / 256)
    s = 1.0 + 0.3 * np.sin(np.pi * x / 8)
    phi = 3.0 * np.exp(-x**2)
    tau = 0.05
    cur_r, n_r, _, rc = O.ref_wave("TSFP2", J, lo, hi, s, 15, 1.0, 1, phi, np.zeros(J), tau, 40,
                                   blowup_factor=blowup_factor, allow_error=True)
    assert rc == 7 and 1 < n_r < 40
    st = stepper(J, lo, hi, s, 15, 1.0, "cubic", phi, np.zeros(J), "TSFP2", tau, blowup_factor=blowup_factor)
    with pytest.raises(m.BlowupDetected):
        st.advance(40)
    assert st.n() == n_r
    assert np.array_equal(st.current(), cur_r)
