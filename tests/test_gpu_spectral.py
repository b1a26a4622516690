"""The reference Grid's spectral utilities and the grids its Grid accepts beyond powers of two,
on the device (VERDICT r1 missing #2 / #9):

* Grid::dft (grid.cpp:134-137) as fw_grid_dft: canonical power-of-two Stockham, Bluestein chirp-z
  for other lengths; Grid::forward / inverse (grid.cpp:171-197);
* apply_constant_order (flap.cpp:137-149), Field and Spectrum forms, with the reference's
  eigenfunction known-answer checks (test_flap.cpp:40-69);
* operators and the seismic stepper on non-power-of-two grids (the full-spectrum C2C form of
  flap.cpp:38-92), against the reference itself (oracle/_ref: FFTW-API shim, mixed radix).

Tolerances: the device transforms are a different (equally exact) DFT algorithm from the
shim's for non-power-of-two lengths, so these checks are to the fp64 floor (rel L2 <= 1e-12
per apply, 1e-10 after steps), bitwise where the canonical plan is shared (power-of-two
constant-order applies)."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def fw():
    import paper_2311_13049_b200 as m

    return m


def rel(a, b):
    nb = np.linalg.norm(np.ravel(b))
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / (nb if nb > 0 else 1.0))


@pytest.mark.parametrize("shape", [(16,), (200,), (4096,), (2048,), (1998,), (6, 10), (200, 200), (64, 96), (12, 20, 8),
                                   (32, 16, 64)])
@pytest.mark.parametrize("sign", [-1, 1])
def test_grid_dft_matches_numpy(shape, sign):
    m = fw()
    g = m.Grid([(0.0, 1.0)] * len(shape), shape)
    rng = np.random.default_rng(sum(shape) + sign)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    got = m.grid_dft(g, x, sign)
    ref = np.fft.fftn(x) if sign < 0 else np.fft.ifftn(x) * x.size
    assert rel(got, ref) <= 5e-15 * np.log2(x.size) + 2e-15, rel(got, ref)


@pytest.mark.parametrize("shape", [(256,), (200,), (32, 32), (30, 36), (8, 12, 10)])
def test_forward_inverse_vs_reference(shape):
    m = fw()
    lo, hi = [-3.0] * len(shape), [5.0] * len(shape)
    g = m.Grid(list(zip(lo, hi)), shape)
    u = np.random.default_rng(len(shape)).standard_normal(shape)
    spec = m.forward(g, u)
    ref = O.ref_forward(shape, lo, hi, u)
    assert rel(spec, ref.reshape(shape)) <= 1e-14
    back, res = m.inverse(g, spec, residue=True)
    assert rel(back, u) <= 1e-14 and res <= 1e-14 * np.abs(u).max()


@pytest.mark.parametrize("J", [(256,), (64, 32), (200,), (40, 30)])
@pytest.mark.parametrize("s", [0.3, 1.0, 1.7])
def test_apply_constant_order_vs_reference(J, s):
    m = fw()
    lo, hi = [-8.0] * len(J), [8.0] * len(J)
    g = m.Grid(list(zip(lo, hi)), J)
    u = np.random.default_rng(7).standard_normal(J)
    got, res = m.apply_constant_order(g, u, s, residue=True)
    ref = O.ref_constant_order(J, lo, hi, u, s)
    ref = ref[0] if isinstance(ref, tuple) else ref
    assert rel(got, ref) <= 1e-12
    if all(n & (n - 1) == 0 for n in J):  # the canonical plan on both sides
        assert np.array_equal(got, ref)
    spec = m.forward(g, u)
    mu2 = O.port_mu2(J, lo, hi) if all(n & (n - 1) == 0 for n in J) else None
    out = m.apply_constant_order(g, spec, s)
    if mu2 is not None:
        f = np.where(mu2 > 0, np.power(np.where(mu2 > 0, mu2, 1.0), s), 0.0)  # numpy pow: within an ulp of glibc
        assert rel(out, spec * f) <= 1e-15


def test_constant_order_eigenfunction_kats():
    """test_flap.cpp:40-69 on the device: cos x is fixed at s = 1 on [0, 2 pi) (|mu| = 1), the mode
    cos 3x scales by 9^s, constants are annihilated, s = 2.5 raises OrderOutOfRange."""
    m = fw()
    J = (64,)
    g = m.Grid([(0.0, 2 * np.pi)], J)
    x = np.arange(64) * (2 * np.pi / 64)
    assert np.abs(m.apply_constant_order(g, np.cos(x), 1.0) - np.cos(x)).max() <= 1e-12
    for s in (0.4, 1.3):
        assert np.abs(m.apply_constant_order(g, np.cos(3 * x), s) - 9.0**s * np.cos(3 * x)).max() <= 1e-11
    assert np.abs(m.apply_constant_order(g, np.full(J, 2.5), 0.8)).max() <= 1e-12
    with pytest.raises(m.OrderOutOfRange):
        m.apply_constant_order(g, np.cos(x), 2.5)


@pytest.mark.parametrize("J,M,m_first", [((200,), 8, 0), ((200,), 8, 1), ((40, 30), 12, 0), ((30, 20, 12), 6, 0),
                                         ((96, 200), 16, 0)])
def test_non_pow2_apply_vs_reference(J, M, m_first):
    """Operators on grids the reference accepts but the real-transform pipeline does not: the
    full-spectrum C2C path (Bluestein transforms) against the reference's apply_matrix_free /
    apply_perturbation."""
    m = fw()
    lo, hi = [-16.0] * len(J), [16.0] * len(J)
    g = m.Grid(list(zip(lo, hi)), J)
    rng = np.random.default_rng(sum(J))
    X = np.meshgrid(*[lo[a] + (hi[a] - lo[a]) * np.arange(J[a]) / J[a] for a in range(len(J))], indexing="ij")
    s = 1.0 + 0.3 * np.sin(np.pi * X[0] / 8)
    u = rng.standard_normal(J)
    op = m.build_expansion(m.OrderField(g, s), M)
    assert not op.persistent
    got, res = op.apply(u, m_first, residue=True)
    ref, rres, _, _ = O.ref_apply(J, lo, hi, s, u, M, mode=2 if m_first else 0)
    assert rel(got, ref) <= 1e-12, rel(got, ref)
    assert res <= 1e-10 * np.linalg.norm(u)


def test_non_pow2_seismic_vs_reference():
    """SeismicStepper on the reference's acceptance-8 grid size (200^2, M = 8, two-layer medium):
    the device stepper after 20 steps against the reference's."""
    m = fw()
    J, lo, hi = (200, 200), (-5.0, -5.0), (5.0, 5.0)
    X, Y = np.meshgrid(*[lo[a] + (hi[a] - lo[a]) * np.arange(J[a]) / J[a] for a in range(2)], indexing="ij")
    gamma = np.where(Y > 0, 0.04, 0.01)
    phi = np.exp(-(X**2 + Y**2) / 0.5)
    g = m.Grid(list(zip(lo, hi)), J)
    st = m.SeismicStepper(m.build_medium(g, gamma, np.ones(J), 1.0, 8), phi, np.zeros(J), 1e-3)
    assert not st.persistent
    st.advance(20)
    cur = st.current()
    rcur, rn = O.ref_seismic(J, lo, hi, gamma, np.ones(J), 1.0, 8, phi, np.zeros(J), 1e-3, 20)
    assert st.n() == rn == 21
    assert rel(cur, rcur) <= 1e-10, rel(cur, rcur)


def test_unsupported_lengths_raise():
    m = fw()
    g = m.Grid([(0.0, 1.0)], (2050,))  # neither a power of two nor within the chirp-z reach
    with pytest.raises(m.Unsupported):
        m.build_expansion(m.OrderField(g, np.full(2050, 1.2)), 4)
