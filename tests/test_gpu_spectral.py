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


# ---------------------------------------------------------------- dense / Toeplitz (flap.cpp:170-285)

def _s1(J, lo, hi):
    X = np.meshgrid(*[lo[a] + (hi[a] - lo[a]) * np.arange(J[a]) / J[a] for a in range(len(J))], indexing="ij")
    return 1.0 + 0.3 * np.sin(np.pi * X[0] / 8)


@pytest.mark.parametrize("J", [(32,), (30,), (16, 12), (8, 6, 4)])
def test_dense_entries_and_apply_vs_reference(J):
    m = fw()
    lo, hi = [-8.0] * len(J), [8.0] * len(J)
    g = m.Grid(list(zip(lo, hi)), J)
    s = _s1(J, lo, hi)
    u = np.random.default_rng(3).standard_normal(J)
    op = m.assemble_dense(m.OrderField(g, s))
    ref_out, ref_ent = O.ref_dense(J, lo, hi, s, u, entries=True)
    assert rel(op.entries, ref_ent) <= 1e-12
    assert rel(m.apply_dense(op, u), ref_out) <= 1e-12


def test_dense_known_answers_and_budget():
    """test_flap.cpp:71-111 on the device: [0, 2pi), J = 4, s = 1 gives a_jj = 1.5; a constant order
    gives a symmetric Toeplitz matrix; the memory budget is a strict bound with the reference's message."""
    m = fw()
    g = m.Grid([(0.0, 2 * np.pi)], (4,))
    a = m.assemble_dense(m.OrderField(g, np.ones(4))).entries
    assert np.allclose(np.diag(a), 1.5, rtol=1e-12, atol=0)
    g2 = m.Grid([(-8.0, 8.0)], (32,))
    a2 = m.assemble_dense(m.OrderField(g2, np.full(32, 0.7))).entries
    assert np.abs(a2 - a2.T).max() < 1e-12 and np.abs(a2[1:, 1:] - a2[:-1, :-1]).max() < 1e-12
    g3 = m.Grid([(0.0, 1.0), (0.0, 1.0)], (256, 256))
    with pytest.raises(m.MemoryBudgetExceeded, match="needs 34359738368 bytes, budget is 34359738368"):
        m.assemble_dense(m.OrderField(g3, np.ones((256, 256))), 32 << 30)


def test_dense_vs_matrix_free_s1_profile():
    """test_flap.cpp:179-186: the matrix-free operator (J = 256 on [-32, 32), M = 15, s1 profile) against
    the dense oracle."""
    m = fw()
    J, lo, hi = (256,), (-32.0,), (32.0,)
    g = m.Grid(list(zip(lo, hi)), J)
    s = _s1(J, lo, hi)
    u = np.random.default_rng(9).standard_normal(J)
    dense = m.apply_dense(m.assemble_dense(m.OrderField(g, s)), u)
    mf = m.apply_matrix_free(m.build_expansion(m.OrderField(g, s), 15), u)
    assert np.abs(mf - dense).max() / np.abs(dense).max() < 1e-10


@pytest.mark.parametrize("J", [(128,), (100,)])
def test_toeplitz_fast_path(J):
    """test_flap.cpp:114-129: against the dense operator and the reference; exact zeros; the errors."""
    m = fw()
    lo, hi = (-8.0,), (8.0,)
    g = m.Grid(list(zip(lo, hi)), J)
    u = np.random.default_rng(5).standard_normal(J)
    of = m.OrderField(g, np.full(J, 0.5))
    fast = m.apply_toeplitz(of, u)
    slow = m.apply_dense(m.assemble_dense(of), u)
    assert np.abs(fast - slow).max() / np.abs(slow).max() < 1e-10
    assert rel(fast, O.ref_toeplitz(J, lo, hi, np.full(J, 0.5), u)) <= 1e-12
    assert np.all(m.apply_toeplitz(of, np.zeros(J)) == 0.0)
    with pytest.raises(m.NotConstantOrder):
        m.apply_toeplitz(m.OrderField(g, _s1(J, lo, hi)), u)
    g2 = m.Grid([(0.0, 1.0), (0.0, 1.0)], (8, 8))
    with pytest.raises(m.DimUnsupported):
        m.apply_toeplitz(m.OrderField(g2, np.full((8, 8), 0.5)), np.zeros((8, 8)))
