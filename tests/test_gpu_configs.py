"""Every BASELINE.json config at its CONFIGURED size against the CPU oracle
(north star: rel L2 <= 1e-12 per apply, <= 1e-10 after the configured steps).

The oracle here is the plain-C restatement (oracle/fw_oracle.c, pinned bit for bit
to the reference compiled against the FFT shim in tests/test_oracle_pins.py): it
streams the terms with the reference recurrences in O(N) memory, so even C4
(512^3, M = 32; 130 GiB of tables in the reference's storage model) fits the host.
The device path under test is asserted (persistent single-launch kernel for C2).
"""
import numpy as np
import pytest

import oracle_lib as O
from paper_2311_13049_b200 import configs as cfgs

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-12
STEP_TOL = 1e-10


def fw():
    import paper_2311_13049_b200 as m

    return m


def rel_l2(a, b):
    nb = np.linalg.norm(np.ravel(b))
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / (nb if nb > 0 else 1.0))


def grid_of(cfg):
    return fw().Grid(list(zip(cfg.lo, cfg.hi)), cfg.J)


def test_c2_200_steps_persistent_vs_oracle():
    """configs[1] as configured: 1024^2, M = 16, tau = 5e-4, 200 SeismicStepper steps
    through the persistent k_step2d kernel (asserted), state (cur, prev, L2prev, n) vs
    the restatement of seismic.cpp:85-133 after the same 200 steps."""
    m = fw()
    cfg = cfgs.c2()
    med = m.build_medium(grid_of(cfg), cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    st = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau)
    assert st.persistent
    st.advance(cfg.steps)
    cur, prev, ap, n = st.state()
    rcur, rprev, rap, rn = O.port_seismic(cfg.J, cfg.lo, cfg.hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M, cfg.phi,
                                          cfg.psi, cfg.tau, cfg.steps)
    assert n == rn == cfg.steps + 1
    assert rel_l2(cur, rcur) <= STEP_TOL and rel_l2(prev, rprev) <= STEP_TOL and rel_l2(ap, rap) <= STEP_TOL
    assert np.array_equal(cur, rcur) and np.array_equal(prev, rprev) and np.array_equal(ap, rap)


@pytest.mark.parametrize("m_first", [0, 1])
@pytest.mark.parametrize("order", ["1+gamma", "1/2+gamma"])
def test_c2_apply_persistent_vs_oracle(order, m_first):
    """configs[1] single applies (apply_matrix_free / apply_perturbation) of both seismic
    orders on the persistent kernel vs the restatement, with the imaginary residue."""
    m = fw()
    cfg = cfgs.c2()
    s = (1.0 if order == "1+gamma" else 0.5) + cfg.gamma
    op = m.build_expansion(m.OrderField(grid_of(cfg), s), cfg.M)
    assert op.persistent
    got, res = op.apply(cfg.phi, m_first, residue=True)
    ref, rres = O.port_apply(cfg.J, cfg.lo, cfg.hi, s, cfg.phi, cfg.M, m_first=m_first)
    assert rel_l2(got, ref) <= APPLY_TOL and np.array_equal(got, ref)
    assert res == rres


@pytest.mark.parametrize("J", [(1024, 1024), (512, 1024)])
def test_persistent_shapes_vs_oracle(J):
    """Every shape the persistent kernel serves (step2d_supported), random s and u,
    both m_first, vs the restatement."""
    m = fw()
    lo, hi = (-16.0, -16.0), (16.0, 16.0)
    g = m.Grid(list(zip(lo, hi)), J)
    rng = np.random.default_rng(J[0] + 3 * J[1])
    s = 1.0 + 0.4 * cfgs.mode_sum(lo, hi, J, *cfgs.random_modes(rng, 6, 3, 2)) / 6.0
    s = np.clip(s, 0.6, 1.4)
    u = rng.standard_normal(J)
    op = m.build_expansion(m.OrderField(g, s), 16)
    assert op.persistent
    for m_first in (0, 1):
        got, res = op.apply(u, m_first, residue=True)
        ref, rres = O.port_apply(J, lo, hi, s, u, 16, m_first=m_first)
        assert np.array_equal(got, ref), (m_first, rel_l2(got, ref))
        assert res == rres


def test_c3_full_size_vs_oracle():
    """configs[2] at 256^3 (M = 16): one apply per seismic order, then the stepper's
    construction + 5 steps, vs the restatement."""
    m = fw()
    cfg = cfgs.c3()
    g = grid_of(cfg)
    for s in cfgs.orders(cfg):
        got = m.apply_matrix_free(m.build_expansion(m.OrderField(g, s), cfg.M), cfg.phi)
        ref, _ = O.port_apply(cfg.J, cfg.lo, cfg.hi, s, cfg.phi, cfg.M)
        assert rel_l2(got, ref) <= APPLY_TOL and np.array_equal(got, ref)
    st = m.SeismicStepper(m.build_medium(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M), cfg.phi, cfg.psi, cfg.tau)
    st.advance(5)
    cur, prev, ap, n = st.state()
    rcur, rprev, rap, rn = O.port_seismic(cfg.J, cfg.lo, cfg.hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M, cfg.phi,
                                          cfg.psi, cfg.tau, 5)
    assert n == rn == 6
    assert rel_l2(cur, rcur) <= STEP_TOL and np.array_equal(cur, rcur)
    assert np.array_equal(prev, rprev) and np.array_equal(ap, rap)


@pytest.mark.parametrize("order", ["1+gamma", "1/2+gamma"])
def test_c4_full_size_apply_vs_oracle(order):
    """configs[3] at 512^3 (M = 32): one apply per seismic order vs the term-streaming
    restatement (the reference's own storage model needs 130 GiB of host tables)."""
    m = fw()
    cfg = cfgs.c4()
    s = (1.0 if order == "1+gamma" else 0.5) + cfg.gamma
    op = m.build_expansion(m.OrderField(grid_of(cfg), s), cfg.M)
    got = m.apply_matrix_free(op, cfg.phi)
    del op
    ref, _ = O.port_apply(cfg.J, cfg.lo, cfg.hi, s, cfg.phi, cfg.M)
    assert rel_l2(got, ref) <= APPLY_TOL and np.array_equal(got, ref)


def test_c2_pipelined_shots_equal_serial_stepper():
    """fw_seis_step_io_async / fw_seis_wait: three independent shots (one context = one stream
    each) stepped round-robin with the host owning every shot's wavefield between steps give,
    for every shot, exactly the fields a lone stepper computes with fw_seis_step_io; the
    persistent kernels of the shots serialise on the device while their copies overlap."""
    m = fw()
    cfg = cfgs.c2()
    med = m.build_medium(grid_of(cfg), cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    nshots, nsteps = 3, 4
    phis = [cfg.phi * (1.0 + 0.125 * i) for i in range(nshots)]
    want = []
    for phi in phis:
        st = m.SeismicStepper(med, phi, cfg.psi, cfg.tau)
        assert st.persistent
        buf = st.current()
        for _ in range(nsteps):
            st.step_io(buf, buf)
        want.append(buf.copy())
        del st
    ctxs = [m.Context(0) for _ in range(nshots)]
    shots = [m.SeismicStepper(med, phi, cfg.psi, cfg.tau, ctx=c) for phi, c in zip(phis, ctxs)]
    bufs = [s.current() for s in shots]
    for r in range(nsteps):
        for s, b in zip(shots, bufs):
            if r:
                s.wait()
                b += 0.0  # the host touches the wavefield between the steps
            s.step_io_async(b, b)
    for s in shots:
        s.wait()
    for b, w, s in zip(bufs, want, shots):
        assert np.array_equal(b, w)
        assert s.n() == nsteps + 1


def test_step_io_async_blowup_reports_at_wait():
    """A blow-up inside an asynchronous call surfaces at fw_seis_wait with the reference's
    semantics (seismic.cpp:124-129): n = the offending step, the pending output = the pre-step
    wavefield, exactly as the synchronous stepper reports it."""
    m = fw()
    J, lo, hi = (128, 128), (-16.0, -16.0), (16.0, 16.0)
    g = m.Grid(list(zip(lo, hi)), J)
    x = np.linspace(-16, 16, J[0], endpoint=False)
    phi = np.exp(-(x[:, None] ** 2 + x[None, :] ** 2) / 0.5)
    med = m.build_medium(g, np.full(J, 0.05), np.ones(J), 1.0, 4)
    tau = 0.5  # far beyond stability (tau c |mu|_max^(1+gamma) >> 2)
    ref = m.SeismicStepper(med, phi, np.zeros(J), tau)
    with pytest.raises(m.BlowupDetected):
        ref.advance(400)
    rcur, _, _, rn = ref.state()
    assert 2 < rn < 400
    st = m.SeismicStepper(med, phi, np.zeros(J), tau)
    out = np.empty(J)
    st.step_io_async(None, out, steps=400)
    with pytest.raises(m.BlowupDetected):
        st.wait()
    assert st.n() == rn and np.array_equal(out, rcur)
