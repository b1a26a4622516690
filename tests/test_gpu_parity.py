"""GPU parity: the sm_100a path (through the C-ABI) vs the CPU oracles.

Tolerances (north star): relative L2 <= 1e-12 for one operator apply, <= 1e-10
after the configured time steps, fp64.  Because the device FFT implements the
same canonical algorithm as the oracle's FFTW shim, most cases
are in fact bit-identical; those are asserted bitwise where stated.
"""
import numpy as np
import pytest

import oracle_lib as O
from conftest import load_golden
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


def grid_of(J, lo, hi):
    return fw().Grid(list(zip(lo, hi)), J)


def gpu_apply(J, lo, hi, s, u, M, m_first=0, s0=None):
    m = fw()
    op = m.build_expansion(m.OrderField(grid_of(J, lo, hi), s, s0), M)
    out, res = op.apply(u, m_first, residue=True)
    return out, res, op


# ------------------------------------------------------------------- golden


def test_golden_applies(manifest):
    for key, c in manifest["cases"].items():
        if c["kind"] != "apply":
            continue
        u, s = load_golden(c, "u"), load_golden(c, "s")
        out, res, op = gpu_apply(tuple(c["J"]), c["lo"], c["hi"], s, u, c["M"])
        assert op.s0 == c["s0"] and op.constant_order == c["constant_order"], key
        assert np.array_equal(out, load_golden(c, "out")), (key, rel_l2(out, load_golden(c, "out")))
        assert res == c["imag_residue"], key
        pert, _, _ = gpu_apply(tuple(c["J"]), c["lo"], c["hi"], s, u, c["M"], m_first=1)
        assert np.array_equal(pert, load_golden(c, "pert")), key


def test_golden_seismic(manifest):
    m = fw()
    for key, c in manifest["cases"].items():
        if c["kind"] != "seismic":
            continue
        J = tuple(c["J"])
        g = grid_of(J, c["lo"], c["hi"])
        phi, gamma = load_golden(c, "phi"), load_golden(c, "gamma")
        l1, _, op1 = gpu_apply(J, c["lo"], c["hi"], 1.0 + gamma, phi, c["M"])
        assert op1.s0 == c["s0_disp"]
        assert rel_l2(l1, load_golden(c, "apply_disp")) <= APPLY_TOL, key
        assert np.array_equal(l1, load_golden(c, "apply_disp")), key
        l2, _, op2 = gpu_apply(J, c["lo"], c["hi"], 0.5 + gamma, phi, c["M"])
        assert op2.s0 == c["s0_atten"]
        assert np.array_equal(l2, load_golden(c, "apply_atten")), key
        st = m.SeismicStepper(m.build_medium(g, gamma, np.ones(J), c["omega0"], c["M"]), phi, np.zeros(J), c["tau"])
        cc, eta, tc = st.coefficients()
        assert np.array_equal(cc, load_golden(c, "c")) and np.array_equal(eta, load_golden(c, "eta"))
        assert np.array_equal(tc, load_golden(c, "tau_coef"))
        st.advance(c["steps"])
        assert st.n() == c["n"]
        cur = st.current()
        ref = load_golden(c, "cur")
        assert rel_l2(cur, ref) <= STEP_TOL, key
        assert np.array_equal(cur, ref), (key, rel_l2(cur, ref))


def test_golden_tsfp2(manifest):
    m = fw()
    c = manifest["cases"]["tsfp2_256"]
    J = tuple(c["J"])
    st = m.TSFP2Stepper(m.OrderField(grid_of(J, c["lo"], c["hi"]), load_golden(c, "s")), c["M"], c["kappa"],
                        load_golden(c, "phi"), np.zeros(J), c["tau"], f="cubic")
    st.advance(c["steps"])
    u, v = st.state()
    assert np.array_equal(u, load_golden(c, "u")) and np.array_equal(v, load_golden(c, "v"))


# ------------------------------------------------------- fresh seeded cases


@pytest.mark.parametrize("J,lo,hi", [
    ((4,), (0.0,), (1.0,)), ((8,), (-1.0,), (1.0,)), ((2048,), (-32.0,), (32.0,)), ((4096,), (-32.0,), (32.0,)),
    ((4, 4), (0.0, 0.0), (1.0, 1.0)), ((8, 128), (-8.0, 0.0), (8.0, 2.0)), ((256, 64), (-8.0, -8.0), (8.0, 8.0)),
    ((4, 8, 16), (0.0, 0.0, 0.0), (1.0, 2.0, 3.0)), ((32, 16, 64), (-4.0, -4.0, -4.0), (4.0, 4.0, 4.0)),
])
@pytest.mark.parametrize("M", [0, 3, 16])
def test_apply_vs_restatement(J, lo, hi, M):
    rng = np.random.default_rng(int(np.prod(J)) + M)
    s = 1.0 + 0.3 * np.sin(np.pi * np.meshgrid(*[np.arange(n) for n in J], indexing="ij")[0] / 8.0)
    u = rng.standard_normal(J)
    for m_first in (0, 1):
        ref, rres = O.port_apply(J, lo, hi, s, u, M, m_first=m_first)
        got, gres, _ = gpu_apply(J, lo, hi, s, u, M, m_first)
        assert rel_l2(got, ref) <= APPLY_TOL
        assert np.array_equal(got, ref), rel_l2(got, ref)
        assert gres == rres


def test_c1_full_config():
    """BASELINE configs[0]: both single applies at <= 1e-12 (bitwise) and 100 steps at <= 1e-10."""
    m = fw()
    cfg = cfgs.c1()
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    for s in cfgs.orders(cfg):
        ref, _ = O.port_apply(cfg.J, cfg.lo, cfg.hi, s, cfg.phi, cfg.M)
        got = m.apply_matrix_free(m.build_expansion(m.OrderField(g, s), cfg.M), cfg.phi)
        assert rel_l2(got, ref) <= APPLY_TOL and np.array_equal(got, ref)
    st = m.SeismicStepper(m.build_medium(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M), cfg.phi, cfg.psi, cfg.tau)
    st.advance(cfg.steps)
    cur, prev, ap, n = st.state()
    rcur, rprev, rap, rn = O.port_seismic(cfg.J, cfg.lo, cfg.hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M, cfg.phi,
                                          cfg.psi, cfg.tau, cfg.steps)
    assert n == rn == 101
    assert rel_l2(cur, rcur) <= STEP_TOL
    assert np.array_equal(cur, rcur) and np.array_equal(prev, rprev) and np.array_equal(ap, rap)


def test_constant_order_collapse_and_perturbation_zero():
    """acceptance criterion 2 / test_flap.cpp:168-177, 208-212 on the device."""
    m = fw()
    J, lo, hi = (256,), (-32.0,), (32.0,)
    g = grid_of(J, lo, hi)
    u = np.random.default_rng(2024).standard_normal(J)
    for s in (0.5, 1.0, 1.3):
        for M in (0, 5, 15):
            op = m.build_expansion(m.OrderField(g, np.full(J, s)), M)
            assert op.constant_order
            a = m.apply_matrix_free(op, u)
            b = O.port_constant_order(J, lo, hi, u, s)
            assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= 1e-13
            p = m.apply_perturbation(op, u)
            assert np.all(p == 0.0)


def test_linearity_and_residue():
    m = fw()
    J, lo, hi = (256, 128), (-32.0, -8.0), (32.0, 8.0)
    g = grid_of(J, lo, hi)
    op = m.build_expansion(m.OrderField(g, cfgs.s1_profile(lo, hi, J)), 15)
    rng = np.random.default_rng(902)
    u, v = rng.standard_normal(J), rng.standard_normal(J)
    lw = m.apply_matrix_free(op, 2.0 * u - 3.0 * v)
    lu, res = m.apply_matrix_free(op, u, residue=True)
    lv = m.apply_matrix_free(op, v)
    assert np.max(np.abs(lw - (2.0 * lu - 3.0 * lv))) / np.max(np.abs(lw)) < 1e-12
    assert res <= 1e-10 * np.linalg.norm(u)


def test_from_tables_matches_build_expansion():
    """Drop-in path: upload a host ExpansionOperator's tables (the reference's own,
    when available) and get the same bits as building on the device."""
    m = fw()
    J, lo, hi = (32, 64), (-8.0, -8.0), (8.0, 8.0)
    s = cfgs.s1_profile(lo, hi, J)
    u = np.random.default_rng(3).standard_normal(J)
    M = 12
    if O.ref_available():
        mu2, base, lw, dev, s0 = O.ref_tables(J, lo, hi, s, M)
    else:
        pytest.skip("reference tables need oracle/_ref")
    op_t = m.ExpansionOperator.from_tables(grid_of(J, lo, hi), M, s0, False, base, lw, dev)
    got = op_t.apply(u)
    ref, _ = O.port_apply(J, lo, hi, s, u, M)
    assert np.array_equal(got, ref)


def test_error_behaviour():
    m = fw()
    g = grid_of((32,), (-8.0,), (8.0,))
    with pytest.raises(m.NegativeM):
        m.build_expansion(m.OrderField(g, np.ones(32)), -1)
    with pytest.raises(m.OrderOutOfRange):
        m.build_expansion(m.OrderField(g, np.full(32, 2.5)), 3)
    with pytest.raises(m.DeviationTooLarge):
        m.build_expansion(m.OrderField(g, np.linspace(0.05, 1.95, 32), 0.05), 3)
    with pytest.raises(m.Unsupported):  # every even length serves up to the device transforms' reach (2048)
        m.build_expansion(m.OrderField(grid_of((4098,), (0.0,), (1.0,)), np.ones(4098)), 3)
    op = m.build_expansion(m.OrderField(g, np.ones(32)), 3)
    with pytest.raises(m.GridMismatch):
        m.apply_matrix_free(op, np.ones(64))
    with pytest.raises(m.GammaOutOfRange):
        m.build_medium(g, np.full(32, 0.6), np.ones(32), 1.0, 4)


def test_blowup_detection_matches_reference():
    """A too-large time step blows up; the device flag reports the same offending
    step as the reference's BlowupDetected (seismic.cpp:124-129), and the state is
    the one before that step."""
    m = fw()
    J, lo, hi = (64,), (-4.0,), (4.0,)
    x = lo[0] + np.arange(64) * (8.0 / 64)
    phi = np.exp(-x**2)
    gamma = np.full(J, 0.05)
    tau = 0.2
    cur_r, prev_r, ap_r, n_r, rc = O.port_seismic(J, lo, hi, gamma, np.ones(J), 1.0, 6, phi, np.zeros(J), tau, 500,
                                                  allow_blowup=True)
    assert rc == 7
    if O.ref_available():
        cur_x, n_x, rc_x = O.ref_seismic(J, lo, hi, gamma, np.ones(J), 1.0, 6, phi, np.zeros(J), tau, 500,
                                         allow_blowup=True)
        assert rc_x == 7 and n_x == n_r and np.array_equal(cur_x, cur_r)
    st = m.SeismicStepper(m.build_medium(grid_of(J, lo, hi), gamma, np.ones(J), 1.0, 6), phi, np.zeros(J), tau)
    with pytest.raises(m.BlowupDetected):
        st.advance(500)
    cur, prev, ap, n = st.state()
    assert n == n_r
    assert np.array_equal(cur, cur_r) and np.array_equal(prev, prev_r) and np.array_equal(ap, ap_r)


def test_rfftn_irfftn_device_bitwise():
    m = fw()
    for shape in [(16,), (4096,), (64, 32), (8, 16, 32)]:
        x = np.random.default_rng(len(shape)).standard_normal(shape)
        H = m.rfftn(x)
        assert np.array_equal(H, O.port_rfftn(x))
        assert np.array_equal(m.irfftn(H, shape), O.port_irfftn(H, shape))


def test_c2_full_size_properties():
    """configs[1] at full size (1024^2): too big for a quick CPU apply, checked
    through size-independent properties + a bitwise check of a row band."""
    m = fw()
    cfg = cfgs.c2()
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    s = 1.0 + cfg.gamma
    op = m.build_expansion(m.OrderField(g, s), cfg.M)
    a = m.apply_matrix_free(op, cfg.phi)
    b = m.apply_matrix_free(op, 2.0 * cfg.phi)
    assert np.array_equal(b, 2.0 * a)  # scaling by 2 is exact in fp64
    full = m.apply_matrix_free(op, cfg.phi)
    assert np.array_equal(a, full)  # deterministic
    ref, _ = O.port_apply(cfg.J, cfg.lo, cfg.hi, s, cfg.phi, cfg.M)
    assert rel_l2(a, ref) <= APPLY_TOL and np.array_equal(a, ref)


# ------------------------------------------- persistent 2D kernel vs multi-pass path


def generic_context():
    import os

    m = fw()
    os.environ["FW_FORCE_GENERIC"] = "1"
    try:
        return m.Context(0)
    finally:
        del os.environ["FW_FORCE_GENERIC"]


@pytest.mark.parametrize("J", [(512, 1024), (1024, 1024)])
def test_persistent_2d_apply_bitwise(J):
    """The single-launch persistent kernel (fw_step2d.cu; asserted to serve these shapes)
    and the multi-pass kernels implement the same canonical arithmetic: identical bits,
    both m_first values, and both equal to the oracle."""
    m = fw()
    lo, hi = (-16.0, -16.0), (16.0, 16.0)
    g = grid_of(J, lo, hi)
    rng = np.random.default_rng(J[0] + J[1])
    s = 1.0 + 0.4 * cfgs.mode_sum(lo, hi, J, *cfgs.random_modes(rng, 6, 3, 2)) / 6.0
    s = np.clip(s, 0.6, 1.4)
    u = rng.standard_normal(J)
    gctx = generic_context()
    op_p = m.build_expansion(m.OrderField(g, s), 16)
    op_g = m.build_expansion(m.OrderField(g, s), 16, ctx=gctx)
    assert op_p.persistent and not op_g.persistent
    for m_first in (0, 1):
        a, ra = op_p.apply(u, m_first, residue=True)
        b, rb = op_g.apply(u, m_first, residue=True)
        assert np.array_equal(a, b), rel_l2(a, b)
        assert ra == rb
        ref, rres = O.port_apply(J, lo, hi, s, u, 16, m_first=m_first)
        assert np.array_equal(a, ref) and ra == rres


@pytest.mark.parametrize("J", [(256, 256), (512, 512), (1024, 512), (2048, 256)])
def test_multipass_2d_apply_vs_oracle(J):
    """2D shapes the persistent kernel does not serve run the multi-pass line kernels
    (asserted): bitwise against the oracle, both m_first values."""
    m = fw()
    lo, hi = (-16.0, -16.0), (16.0, 16.0)
    g = grid_of(J, lo, hi)
    rng = np.random.default_rng(7 * J[0] + J[1])
    s = np.clip(1.0 + 0.4 * cfgs.mode_sum(lo, hi, J, *cfgs.random_modes(rng, 6, 3, 2)) / 6.0, 0.6, 1.4)
    u = rng.standard_normal(J)
    op = m.build_expansion(m.OrderField(g, s), 16)
    assert not op.persistent
    for m_first in (0, 1):
        a, ra = op.apply(u, m_first, residue=True)
        ref, rres = O.port_apply(J, lo, hi, s, u, 16, m_first=m_first)
        assert np.array_equal(a, ref) and ra == rres


def test_persistent_2d_seismic_bitwise():
    """7 seismic steps at 1024^2: persistent kernel (asserted) = multi-pass path = oracle."""
    m = fw()
    cfg = cfgs.c2(1024)
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    med = m.build_medium(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    st_p = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau)
    st_g = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau, ctx=generic_context())
    assert st_p.persistent and not st_g.persistent
    st_p.advance(7)
    st_g.advance(7)
    for a, b in zip(st_p.state(), st_g.state()):
        assert np.array_equal(a, b)
    rcur, rprev, rap, rn = O.port_seismic(cfg.J, cfg.lo, cfg.hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M,
                                          cfg.phi, cfg.psi, cfg.tau, 7)
    cur, prev, ap, n_ = st_p.state()
    assert n_ == rn and np.array_equal(cur, rcur) and np.array_equal(prev, rprev) and np.array_equal(ap, rap)


def test_c2_200_steps_vs_multipass():
    """configs[1] exactly as configured (1024^2, M=16, 200 steps): persistent vs multi-pass
    bitwise, and rel L2 <= 1e-10 trivially satisfied."""
    m = fw()
    cfg = cfgs.c2()
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    med = m.build_medium(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    st_p = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau)
    st_g = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau, ctx=generic_context())
    assert st_p.persistent and not st_g.persistent
    st_p.advance(cfg.steps)
    st_g.advance(cfg.steps)
    a, b = st_p.current(), st_g.current()
    assert st_p.n() == cfg.steps + 1
    assert rel_l2(a, b) <= STEP_TOL and np.array_equal(a, b)


# ------------------------------------------------------------- configs[2..4]


def test_c5_fields_accuracy_vs_M():
    """configs[4] construction at full size (512^2 fields): every M of the sweep
    matches the oracle bitwise, and the truncation error against a converged
    M = 96 reference falls monotonically with M."""
    m = fw()
    for f in (0, 1):
        fld = cfgs.c5_field(f)
        g = grid_of(fld.J, fld.lo, fld.hi)
        ref96, _ = O.port_apply(fld.J, fld.lo, fld.hi, fld.s, fld.u, 96)
        trunc = []
        for M in cfgs.C5_M:
            got = m.apply_matrix_free(m.build_expansion(m.OrderField(g, fld.s), M), fld.u)
            ref, _ = O.port_apply(fld.J, fld.lo, fld.hi, fld.s, fld.u, M)
            assert rel_l2(got, ref) <= APPLY_TOL and np.array_equal(got, ref), (f, M)
            trunc.append(rel_l2(got, ref96))
        assert all(a > b for a, b in zip(trunc[:3], trunc[1:4])), trunc
        assert trunc[3] < 1e-10, trunc


def test_c3_proxy_bitwise_and_full_size_properties():
    """configs[2] construction: a 64^3 proxy (same h = 1/16 ... here [-2,2)^3) bitwise
    against the oracle for both seismic orders and 3 steps; full 256^3 apply checked
    for determinism and exact scaling."""
    m = fw()
    cfg = cfgs.c3(64, L=2.0)
    for s in cfgs.orders(cfg):
        got = m.apply_matrix_free(m.build_expansion(m.OrderField(grid_of(cfg.J, cfg.lo, cfg.hi), s), cfg.M),
                                  cfg.phi)
        ref, _ = O.port_apply(cfg.J, cfg.lo, cfg.hi, s, cfg.phi, cfg.M)
        assert np.array_equal(got, ref)
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    st = m.SeismicStepper(m.build_medium(g, cfg.gamma, cfg.c0, 1.0, cfg.M), cfg.phi, cfg.psi, cfg.tau)
    st.advance(3)
    rcur, _, _, _ = O.port_seismic(cfg.J, cfg.lo, cfg.hi, cfg.gamma, cfg.c0, 1.0, cfg.M, cfg.phi, cfg.psi,
                                   cfg.tau, 3)
    assert np.array_equal(st.current(), rcur)
    full = cfgs.c3()
    op = m.build_expansion(m.OrderField(grid_of(full.J, full.lo, full.hi), 1.0 + full.gamma), full.M)
    a = m.apply_matrix_free(op, full.phi)
    assert np.array_equal(m.apply_matrix_free(op, 2.0 * full.phi), 2.0 * a)
    assert np.isfinite(a).all() and np.abs(a).max() > 0


def test_slab_device_stages_equal_single_gpu_apply():
    """The slab-decomposed orchestration on the device stages (P = 1 here: one GPU in
    this run) gives the single-GPU apply's bits; the P = 2 decomposition logic is
    checked bitwise against P = 1 on CPU in tests/test_slab.py."""
    import torch

    m = fw()
    from paper_2311_13049_b200.slab import SlabGeometry, slab_apply_device

    cfg = cfgs.c3(64, L=2.0)
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    op = m.build_expansion(m.OrderField(g, 1.0 + cfg.gamma), cfg.M)
    ref = op.apply(cfg.phi)
    geo = SlabGeometry(cfg.J, 1, 0)
    u = torch.from_numpy(np.ascontiguousarray(cfg.phi)).cuda()
    for m_first in (0, 1):
        got = slab_apply_device(op, u, geo, op.ctx, m_first=m_first)
        op.ctx.sync()
        want = ref if m_first == 0 else op.apply(cfg.phi, 1)
        assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("J,nf", [((512, 512), 6), ((64, 128), 3), ((32, 32, 16), 2)])
def test_batched_apply_equals_per_field(J, nf):
    """fw_apply_batch_device (one batched pipeline for all fields, configs[4]) gives the
    bits of one apply per field, and of the oracle for a small case."""
    m = fw()
    lo, hi = tuple(-4.0 for _ in J), tuple(4.0 for _ in J)
    g = grid_of(J, lo, hi)
    rng = np.random.default_rng(17 + len(J))
    ops, us = [], []
    for f in range(nf):
        s = 0.9 + 0.2 * rng.random(J)
        ops.append(m.build_expansion(m.OrderField(g, s), 8))
        us.append(rng.standard_normal(J))
    got = m.apply_batch(ops, us)
    for op, u, x in zip(ops, us, got):
        assert np.array_equal(x, op.apply(u))


def chunk_context(l2_mb, group):
    import os

    m = fw()
    os.environ["FW_BATCH_L2_MB"] = str(l2_mb)
    os.environ["FW_BATCH_GROUP"] = str(group)
    try:
        return m.Context(0)
    finally:
        del os.environ["FW_BATCH_L2_MB"]
        del os.environ["FW_BATCH_GROUP"]


@pytest.mark.parametrize("J,nf,M,l2_mb,group", [((512, 512), 5, 9, 5, 2), ((256, 256), 7, 6, 2, 3),
                                                ((256, 256, 256), 2, 3, 300, 1)])
def test_batched_apply_in_l2_chunks_equals_per_field(J, nf, M, l2_mb, group):
    """The batched pipeline in L2-resident chunks (groups of fields x a few terms at a time; the
    row C2R resumes the ascending-m recombination from the earlier chunks' partial sums and
    regenerates the running power (s-s0)^{m-1}): identical bits to one apply per field.  The
    budgets force chunks of 1-2 terms, ragged last chunks and a ragged last field group."""
    m = fw()
    lo, hi = tuple(-4.0 for _ in J), tuple(4.0 for _ in J)
    rng = np.random.default_rng(23 + len(J))
    ctx = chunk_context(l2_mb, group)
    g = grid_of(J, lo, hi)
    ops, ops_c, us = [], [], []
    for f in range(nf):
        s = 0.9 + 0.2 * rng.random(J)
        ops.append(m.build_expansion(m.OrderField(g, s), M))
        ops_c.append(m.build_expansion(m.OrderField(g, s), M, ctx=ctx))
        us.append(rng.standard_normal(J))
    got = m.apply_batch(ops_c, us)
    for op, u, x in zip(ops, us, got):
        assert np.array_equal(x, op.apply(u))


def lines_context():
    import os

    m = fw()
    os.environ["FW_GENERIC_LINES"] = "1"
    try:
        return m.Context(0)
    finally:
        del os.environ["FW_GENERIC_LINES"]


@pytest.mark.parametrize("J", [(256, 16, 8), (512, 8, 8), (1024, 4, 8), (16, 256, 8), (8, 512, 4), (256, 64),
                               (1024, 32), (512, 512), (4, 256), (4, 512), (12, 256), (4, 4, 512)])
def test_register_line_ffts_equal_shared_memory_path(J):
    """fw_lines.cu (register-resident line FFTs for n in {256, 512, 1024}) against the
    shared-memory line kernels: identical bits, both directions (forward + inverse)."""
    m = fw()
    lo, hi = tuple(-3.0 for _ in J), tuple(3.0 for _ in J)
    g = grid_of(J, lo, hi)
    rng = np.random.default_rng(sum(J))
    s = 0.8 + 0.4 * rng.random(J)
    u = rng.standard_normal(J)
    op_a = m.build_expansion(m.OrderField(g, s), 5)
    op_b = m.build_expansion(m.OrderField(g, s), 5, ctx=lines_context())
    for m_first in (0, 1):
        a, ra = op_a.apply(u, m_first, residue=True)
        b, rb = op_b.apply(u, m_first, residue=True)
        assert np.array_equal(a, b) and ra == rb


@pytest.mark.parametrize("J", [(64, 256), (32, 512), (16, 1024), (8, 8, 256), (4, 16, 512), (300 // 75 * 2, 256)])
def test_register_row_c2r_equal_shared_memory_path(J):
    """fw_lines.cu k_rows_c2r (row C2R + ascending-m recombination with registers) against
    the shared-memory k_c2r_accum: identical bits incl. the imaginary residue."""
    m = fw()
    lo, hi = tuple(-3.0 for _ in J), tuple(3.0 for _ in J)
    g = grid_of(J, lo, hi)
    rng = np.random.default_rng(7 * sum(J))
    s = 0.8 + 0.4 * rng.random(J)
    u = rng.standard_normal(J)
    op_a = m.build_expansion(m.OrderField(g, s), 6)
    op_b = m.build_expansion(m.OrderField(g, s), 6, ctx=lines_context())
    for m_first in (0, 1):
        a, ra = op_a.apply(u, m_first, residue=True)
        b, rb = op_b.apply(u, m_first, residue=True)
        assert np.array_equal(a, b) and ra == rb


@pytest.mark.parametrize("J", [(1024, 1024), (512, 1024)])
def test_persistent_multistep_blowup_state(J):
    """A blow-up in the middle of a multi-step persistent launch: the later steps of the
    launch must not overwrite the state the host restores (same offending step and
    pre-step state as the multi-pass path, which matches the reference)."""
    m = fw()
    lo, hi = (-16.0, -16.0), (16.0, 16.0)
    g = grid_of(J, lo, hi)
    phi = np.exp(-(np.linspace(-16, 16, J[0], endpoint=False)[:, None] ** 2
                   + np.linspace(-16, 16, J[1], endpoint=False)[None, :] ** 2) / 0.5)
    gamma = np.full(J, 0.05)
    tau = 0.08  # far beyond stability: |u| explodes within a few dozen steps
    med = m.build_medium(g, gamma, np.ones(J), 1.0, 4)
    st_p = m.SeismicStepper(med, phi, np.zeros(J), tau)
    st_g = m.SeismicStepper(med, phi, np.zeros(J), tau, ctx=generic_context())
    with pytest.raises(m.BlowupDetected):
        st_g.advance(400)
    with pytest.raises(m.BlowupDetected):
        st_p.advance(400)  # one launch of 400 steps
    ref = st_g.state()
    got = st_p.state()
    assert got[3] == ref[3] and 2 < got[3] < 400  # blew up inside the launch, steps left after it
    for a, b in zip(got[:3], ref[:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("P,J", [(2, (256, 256, 32)), (4, (512, 256, 16)), (2, (256, 1024, 8))])
def test_fused_transpose_slab_equals_single_gpu_apply(P, J):
    """Slab decomposition with both transposes fused into the C2C stages
    (fw_stage_c2c_scatter): P virtual ranks on one device, their phases interleaved by the
    host (no kernel waits on another rank); the gathered result is the single-GPU apply's bits."""
    import torch

    m = fw()
    from paper_2311_13049_b200.slab import DeviceStages, FusedSlabApply, LocalPeers, SlabGeometry

    lo, hi = tuple(-3.0 for _ in J), tuple(3.0 for _ in J)
    g = grid_of(J, lo, hi)
    rng = np.random.default_rng(P * 1000 + J[0])
    s = 0.8 + 0.4 * rng.random(J)
    u = rng.standard_normal(J)
    M = 6
    op = m.build_expansion(m.OrderField(g, s), M)
    st = DeviceStages(op.ctx)
    peers = LocalPeers(SlabGeometry(J, P, 0), M + 1, op.ctx)
    for m_first in (0, 1):
        ranks = []
        for r in range(P):
            geo = SlabGeometry(J, P, r)
            wl, dl, ml = st.local_tables(op, geo)
            ranks.append((geo, FusedSlabApply(geo, st, peers, wl, dl, ml)))
        for geo, fa in ranks:
            fa.phase_forward(torch.from_numpy(np.ascontiguousarray(u[geo.rows])).cuda())
        peers.barrier()
        for geo, fa in ranks:
            fa.phase_inverse(m_first)
        peers.barrier()
        parts = [fa.phase_finish(m_first) for geo, fa in ranks]
        op.ctx.sync()
        got = np.concatenate([p.cpu().numpy() for p in parts])
        assert np.array_equal(got, op.apply(u, m_first))


def _slab_case():
    J, lo, hi = (256, 256, 8), (-4.0, -4.0, -1.0), (4.0, 4.0, 1.0)
    x = [lo[a] + (hi[a] - lo[a]) * np.arange(J[a]) / J[a] for a in range(3)]
    X, Y, Z = np.meshgrid(*x, indexing="ij")
    gamma = 0.02 + 0.015 * np.sin(X) * np.cos(0.5 * Y)
    phi = np.exp(-(X**2 + Y**2 + Z**2) / 0.5)
    return J, lo, hi, gamma, phi


def _slab_run(P, tau, blowup_factor, nsteps):
    """P virtual ranks of SlabSeismicStepper on one device (phases interleaved by the host)
    next to the single-GPU SeismicStepper.  Returns (ref stepper, ref exception or None,
    slab states (cur, prev, L2prev) concatenated, slab n, slab offending step or None)."""
    m = fw()
    from paper_2311_13049_b200.slab import LocalPeers, SlabGeometry, SlabSeismicStepper

    # the fused transposes need axis lengths 256/512/1024 for the two transposed axes
    J, lo, hi, gamma, phi = _slab_case()
    c0, psi = np.ones(J), np.zeros(J)
    g = m.Grid(list(zip(lo, hi)), list(J))
    from paper_2311_13049_b200.slab import SlabGeometry as _SG  # noqa: F401
    ref = m.SeismicStepper(m.build_medium(g, gamma, c0, 1.0, 6), phi, psi, tau, blowup_factor=blowup_factor)
    ref_exc = None
    try:
        ref.advance(nsteps)
    except m.BlowupDetected as e:
        ref_exc = e
    ctx = m.default_context()
    shared = {}

    def peers_factory(k, geo, nt, ctx_):
        if k not in shared:
            shared[k] = LocalPeers(SlabGeometry(J, P, 0), nt, ctx_)
        return shared[k]

    sts = [SlabSeismicStepper(g, gamma, c0, 1.0, 6, phi, psi, tau, SlabGeometry(J, P, r), ctx, peers_factory,
                              blowup_factor=blowup_factor, construct=False) for r in range(P)]
    # constructor applies, phase by phase over the virtual ranks
    outs = {}
    for key, k, field in (("l1phi", 0, "phi_l"), ("l2psi", 1, "psi_l"), ("l2phi", 1, "phi_l")):
        for st in sts:
            st.apps[k].phase_forward(getattr(st, field))
        ctx.sync()
        for st in sts:
            st.apps[k].phase_inverse(0)
        ctx.sync()
        outs[key] = [st.apps[k].phase_finish(0) for st in sts]
    for r, st in enumerate(sts):
        st.start(outs["l1phi"][r], outs["l2psi"][r], outs["l2phi"][r])
    for _ in range(nsteps):  # no per-step flag read: the updates freeze once any rank flagged
        for st in sts:
            st.phase_forward()
        ctx.sync()
        for st in sts:
            st.phase_inverse()
        ctx.sync()
        for st in sts:
            st.phase_update()
    bad = None
    for st in sts:  # once, at the end (as advance(): every rank reads the same agreed step)
        try:
            st.check()
        except m.BlowupDetected:
            bad = st.n
    ctx.sync()
    got = [np.concatenate([st.state()[i].cpu().numpy() for st in sts]) for i in range(3)]
    return ref, ref_exc, got, sts[0].n, bad


@pytest.mark.parametrize("P", [1, 2])
def test_slab_seismic_stepper_equals_single_gpu(P):
    """The slab-decomposed SeismicStepper (fused transposes, shared forward transform, fused
    update) with P virtual ranks on one device: cur, prev, L2prev and n identical to the
    single-GPU SeismicStepper after 5 steps."""
    ref, ref_exc, got, n, bad = _slab_run(P, 1e-3, 1e8, 5)
    assert ref_exc is None and bad is None
    cur_r, prev_r, ap_r, n_r = ref.state()
    assert n == n_r
    for a, b in zip(got, (cur_r, prev_r, ap_r)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("P", [1, 2])
def test_slab_seismic_stepper_blowup_matches_single_gpu(P):
    """A blow-up inside the slab stepper: the offending rank's update mins the step into every
    rank's flag, later updates freeze, and the single read at the end agrees with the single-GPU
    stepper's BlowupDetected step; the slab state is rewound to the pre-step state (seismic.cpp:124-129)."""
    m = fw()
    J, lo, hi, gamma, phi = _slab_case()
    tau = 0.2  # far above the explicit scheme's stability limit: sup|u| grows every step from n = 2
    probe = m.SeismicStepper(m.build_medium(m.Grid(list(zip(lo, hi)), list(J)), gamma, np.ones(J), 1.0, 6), phi,
                             np.zeros(J), tau, blowup_factor=1e300)
    sups = []
    for _ in range(4):
        probe.step()
        sups.append(np.abs(probe.current()).max())
    assert sups[3] > max(sups[:3]) > 0
    factor = np.sqrt(max(max(sups[:3]), 1.0) * sups[3]) / np.abs(phi).max()  # first exceeded at n = 5
    ref, ref_exc, got, n, bad = _slab_run(P, tau, factor, 6)
    assert ref_exc is not None and ref.n() == 5 and bad == 5
    cur_r, prev_r, ap_r, _ = ref.state()
    for a, b in zip(got, (cur_r, prev_r, ap_r)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("J", [(32, 64), (16, 32, 16)])
def test_multipass_batched_step_blowup_matches_restatement(J):
    """2D/3D multi-pass seismic step (both operators' inverses batched, grid.z = operator,
    the C2R guarded by the blow-up flag): same offending step and pre-step state as the
    restatement of seismic.cpp:111-133, and bit-identical states before the blow-up."""
    m = fw()
    d = len(J)
    lo, hi = (-4.0,) * d, (4.0,) * d
    axes = [lo[a] + np.arange(J[a]) * (8.0 / J[a]) for a in range(d)]
    r2 = sum(np.meshgrid(*[x**2 for x in axes], indexing="ij"))
    phi = np.exp(-r2)
    rng = np.random.default_rng(7)
    gamma = 0.02 + 0.06 * rng.random(J)
    ctx = generic_context()
    med = m.build_medium(grid_of(J, lo, hi), gamma, np.ones(J), 1.0, 5)
    # stable run: bitwise after 12 steps
    cur_r, prev_r, ap_r, n_r = O.port_seismic(J, lo, hi, gamma, np.ones(J), 1.0, 5, phi, np.zeros(J), 1e-3, 12)
    st = m.SeismicStepper(med, phi, np.zeros(J), 1e-3, ctx=ctx)
    st.advance(12)
    cur, prev, ap, n = st.state()
    assert n == n_r == 13  # SeismicStepper::n counts the start step
    assert np.array_equal(cur, cur_r) and np.array_equal(prev, prev_r) and np.array_equal(ap, ap_r)
    # unstable run: the same offending step and pre-step state
    tau = 0.35
    cur_r, prev_r, ap_r, n_r, rc = O.port_seismic(J, lo, hi, gamma, np.ones(J), 1.0, 5, phi, np.zeros(J), tau, 400,
                                                  allow_blowup=True)
    assert rc == 7
    st = m.SeismicStepper(med, phi, np.zeros(J), tau, ctx=ctx)
    with pytest.raises(m.BlowupDetected):
        st.advance(400)
    cur, prev, ap, n = st.state()
    assert n == n_r
    assert np.array_equal(cur, cur_r) and np.array_equal(prev, prev_r) and np.array_equal(ap, ap_r)


@pytest.mark.parametrize("J", [(1024, 1024), (64, 32)])
def test_seis_step_io_equals_set_step_get(J):
    """fw_seis_step_io (host wavefield in, steps, host wavefield out, one sync) is
    set_current + step + current: identical bits, also on the persistent 1024^2 path,
    and on a blow-up it returns the pre-step state like fw_seis_get."""
    m = fw()
    lo, hi = (-16.0, -16.0), (16.0, 16.0)
    g = grid_of(J, lo, hi)
    x0 = np.linspace(-16, 16, J[0], endpoint=False)[:, None]
    x1 = np.linspace(-16, 16, J[1], endpoint=False)[None, :]
    phi = np.exp(-(x0**2 + x1**2) / 0.5)
    gamma = 0.02 + 0.01 * np.tanh(x1) + 0.0 * x0
    med = m.build_medium(g, gamma, np.ones(J), 1.0, 6)
    a = m.SeismicStepper(med, phi, np.zeros(J), 5e-4)
    b = m.SeismicStepper(med, phi, np.zeros(J), 5e-4)
    u = phi * 0.5
    out = np.empty(J)
    for k in range(3):
        a.set_current(u)
        a.advance(2)
        ref = a.current()
        b.step_io(u, out, steps=2)
        assert np.array_equal(out, ref)
        u = ref * 0.9
    assert a.n() == b.n()
    # blow-up: both report the same offending step and state
    big = m.SeismicStepper(med, phi, np.zeros(J), 0.08 if J[0] == 1024 else 4.0)  # far beyond stability
    with pytest.raises(m.BlowupDetected):
        for _ in range(400):
            big.step_io(None, out)
    cur, _, _, n = big.state()
    assert np.array_equal(out, cur) and n > 1


def test_time_multiplexed_step2d_variant_bitwise():
    """The time-multiplexed persistent kernel (fw_step2d_tm.cu, FW_STEP2D_TM=1; measured slower than
    the warp-specialised default, kept for A/B) computes the same bits: applies (both m_first) and
    5 seismic steps at 1024^2 against the default kernel."""
    import os

    m = fw()
    os.environ["FW_STEP2D_TM"] = "1"
    try:
        tctx = m.Context(0)
    finally:
        del os.environ["FW_STEP2D_TM"]
    cfg = cfgs.c2()
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    s = 1.0 + cfg.gamma
    op_d = m.build_expansion(m.OrderField(g, s), cfg.M)
    op_t = m.build_expansion(m.OrderField(g, s), cfg.M, ctx=tctx)
    assert op_d.persistent and op_t.persistent
    for m_first in (0, 1):
        a, ra = op_d.apply(cfg.phi, m_first, residue=True)
        b, rb = op_t.apply(cfg.phi, m_first, residue=True)
        assert np.array_equal(a, b) and ra == rb
    med = m.build_medium(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    st_d = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau)
    st_t = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau, ctx=tctx)
    st_d.advance(5)
    st_t.advance(5)
    for a, b in zip(st_d.state(), st_t.state()):
        assert np.array_equal(a, b)


def test_persistent_kernel_repeatable_race_probe():
    """compute-sanitizer is closed on this GPU pool, so the persistent kernel's cross-CTA protocol
    (counters, mbarriers, TMA tiles; fw_step2d.cu) is probed by repetition instead: 24 applies of the
    C2 operator and two 60-step seismic runs must reproduce the same bits every time (a missed
    acquire/release or an early tile read would show up as run-to-run differences; the reference's
    determinism contract is flap.cpp:82-90)."""
    m = fw()
    cfg = cfgs.c2()
    g = grid_of(cfg.J, cfg.lo, cfg.hi)
    op = m.build_expansion(m.OrderField(g, 1.0 + cfg.gamma), cfg.M)
    assert op.persistent
    rng = np.random.default_rng(11)
    u = rng.standard_normal(cfg.J)
    first = op.apply(u)
    for _ in range(23):
        assert np.array_equal(op.apply(u), first)
    med = m.build_medium(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    runs = []
    for _ in range(2):
        st = m.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau)
        st.advance(60)
        runs.append(st.state())
    for a, b in zip(runs[0], runs[1]):
        assert np.array_equal(a, b)
