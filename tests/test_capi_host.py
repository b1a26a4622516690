"""CPU-side checks of the product boundary (no GPU compute):
the C-ABI library loads and exports every symbol include/fw_capi.h declares,
errors map onto the reference's exception types, host-side validation matches
grid.cpp / seismic.cpp, and the synthetic config generators are deterministic."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
import oracle_lib as O

import paper_2311_13049_b200 as fw
from paper_2311_13049_b200 import _capi, configs


def header_symbols():
    with open(os.path.join(ROOT, "include", "fw_capi.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fw_[a-z0-9_]+)\s*\(", src)))


def test_library_built():
    assert os.path.exists(_capi.library_path()), "run __graft_entry__.build()"


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(_capi.library_path())
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_capi.EXPORTED_SYMBOLS) <= set(syms)


def test_version_and_no_device_behaviour():
    lib = fw.load_library()
    assert lib.fw_version() == 1
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        # no silent CPU fallback: creating a context fails loudly
        with pytest.raises(fw.CudaError):
            fw.Context(0)


def test_error_classes_map_reference_hierarchy():
    assert issubclass(fw.BlowupDetected, fw.Error) and issubclass(fw.Error, RuntimeError)
    codes = {c.code for c in (fw.GridMismatch, fw.NegativeM, fw.OrderOutOfRange, fw.DeviationTooLarge,
                              fw.GammaOutOfRange, fw.BlowupDetected, fw.OddSize, fw.EmptyInterval,
                              fw.DimOutOfRange)}
    assert codes == {2, 3, 4, 5, 6, 7, 8, 9, 10}


def test_grid_validation_matches_reference():
    """test_grid.cpp:33-41."""
    fw.Grid([(-32.0, 32.0)], [64])
    with pytest.raises(fw.OddSize):
        fw.Grid([(-32.0, 32.0)], [63])
    with pytest.raises(fw.EmptyInterval):
        fw.Grid([(1.0, 1.0)], [64])
    with pytest.raises(fw.EmptyInterval):
        fw.Grid([(2.0, -2.0)], [64])
    with pytest.raises(fw.DimOutOfRange):
        fw.Grid([], [])
    with pytest.raises(fw.DimOutOfRange):
        fw.Grid([(0.0, 1.0)] * 4, [4] * 4)
    g = fw.Grid([(-32.0, 32.0), (0.0, 4.0)], [64, 8])
    assert g.total() == 512 and g.step(0) == 1.0 and g.step(1) == 0.5


def test_gamma_range_checked_on_host():
    g = fw.Grid([(0.0, 2.0)], [32])
    with pytest.raises(fw.GammaOutOfRange):
        fw.build_medium(g, np.full(32, 0.6), np.ones(32), 1.0, 10)
    with pytest.raises(fw.GammaOutOfRange):
        fw.build_medium(g, np.full(32, -0.1), np.ones(32), 1.0, 10)


def test_config_generators_deterministic_and_in_range():
    a, b = configs.c3(16), configs.c3(16)
    assert np.array_equal(a.gamma, b.gamma) and np.array_equal(a.phi, b.phi)
    for cfg in (configs.c1(), configs.c2(64), configs.c3(16), configs.c4(16)):
        assert np.all(cfg.gamma >= 0.0) and np.all(cfg.gamma < 0.5)
        assert abs(cfg.phi).max() > 0
    f = configs.c5_field(7, 64)
    assert 0.55 - 1e-12 <= f.s.min() and f.s.max() <= 1.45 + 1e-12
    # C2 two-layer medium: Q -> 20 (gamma ~ 0.0159) for y > 0, 100 for y < 0
    c2 = configs.c2(64)
    assert abs(c2.gamma[:, -1].mean() - np.arctan(1 / 20) / np.pi) < 1e-4
    assert abs(c2.gamma[:, 0].mean() - np.arctan(1 / 100) / np.pi) < 1e-4


def test_roofline_byte_model():
    """C2 B_apply = 222.4 MB, B_step = 512.0 MB."""
    cfg = configs.c2()
    ba = configs.bytes_per_apply(cfg.N, cfg.N_half, cfg.M)
    bs = configs.bytes_per_seismic_step(cfg.N, cfg.N_half, cfg.M)
    assert abs(ba / 1e6 - 222.4) < 0.1
    assert abs(bs / 1e6 - 512.0) < 0.1


@pytest.mark.skipif(not O.ref_available(), reason="reference (oracle/_ref) not built")
@pytest.mark.parametrize("J,lo,hi,nu0,xc", [
    ((64,), (-8.0,), (8.0,), 2.0, (0.0,)),
    ((32, 48), (-4.0, -2.0), (4.0, 6.0), 1.5, (0.25, 1.0)),
    ((16, 16, 8), (-8.0, -8.0, -8.0), (8.0, 8.0, 8.0), 2.0, (0.0, 0.0, 0.0)),
])
def test_ricker_initial_bitwise_vs_reference(J, lo, hi, nu0, xc):
    """fw_ricker_initial (host, glibc exp) reproduces the reference's ricker_initial (seismic.cpp:70-83)
    bit for bit on the reference's Grid::point coordinates, including non-power-of-two axes."""
    import paper_2311_13049_b200 as fw

    g = fw.Grid(list(zip(lo, hi)), J)
    got = fw.ricker_initial(nu0, xc, g)
    ref = O.ref_ricker(J, lo, hi, nu0, xc)
    assert np.array_equal(got, ref)
    assert got.flat[int(np.argmin(np.abs(got - 1.0)))] <= 1.0  # value 1 at the centre (test_seismic.cpp:51-58)


@pytest.mark.skipif(not O.ref_available(), reason="reference (oracle/_ref) not built")
def test_truncation_indicator_vs_reference():
    """truncation_indicator (flap.cpp:287-294) bit for bit, and NonpositiveFrequency for |mu| <= 0."""
    import paper_2311_13049_b200 as fw

    for M, mu, s0 in [(0, 3.0, 1.2), (8, 17.5, 1.01), (16, 100.0, 0.55), (32, 0.3, 1.4)]:
        assert fw.truncation_indicator(M, mu, s0) == O.ref_truncation_indicator(M, mu, s0)
    with pytest.raises(fw.NonpositiveFrequency):
        fw.truncation_indicator(4, 0.0, 1.0)
