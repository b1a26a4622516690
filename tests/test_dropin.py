"""The drop-in: the reference's OWN test suites, linked against the B200 backend
(paper_2311_13049_b200/cpp: flap.cpp's apply_matrix_free / _serial /
apply_perturbation replaced by flap_gpu.cpp over the C-ABI).  Every operator
apply made by the reference's tests, SeismicStepper and Laplacian seam runs on
the GPU."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BUILD = os.path.join(ROOT, "paper_2311_13049_b200", "cpp", "build")
UNIT = os.path.join(BUILD, "unit_tests_gpu")
ACC = os.path.join(BUILD, "acceptance_gpu")
needs_build = pytest.mark.skipif(not os.path.exists(UNIT), reason="drop-in not built (needs /root/reference)")


@needs_build
def test_dropin_links_the_b200_library():
    out = subprocess.run(["ldd", os.path.join(BUILD, "libfracwave_b200dropin.so")], capture_output=True,
                         text=True).stdout
    assert "libfw_b200.so" in out and "not found" not in out


@needs_build
def test_dropin_links_no_oracle_code():
    """The drop-in library carries no CPU FFT: the reference's FFTW calls resolve to the device-backed
    entry points (cpp/fftw_gpu.cpp), nothing from oracle/ (fwcanon / fwshim) is linked."""
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(BUILD, "libfracwave_b200dropin.so")],
                         capture_output=True, text=True).stdout
    assert "fftw_execute_dft" in out and "fftw_plan_dft" in out
    assert not re.search(r"\b(fwc_|fwshim)", out), [ln for ln in out.splitlines() if "fwc_" in ln or "fwshim" in ln][:5]


def _run(cmd, tmp_path):
    env = dict(os.environ, FW_DROPIN_REPORT="1")
    r = subprocess.run(cmd, cwd=tmp_path, capture_output=True, text=True, timeout=900, env=env)
    m = re.search(r"\[fw-dropin\] (\d+) operator applies ran on the B200 backend", r.stderr)
    return r, int(m.group(1)) if m else 0


@pytest.mark.gpu
@needs_build
@pytest.mark.parametrize("suite", ["flap", "seismic", "stepping", "grid"])
def test_reference_unit_suites_on_b200(suite, tmp_path):
    r, n = _run([UNIT, f"-ts={suite}"], tmp_path)
    assert r.returncode == 0 and "0 failed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
    if suite != "grid":
        assert n > 0  # the applies really went through the GPU


@pytest.mark.gpu
@needs_build
@pytest.mark.parametrize("criterion", [1, 2, 5, 8, 9])
def test_reference_acceptance_on_b200(criterion, tmp_path):
    """The reference's acceptance criteria through the drop-in; 8 includes the two-layer 200^2 seismic
    runs (acceptance.cpp:406-432): a non-power-of-two grid on the full-spectrum (Bluestein) path."""
    r, n = _run([ACC, "--criterion", str(criterion)], tmp_path)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
    if criterion != 5:  # criterion 5 uses constant orders only: its perturbations are exact host zeros
        assert n > 0


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(os.path.join(BUILD, "seismic_gpu_check")), reason="drop-in not built")
def test_cpp_gpu_seismic_stepper(tmp_path):
    """fwave::gpu::SeismicStepper (reference API, fused device stepper) against the
    reference's classical-limit LFFP test and against the reference CPU stepper."""
    r = subprocess.run([os.path.join(BUILD, "seismic_gpu_check")], cwd=tmp_path, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(os.path.join(BUILD, "slab_seis_check")), reason="drop-in not built")
def test_cpp_slab_stepper(tmp_path):
    """A C++ host of the reference drives the slab-decomposed stepper of the C-ABI (fw_slab_seis_*)
    on a 3D grid (P = 1 on this one-GPU run; FW_WORLD / FW_RANK / FW_NCCL_ID_FILE select P > 1)
    against the reference's own SeismicStepper."""
    r = subprocess.run([os.path.join(BUILD, "slab_seis_check")], cwd=tmp_path, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(os.path.join(BUILD, "stepper_gpu_check")), reason="drop-in not built")
def test_cpp_gpu_stepper(tmp_path):
    """fwave::gpu::Stepper (reference Stepper API; LFFP / CNFP / TSFP2 on the device)
    against the reference's own Stepper on the same WaveProblem / StepperConfig."""
    r = subprocess.run([os.path.join(BUILD, "stepper_gpu_check")], cwd=tmp_path, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout + r.stderr
