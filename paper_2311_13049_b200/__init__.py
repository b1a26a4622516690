"""B200-native variable-order fractional-Laplacian apply (fracwave hot path).

Python mirror of the reference's operator / solver interface
(/root/reference/proj/include/fracwave/{grid,orderfield,flap,seismic,stepping}.hpp)
over the C-ABI in ``include/fw_capi.h``.  All compute runs in the sm_100a kernels
of ``lib/libfw_b200.so``; there is no CPU fallback -- importing the compute entry
points without the built library or without a CUDA device raises.

    grid = Grid([(-16.0, 16.0), (-16.0, 16.0)], [1024, 1024])
    op = build_expansion(OrderField(grid, s_values), M=16)      # flap.hpp:24
    Lu = apply_matrix_free(op, u)                               # flap.hpp:34
    med = build_medium(grid, gamma, c0, omega0=1.0, M=16)       # seismic.hpp:25-28
    st = SeismicStepper(med, phi, psi, tau=5e-4)                # seismic.hpp:36-46
    st.advance(200); u = st.current()
"""
from __future__ import annotations

from ._capi import (  # noqa: F401
    BlowupDetected,
    CgStagnated,
    CudaError,
    DeviationTooLarge,
    DimOutOfRange,
    EmptyInterval,
    Error,
    GammaOutOfRange,
    GridMismatch,
    DimUnsupported,
    MemoryBudgetExceeded,
    NotConstantOrder,
    NonpositiveFrequency,
    NegativeM,
    OddSize,
    OrderOutOfRange,
    OutOfMemory,
    PicardDiverged,
    Unsupported,
    library_path,
    load_library,
)
from .api import (  # noqa: F401
    Context,
    ExpansionOperator,
    Grid,
    OrderField,
    SeismicMedium,
    SeismicStepper,
    SlabSeismicStepperC,
    Stepper,
    StepperConfig,
    TSFP2Stepper,
    WaveProblem,
    apply_batch,
    apply_batch_device,
    apply_matrix_free,
    apply_matrix_free_serial,
    apply_perturbation,
    build_expansion,
    build_grid,
    build_medium,
    build_slab_expansion,
    nccl_unique_id,
    default_context,
    DenseOperator,
    apply_constant_order,
    apply_dense,
    apply_toeplitz,
    assemble_dense,
    forward,
    grid_dft,
    inverse,
    irfftn,
    rfftn,
    ricker_initial,
    truncation_indicator,
)

__all__ = [n for n in dir() if not n.startswith("_")]
