/*
 * fw_capi.h — C-ABI of the B200-native variable-order fractional-Laplacian
 * apply (the hot path of fracwave, arXiv 2311.13049 reference).
 *
 * Plain pointers and sizes only; no exceptions or C++/torch types cross this
 * boundary.  Every call returns an FW_* status; fw_last_error() gives the
 * thread-local message.  Status codes map 1:1 onto the reference's exception
 * types in proj/include/fracwave/errors.hpp (see INTEGRATION.md for the C++
 * shim that re-throws them).
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj):
 *   fw_op_create            build_expansion(OrderField(grid, s, s0), M)   flap.hpp:24, flap.cpp:96-135
 *                           (with OrderField validation orderfield.cpp:10-36, Grid validation grid.cpp:35-58)
 *   fw_op_create_from_tables  uploading a host ExpansionOperator          flap.hpp:14-22
 *   fw_apply                apply_matrix_free / _serial / apply_perturbation  flap.hpp:34-41, flap.cpp:151-168
 *   fw_apply_device         same, device-resident buffers (no reference equivalent: the GPU-resident form)
 *   fw_apply_batch_device   a batch of independent applies (config 5 sweep; reference runs them serially)
 *   fw_seis_create          derive_medium + SeismicStepper ctor           seismic.cpp:11-44, 85-109
 *                           (grids: every even J >= 4 up to the device transforms' reach; power-of-two
 *                           axes take the real-transform pipeline, others the full-spectrum C2C one)
 *   fw_seis_step            SeismicStepper::step / advance               seismic.cpp:111-137
 *   fw_seis_get             SeismicStepper::current / n                  seismic.hpp:44-46
 *   fw_seis_step_io         current() = u; step(); u = current()         seismic.cpp:111-133, seismic.hpp:44
 *   fw_seis_step_io_async / fw_seis_wait   the same, split for overlapping independent steppers
 *   fw_tsfp2_*              Stepper (Method::TSFP2) ctor / step            stepping.cpp:119-138, 266-304
 *   fw_wave_*               Stepper (Method::LFFP / CNFP) ctor / step      stepping.cpp:88-104, 119-138, 170-264
 *                           (the Laplacian seam stepping.hpp:52-60 served by the device apply)
 *   fw_ricker_initial       ricker_initial                               seismic.cpp:70-83
 *   fw_grid_dft[_device]    Grid::dft (in-place unnormalised C2C)         grid.cpp:134-137, grid.hpp:49-51
 *   fw_grid_forward/inverse Grid::forward / Grid::inverse                 grid.cpp:171-197
 *   fw_apply_constant_order apply_constant_order(Field / Spectrum, s)     flap.cpp:137-149
 *   fw_dense_*              assemble_dense / apply_dense                  flap.cpp:170-243
 *   fw_apply_toeplitz       apply_toeplitz                               flap.cpp:245-285
 */
#ifndef FW_CAPI_H
#define FW_CAPI_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FW_CAPI_VERSION 1

enum fw_status {
  FW_OK = 0,
  FW_E_ARG = 1,             /* invalid argument (null pointer, bad handle, bad m_first) */
  FW_E_GRID_MISMATCH = 2,   /* fwave::GridMismatch */
  FW_E_NEGATIVE_M = 3,      /* fwave::NegativeM */
  FW_E_ORDER_RANGE = 4,     /* fwave::OrderOutOfRange */
  FW_E_DEVIATION = 5,       /* fwave::DeviationTooLarge */
  FW_E_GAMMA_RANGE = 6,     /* fwave::GammaOutOfRange */
  FW_E_BLOWUP = 7,          /* fwave::BlowupDetected */
  FW_E_ODD_SIZE = 8,        /* fwave::OddSize */
  FW_E_EMPTY_INTERVAL = 9,  /* fwave::EmptyInterval */
  FW_E_DIM_RANGE = 10,      /* fwave::DimOutOfRange */
  FW_E_OOM = 11,            /* device allocation failed */
  FW_E_CUDA = 12,           /* CUDA runtime error / no device */
  FW_E_UNSUPPORTED = 13,    /* valid for the reference but beyond this backend (axis length past the device
                               transforms; TSFP2 / LFFP / CNFP and the rfftn hooks on non-power-of-two grids) */
  FW_E_NCCL = 14,           /* collective failure (slab-decomposed grids) */
  FW_E_PICARD_DIVERGED = 15,/* fwave::PicardDiverged */
  FW_E_CG_STAGNATED = 16,   /* fwave::CgStagnated */
  FW_E_MEMORY_BUDGET = 17,  /* fwave::MemoryBudgetExceeded */
  FW_E_NOT_CONSTANT = 18,   /* fwave::NotConstantOrder */
  FW_E_DIM_UNSUPPORTED = 19,/* fwave::DimUnsupported */
  FW_E_NONPOSITIVE_FREQ = 20/* fwave::NonpositiveFrequency */
};

typedef struct fw_ctx_s* fw_ctx;
typedef struct fw_op_s* fw_op;
typedef struct fw_seis_s* fw_seis;
typedef struct fw_tsfp2_s* fw_tsfp2;
typedef struct fw_wave_s* fw_wave;
typedef struct fw_dense_s* fw_dense;
typedef struct fw_slab_seis_s* fw_slab_seis;

const char* fw_last_error(void);
int fw_version(void);

/* ---- context: one CUDA device + one stream ---- */
int fw_ctx_create(int device, fw_ctx* out);
void fw_ctx_destroy(fw_ctx ctx);
int fw_ctx_sync(fw_ctx ctx);
/* the CUDA stream (cudaStream_t) all work of this context is issued on */
void* fw_ctx_stream(fw_ctx ctx);
/* the CUDA device index of this context (-1 for a null context) */
int fw_ctx_device(fw_ctx ctx);
/* number of kernels this context has launched so far (diagnostics / bench) */
long long fw_ctx_launches(fw_ctx ctx);
/* diagnostics: the persistent 2D kernel's watchdog records (needs FW_TRACE=1 at context
 * creation; mapped host memory, readable even after the kernel trapped): out receives
 * 156672 unsigned 64-bit words: the watchdog records first (1024 x 16 words, per CTA two records
 * (producer, compute warps) of 8 words {wait site, thread, value seen, target, term, globaltimer}),
 * or, in a trace build (-DFW_STEP2D_TRACE=1), the phase marks read by tools/trace_step2d.py */
int fw_ctx_trace(fw_ctx ctx, unsigned long long* out);

/* ---- operator: ExpansionOperator resident on the device ----
 * grid: dim in {1,2,3}, J[dim] points per axis (even, >= 4: powers of two <= 4096 take the
 * real-transform pipeline; other lengths <= 2048 the full-spectrum C2C form of flap.cpp:38-92
 * through Bluestein transforms), periodic [lo, hi) per axis, row-major with axis 0 slowest.
 * order_values: s(x_j), N = prod(J) doubles.  s0_override: NULL -> serial mean
 * (or s exactly when constant), else the given value.  M >= 0 terms. */
int fw_op_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                 const double* order_values, const double* s0_override, int M, fw_op* out);

/* Upload the tables of an existing host ExpansionOperator (flap.hpp:14-22):
 * base_symbol[N], log_weights[M][N], deviation_powers[M][N] (row pointers).
 * Only the Hermitian half of the spectral tables and deviation_powers[0]
 * are uploaded; higher deviation powers are regenerated on the device with the
 * reference recurrence (flap.cpp:131), which is bit-identical. */
int fw_op_create_from_tables(fw_ctx ctx, int dim, const int* J, const double* lo,
                             const double* hi, int M, double s0, int constant_order,
                             const double* base_symbol, const double* const* log_weights,
                             const double* const* deviation_powers, fw_op* out);
void fw_op_destroy(fw_op op);

typedef struct {
  int dim, J[3], M, constant_order;
  double lo[3], hi[3];
  double s0, smin, smax;
  size_t N, N_half;        /* grid points, Hermitian half-spectrum bins */
  size_t device_bytes;     /* resident table bytes */
} fw_op_info_t;
int fw_op_info(fw_op op, fw_op_info_t* info);
/* which device pipeline serves this operator's applies (diagnostics / tests):
 * FW_PATH_PERSISTENT_2D = the single-launch persistent 2D kernel (fw_step2d.cu),
 * FW_PATH_MULTIPASS = the per-axis line kernels (fw_lines.cu / fw_kernels.cu) */
enum fw_path { FW_PATH_MULTIPASS = 0, FW_PATH_PERSISTENT_2D = 1 };
int fw_op_path(fw_op op);

/* Host buffers in/out (the reference call: Field in, new Field out).
 * m_first: 0 = apply_matrix_free, 1 = apply_perturbation.
 * imag_residue (nullable): max |Im| of the discarded imaginary parts. */
int fw_apply(fw_op op, const double* u_host, double* out_host, int m_first,
             double* imag_residue);
/* Device buffers (u_dev, out_dev: N doubles each), enqueued on the ctx stream;
 * no synchronization.  imag_residue_dev (nullable) is a device double that
 * receives max(|Im|) (it is max-accumulated: caller zeroes it). */
int fw_apply_device(fw_op op, const double* u_dev, double* out_dev, int m_first,
                    double* imag_residue_dev);
/* nfields independent applies ops[i](u[i]) -> out[i] (device pointers); all ops
 * must share one grid and one M. */
int fw_apply_batch_device(fw_op const* ops, int nfields, const double* const* u_dev,
                          double* const* out_dev);

/* ---- fused viscoacoustic stepper (SeismicStepper) ----
 * gamma, c0: N doubles (gamma in [0, 0.5)); derive_medium is evaluated on the
 * host with the reference formulas (seismic.cpp:30-39), both operators built
 * with their own s0.  phi, psi: initial field and velocity. */
int fw_seis_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                   const double* gamma, const double* c0, double omega0, int M,
                   const double* phi, const double* psi, double tau, double blowup_factor,
                   fw_seis* out);
void fw_seis_destroy(fw_seis s);
/* nsteps calls of step().  Blow-up is detected on the device; on FW_E_BLOWUP
 * the state is the one before the offending step and n() is the offending step
 * (as after the reference's throw, seismic.cpp:124-129). */
int fw_seis_step(fw_seis s, int nsteps);
/* enqueue nsteps without checking for blow-up (the check happens at the next
 * fw_seis_step / fw_seis_get); for timing loops. */
int fw_seis_enqueue(fw_seis s, int nsteps);
/* current() -> cur_host (N), optional prev / atten_prev, n */
int fw_seis_get(fw_seis s, double* cur_host, double* prev_host, double* atten_prev_host,
                long* n);
/* overwrite the current wavefield from host memory (host-owned state between
 * steps: source injection / receivers), then the caller steps on. */
int fw_seis_set_current(fw_seis s, const double* cur_host);
/* set_current + step(nsteps) + current() in one call with one host synchronisation
 * (both host buffers nullable, may alias; pinned memory for full PCIe speed).  On
 * FW_E_BLOWUP cur_out_host holds the pre-step state, as fw_seis_get would return. */
int fw_seis_step_io(fw_seis s, const double* cur_in_host, int nsteps, double* cur_out_host);
/* The two halves of fw_seis_step_io for pipelines of independent steppers (e.g. the shots of a
 * survey, one fw_ctx = one stream each): _async enqueues the upload, the steps and the download on
 * the stepper's context stream and returns without a host synchronisation; fw_seis_wait is the
 * synchronisation and the blow-up check of everything enqueued so far (on FW_E_BLOWUP the pending
 * cur_out_host is rewritten with the pre-step state).  The host buffers must stay valid until
 * fw_seis_wait; with pinned buffers the copies of one stepper run under the steps of another. */
int fw_seis_step_io_async(fw_seis s, const double* cur_in_host, int nsteps, double* cur_out_host);
int fw_seis_wait(fw_seis s);
/* device pointer of the current wavefield (valid until the next step) */
const double* fw_seis_current_device(fw_seis s);
/* the two operators, for diagnostics */
int fw_seis_ops(fw_seis s, fw_op* disp, fw_op* atten);
int fw_seis_medium(fw_seis s, double* c, double* eta, double* tau_coef);

/* ---- TSFP2 time-splitting stepper (Stepper, Method::TSFP2) ----
 * f: 0 = none, 1 = cubic u^3.  blowup_factor: StepperConfig::blowup_factor (threshold =
 * factor * max(sup|phi|, 1e-300), stepping.cpp:121).  fw_tsfp2_step(t, k) runs k steps and
 * stops at the first one whose sup|u| exceeds the threshold: FW_E_BLOWUP, n = that step,
 * (u, v) = the state right after it (the reference's throw from step_tsfp2, stepping.cpp:302-303). */
int fw_tsfp2_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                    const double* order_values, int M, double kappa, int f_kind,
                    const double* phi, const double* psi, double tau, double blowup_factor,
                    fw_tsfp2* out);
void fw_tsfp2_destroy(fw_tsfp2 t);
int fw_tsfp2_step(fw_tsfp2 t, int nsteps);
int fw_tsfp2_get(fw_tsfp2 t, double* u_host, double* v_host, long* n);

/* ---- two-level integrators (Stepper, Method::LFFP = 0 / Method::CNFP = 1) ----
 * u_tt = -kappa (-Delta)^{s(x)} u + f(u), f: 0 = none, 1 = cubic u^3.  The constructor
 * takes the Taylor start u^0 = phi, u^1 = phi + tau psi + tau^2/2 (-kappa L phi + f(phi))
 * (n = 1).  StepperConfig fields as in stepping.hpp:39-48 (use_dense is not offered: the
 * dense operator is out of scope).  State and every CG / Picard vector stay on the device;
 * the operator is the hot-path apply.  step: FW_E_BLOWUP (n incremented, state = the
 * pre-step levels, as the reference), FW_E_CG_STAGNATED, FW_E_PICARD_DIVERGED. */
int fw_wave_create(fw_ctx ctx, int method, int dim, const int* J, const double* lo, const double* hi,
                   const double* order_values, int M, double kappa, int f_kind, const double* phi,
                   const double* psi, double tau, double picard_tol, int picard_max_iters,
                   double inner_cg_tol, int cg_max_iters, double blowup_factor, fw_wave* out);
void fw_wave_destroy(fw_wave w);
int fw_wave_step(fw_wave w, int nsteps);
/* cur = u^n, prev = u^{n-1} (host, nullable); n; total Picard iterations (CNFP) */
int fw_wave_get(fw_wave w, double* cur_host, double* prev_host, long* n, long* picard_total);

/* ---- spectral utilities of the reference's Grid and the constant-order operator ----
 * Every even axis length the reference Grid accepts up to the device transforms' reach: powers of
 * two <= 4096 by the canonical Stockham plan, other lengths <= 2048 by Bluestein's chirp-z form
 * through it (FW_E_UNSUPPORTED beyond).  Spectra are full (N complex, interleaved re, im),
 * row-major, standard FFT order (grid.hpp:16-19).
 *   fw_grid_dft            in-place unnormalised C2C of data[2N] (sign -1 = FFTW_FORWARD, +1 = FFTW_BACKWARD)
 *   fw_grid_forward        spec = DFT(u) / N                                  (Grid::forward)
 *   fw_grid_inverse        u = Re IDFT(spec), *imag_residue = max |Im|         (Grid::inverse)
 *   fw_apply_constant_order  u -> (-Delta)^s u = inverse(|mu|^{2s} .* forward(u)); s in (0, 2)
 *                          else FW_E_ORDER_RANGE (flap.cpp:13-16, 146-149)
 *   fw_apply_constant_order_spectrum  spec .* |mu|^{2s}                        (flap.cpp:137-145) */
int fw_grid_dft(fw_ctx ctx, int dim, const int* J, double* data_host, int sign);
int fw_grid_dft_device(fw_ctx ctx, int dim, const int* J, double* data_dev, int sign);
int fw_grid_forward(fw_ctx ctx, int dim, const int* J, const double* u_host, double* spec_host);
int fw_grid_inverse(fw_ctx ctx, int dim, const int* J, const double* spec_host, double* u_host,
                    double* imag_residue);
int fw_apply_constant_order(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                            const double* u_host, double s, double* out_host, double* imag_residue);
int fw_apply_constant_order_spectrum(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                                     const double* spec_host, double s, double* out_host);

/* ---- the dense verification operator and the Toeplitz fast path (flap.hpp:43-58) ----
 *   fw_dense_create   assemble_dense(OrderField(grid, s), memory_budget) (flap.cpp:170-230): row j is
 *                     the inverse DFT of |mu|^{2 s(x_j)} at the periodic shifts, assembled on the device
 *                     (batched row DFTs) and kept there; FW_E_MEMORY_BUDGET when N^2 x 8 >= budget
 *                     (MemoryBudgetExceeded's message), order validation as OrderField
 *   fw_dense_apply    apply_dense (flap.cpp:233-243): out = A u (one warp per row, tree-ordered sums)
 *   fw_dense_entries  the N x N row-major entries (DenseOperator::entries)
 *   fw_apply_toeplitz apply_toeplitz (flap.cpp:245-285): constant order (else FW_E_NOT_CONSTANT),
 *                     1D (else FW_E_DIM_UNSUPPORTED), circulant embedding at 2J through device DFTs
 * The reference's tolerances apply (its dense checks are 1e-10 .. 1e-12 relative): the symbol
 * |mu|^{2s} of the dense rows is evaluated by the device pow. */
int fw_dense_create(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                    const double* order_values, unsigned long long memory_budget, fw_dense* out);
void fw_dense_destroy(fw_dense d);
int fw_dense_apply(fw_dense d, const double* u_host, double* out_host);
int fw_dense_entries(fw_dense d, double* entries_host);
int fw_apply_toeplitz(fw_ctx ctx, int dim, const int* J, const double* lo, const double* hi,
                      const double* order_values, const double* u_host, double* out_host);
/* truncation_indicator(M, |mu|, s0) (flap.cpp:287-294): |mu|^{2 s0} (2 ln|mu|)^M / M!, the magnitude of
 * the first dropped expansion term (host, the reference's operation order); FW_E_NONPOSITIVE_FREQ
 * unless |mu| > 0 */
int fw_truncation_indicator(int M, double mu_abs, double s0, double* out);

/* ---- canonical transforms (test hooks) ----
 * forward: real x[N] -> half spectrum H[N_half] (interleaved re,im), unscaled;
 * backward: H -> real x (unnormalized C2R). */
int fw_rfftn(fw_ctx ctx, int dim, const int* J, const double* x_host, double* H_host);
int fw_irfftn(fw_ctx ctx, int dim, const int* J, const double* H_host, double* x_host);

/* ---- stage entry points (device pointers, enqueued on the ctx stream) ----
 * The single-device pipeline's kernels applied to caller-provided sub-arrays, for
 * distributed orchestration (slab decomposition: paper_2311_13049_b200/slab.py).
 * Arrays are real [J0]..[J_{d-1}] / Hermitian-half [J0]..[J_{d-1}/2+1] (interleaved).
 *   fw_stage_r2c       R2C along the last axis (x scale when scale != 1)
 *   fw_stage_c2c       C2C along axis (< d-1) for nterms terms (src/dst/w advance by their
 *                      term strides, in complex / real elements); w (nullable) multiplies
 *                      the source element-wise; x scale when != 1
 *   fw_stage_c2r_accum per row: out = sum_{m=m_first}^{m_last} (s-s0)^m .* C2R(src_m),
 *                      ascending m, (s-s0)^m regenerated from dev1 = s - s0
 *   fw_op_device_tables  the operator's resident tables: w[(M+1)][N_half], dev1[N]
 *   fw_stage_c2c_scatter  fw_stage_c2c with the slab transpose FUSED into its last pass:
 *                      output element j of line (o, in) of term t goes to
 *                      dst_q[j / blk][t*tstride + (j % blk)*jstride + o*ostride + in + base]
 *                      (complex elements), i.e. straight into the destination ranks'
 *                      receive buffers (peer memory mapped on this device: NVLink stores),
 *                      no separate all-to-all; nq <= 8, axis length 256 / 512 / 1024
 *                      (else FW_E_UNSUPPORTED).  Replaces the copy + all-to-all the
 *                      reference's FFTW path has no equivalent of (grid.cpp:134-137 is serial). */
int fw_stage_r2c(fw_ctx ctx, int dim, const int* J, const double* x_dev, double* H_dev, double scale);
int fw_stage_c2c(fw_ctx ctx, int dim, const int* J, int axis, int dir, const double* src_dev, double* dst_dev,
                 const double* w_dev, long long src_ts, long long dst_ts, long long w_ts, int nterms, double scale);
int fw_stage_c2r_accum(fw_ctx ctx, int dim, const int* J, const double* src_dev, long long src_ts, int m_first,
                       int m_last, const double* dev1_dev, double* out_dev, double* residue_dev);
int fw_op_device_tables(fw_op op, const double** w_dev, const double** dev1_dev, int* m_last);
/* one rank's operator tables of a slab-decomposed 3D grid J (axis 0 split over P ranks):
 * w [M+1][J0][J1/P][J2/2+1] on the rank's spectral columns, s - s0 [J0/P][J1][J2] on its planes;
 * s0 and the OrderField checks from the GLOBAL order values (N doubles), so the tables equal the
 * single-device operator's slices bit for bit.  Resident table bytes fall as 1/P (fw_op_info).
 * The op serves the stage entry points only (fw_apply on it: FW_E_ARG). */
int fw_op_create_slab(fw_ctx ctx, const int* J, const double* lo, const double* hi, const double* order_values,
                      const double* s0_override, int M, int P, int rank, fw_op* out);
/* the slab stepper's update (seismic.cpp:116-129) on a rank's planes with the state levels kept:
 * next and l2out (the new L2prev = l2) are written unless *flag_dev already holds a step (a blow-up
 * on some rank in an earlier step: every later update is frozen so the levels before the offending
 * step survive); a blow-up mins `step` into *flag_dev and into every peer's flag (npeers <= 8 device
 * addresses valid on this device, peer memory through fw_ipc_open), so after the next barrier all
 * ranks agree without a collective. */
int fw_stage_seis_update_peers(fw_ctx ctx, long long n, double tau, const double* cur, const double* prev,
                               const double* l2prev, const double* l1, const double* l2, const double* c,
                               const double* eta, const double* tau_coef, double* next, double* l2out, double thr,
                               int step, int* flag_dev, int npeers, int* const* peer_flags_dev);
/* distributed seismic stepper pieces (slab.SlabSeismicStepper), element-wise on a slab:
 *   fw_medium_coefficients  host: c, eta, tau_c from gamma, c0 (derive_medium, seismic.cpp:30-39; glibc
 *                           pow/cos/sin exactly as the reference), FW_E_GAMMA_RANGE outside [0, 0.5)
 *   fw_stage_seis_start     cur = phi + tau psi + tau^2/2 c^2 (eta L1phi + tau_c L2psi)   (seismic.cpp:100-106)
 *   fw_stage_seis_update    next = 2 cur - prev + tau^2 c^2 (eta L1 + tau_c (L2 - L2prev)/tau)
 *                           (seismic.cpp:116-122); *flag_dev = min(*flag_dev, step) when
 *                           |next| > thr somewhere (the blow-up check of seismic.cpp:124-129) */
int fw_medium_coefficients(long long n, const double* gamma, const double* c0, double omega0, double* c_out,
                           double* eta_out, double* tau_coef_out);
/* ricker_initial(nu0, xc, grid) (seismic.cpp:70-83): out[j] = (1 - 2 a r^2) exp(-a r^2), a = pi^2 nu0^2,
 * r = |x_j - xc| with x_j = Grid::point(j) (grid.cpp:107-116); host, glibc exp as the reference
 * (bit-identical); grid validation as Grid::Grid (FW_E_ODD_SIZE, FW_E_EMPTY_INTERVAL, FW_E_DIM_RANGE) */
int fw_ricker_initial(int dim, const int* J, const double* lo, const double* hi, double nu0, const double* xc,
                      double* out);
int fw_stage_seis_start(fw_ctx ctx, long long n, double tau, const double* phi, const double* psi, const double* c,
                        const double* eta, const double* tau_coef, const double* l1phi, const double* l2psi,
                        double* cur);
int fw_stage_seis_update(fw_ctx ctx, long long n, double tau, const double* cur, const double* prev,
                         const double* l2prev, const double* l1, const double* l2, const double* c, const double* eta,
                         const double* tau_coef, double* next, double thr, int step, int* flag_dev);
/* CUDA IPC helpers for the fused-transpose slab path (one process per GPU of a node):
 * export a device allocation, map a peer's allocation into this device's address space */
/* fw_ipc_alloc / fw_ipc_free: plain device allocations for exported buffers (a handle maps the
 * allocation base: fw_ipc_handle refuses interior pointers with FW_E_ARG) */
int fw_ipc_alloc(fw_ctx ctx, size_t bytes, void** dev_ptr_out);
int fw_ipc_free(fw_ctx ctx, void* dev_ptr);
int fw_ipc_handle(const void* dev_ptr, unsigned char handle_out[64]);
int fw_ipc_open(const unsigned char handle[64], void** dev_ptr_out);
int fw_ipc_close(void* dev_ptr);
int fw_stage_c2c_scatter(fw_ctx ctx, int dim, const int* J, int axis, int dir, const double* src_dev,
                         const double* w_dev, long long src_ts, long long w_ts, int nterms, double scale, int nq,
                         double* const* dst_q, long long blk, long long jstride, long long ostride,
                         long long tstride, long long base);

/* ---- the slab-decomposed SeismicStepper for C / C++ hosts (one process per GPU) ----
 * SeismicStepper (seismic.hpp:36-46, seismic.cpp:85-142) on a 3D grid whose axis 0 is split over
 * P <= 8 ranks: rank r owns planes [r J0/P, (r+1) J0/P) and only its slab of both operators'
 * tables (fw_op_create_slab).  Transposes: the last FFT pass of each stage stores into the owning
 * rank's buffer (CUDA IPC peer memory over NVLink); the NCCL communicator (fw_nccl_unique_id on
 * rank 0, the id handed to every rank by the host) exchanges the IPC handles once and is the
 * stream-ordered barrier between the phases.  gamma, c0, phi, psi are the GLOBAL fields (N
 * doubles; every rank passes the same arrays).  fw_slab_seis_step(s, k) runs k steps and reads
 * the blow-up flag once: FW_E_BLOWUP with n = the offending step and the pre-step state, as the
 * reference's throw (seismic.cpp:124-129).  fw_slab_seis_get returns this rank's planes
 * ([J0/P][J1][J2]).  FW_E_NCCL when P > 1 and libnccl.so.2 cannot be loaded. */
int fw_nccl_unique_id(unsigned char id_out[128]);
int fw_slab_seis_create(fw_ctx ctx, const unsigned char nccl_id[128], int P, int rank, const int* J, const double* lo,
                        const double* hi, const double* gamma, const double* c0, double omega0, int M,
                        const double* phi, const double* psi, double tau, double blowup_factor, fw_slab_seis* out);
void fw_slab_seis_destroy(fw_slab_seis s);
int fw_slab_seis_step(fw_slab_seis s, int nsteps);
int fw_slab_seis_get(fw_slab_seis s, double* cur_host, double* prev_host, double* atten_prev_host, long* n);
int fw_slab_seis_info(fw_slab_seis s, size_t* table_bytes, int* P, int* rank);

#ifdef __cplusplus
}
#endif

#endif
