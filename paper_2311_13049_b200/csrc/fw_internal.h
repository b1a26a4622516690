// fw_internal.h — launch interface between the C-ABI (fw_capi.cu) and the
// sm_100a kernels (fw_kernels.cu).  Internal; not part of the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include <atomic>
#include <vector>

namespace fw {

// Kernel attributes (cudaFuncSetAttribute) are per device: run `f` once for every device
// that becomes current here (a repeat by a racing thread is harmless).
template <class F>
inline void once_per_device(std::atomic<unsigned long long>& done, F f) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_release);
}

struct GridGeom {
  int d = 0;
  int J[3] = {1, 1, 1};
  size_t N = 0;      // real points
  size_t Nh = 0;     // Hermitian half-spectrum bins: rows * (J[d-1]/2 + 1)
  size_t rows = 0;   // N / J[d-1]
  int nl = 0;        // last-axis length
  int hp1 = 0;       // nl/2 + 1
};

struct LaunchCtx {
  cudaStream_t stream = nullptr;
  const double2* master = nullptr;  // master twiddle table (kTwMaster entries)
  long long* launches = nullptr;    // host-side launch counter
  bool generic_lines = false;       // FW_GENERIC_LINES=1: shared-memory line FFTs only (tests)
};

// every rank's blow-up flag (device addresses valid on this device: local or peer memory)
constexpr int kMaxPeers = 8;
struct PeerFlags {
  int n = 0;
  int* f[kMaxPeers] = {};
};
void launch_seis_update_peers(const LaunchCtx& L, size_t N, double tau, const double* cur, const double* prev,
                              const double* ap, const double* l1, const double* l2, const double* c, const double* eta,
                              const double* tc, double* next, double* l2out, double thr, int step, int* flag,
                              const PeerFlags& peers);

// every line of length n (power of two <= 4096) along a strided axis of a complex array, in
// place: element j of line (o, in) at o n S + j S + in (in < S); canonical plan; x sc if scale
void launch_c2c_lines(const LaunchCtx& L, int n, long long S, long long outer, int dir, double2* x, double sc,
                      bool scale);

// ---- general-length complex DFTs (fw_dft.cu): Grid::dft of any supported axis lengths
constexpr int kMaxBluestein = 2048;  // non-power-of-two axes: chirp-z through a pow2 FFT of <= 4096
bool dft_length_supported(int n);
struct ChirpCache {  // per (length, sign): chirp w_j and the transformed filter, device-resident
  struct Entry {
    int n = 0, sign = 0, m = 0;
    double2* w = nullptr;
    double2* bhat = nullptr;
  };
  std::vector<Entry> entries;
  cudaError_t get(const LaunchCtx& L, int n, int sign, const Entry** out);
  void release();
};
// in place, unnormalised C2C over every axis of x[J0]..[J_{d-1}] (sign -1 forward, +1 backward)
cudaError_t launch_dft(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, int sign, double2* x);
// uh = DFT(u) (x 1/N when scale): Grid::forward / flap.cpp:46-50 in the C2C form
cudaError_t launch_full_forward(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long N,
                                const double* u, double2* uh, bool scale);
// flap.cpp:52-91 in the C2C form: out = sum_m (s-s0)^m Re IDFT(w_m .* uh), ascending m from 0
struct FullApplyArgs {
  const double2* uh;
  const double* w;     // (M+1) x N weights on the full spectrum
  const double* dev1;  // s - s0
  double* devm;        // scratch N: (s-s0)^m by the reference recurrence
  double2* buf;        // scratch N complex
  double* out;
  int m_first, m_last;
  double* residue;
  const int* guard;
};
cudaError_t launch_full_apply(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long N,
                              const FullApplyArgs& a);
cudaError_t launch_real_part(const LaunchCtx& L, long long N, const double2* x, double* out, double* residue);
// the same over `batch` consecutive arrays (an extra outermost axis that is not transformed)
cudaError_t launch_dft_batched(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long batch, int sign,
                               double2* x);
// dense operator entries A[N][N] (flap.cpp:170-230), rows in batches through scratch G (rows x N complex)
cudaError_t launch_dense_assemble(const LaunchCtx& L, ChirpCache& chirps, int d, const int* J, long long N,
                                  const double* mu2, const double* s, double2* G, long long rows_per_batch,
                                  double* A);
cudaError_t launch_dense_matvec(const LaunchCtx& L, long long N, const double* A, const double* u, double* out);
// apply_toeplitz (flap.cpp:245-285): t (J complex, in: |mu|^{2s}, overwritten), c / x scratch 2J complex
cudaError_t launch_toeplitz(const LaunchCtx& L, ChirpCache& chirps, int J, double2* t, const double* u, double2* c,
                            double2* x, double* out);
cudaError_t launch_spectrum_mul(const LaunchCtx& L, long long n, const double* f, double2* x);

// u (N reals) -> Uh (Nh bins), scaled by 1/N (flap.cpp:46-50)
void launch_forward(const LaunchCtx& L, const GridGeom& g, const double* u, double2* Uh, bool scale);

// Inverse + recombination of one operator (flap.cpp:52-91):
//   out = sum_{m=m_first}^{m_last} dev_m .* Re IFFT(w_m .* Uh)  (ascending m)
// w: (M+1) x Nh weights (w_0 = base symbol), dev1: s - s0 (N),
// T: scratch (m_last-m_first+1) x Nh bins (d >= 2 only),
// residue (nullable): max-accumulated max|Im|, guard (nullable): if *guard != kNoBlowup the
// kernels writing `out` are no-ops.
struct InverseArgs {
  const double2* Uh;
  const double* w;
  const double* dev1;
  double2* T;
  double* out;
  int m_first, m_last;
  double* residue;
  const int* guard;
};
void launch_inverse(const LaunchCtx& L, const GridGeom& g, const InverseArgs& a);
// Row stride (complex elements) of the term scratch T the inverse pipelines write between the
// axes, and its elements per term.  2D grids served by the register-resident line kernels pad
// the rows of T from J1/2 + 1 (odd) to a multiple of 8 elements, so that the strided 128-B runs
// of the axis-0 pass and the rows the C2R fetches are 128-B aligned; everything else keeps the
// Spectrum layout.
#ifndef FW_TERM_PAD
#define FW_TERM_PAD 1  // 2D term scratch rows padded to 128 B (0: Spectrum layout; A/B)
#endif
// (nterms: terms of the launch; a single term takes the one-term line kernel, which keeps the
// Spectrum layout.  term_elems = the allocation per term, an upper bound for every launch.)
long long term_row_stride(const LaunchCtx& L, const GridGeom& g, int nterms);
inline size_t term_elems(const LaunchCtx& L, const GridGeom& g) { return g.rows * (size_t)term_row_stride(L, g, 2); }
// true when the register-resident kernels serve every pass of the grid's inverse, i.e. the row
// C2R can resume a recombination from the partial sums of earlier term chunks
bool rows_resumable(const LaunchCtx& L, const GridGeom& g);

constexpr int kNoBlowup = 0x7fffffff;

// tables: w[m][k] = base[k] * lw_m[k] with the reference recurrences (flap.cpp:108-122)
void launch_build_weights(const LaunchCtx& L, size_t Nh, int M, const double* mu2h, const double* base,
                          const double* logm, double* w);
// w[m][k] = base[k] * lw[m-1][k] from uploaded half log-weight rows
void launch_weights_from_lw(const LaunchCtx& L, size_t Nh, int M, const double* base, const double* lw,
                            double* w);
// dev1[j] = s[j] - s0
void launch_dev1(const LaunchCtx& L, size_t N, const double* s, double s0, double* dev1);

// seismic Taylor start (seismic.cpp:100-106)
void launch_seis_start(const LaunchCtx& L, size_t N, double tau, const double* phi, const double* psi,
                       const double* c, const double* eta, const double* tc, const double* l1phi,
                       const double* l2psi, double* cur);
// seismic update (seismic.cpp:116-129); sets *flag = min(*flag, step) when |next| > thr
void launch_seis_update(const LaunchCtx& L, size_t N, double tau, const double* cur, const double* prev,
                        const double* ap, const double* l1, const double* l2, const double* c,
                        const double* eta, const double* tc, double* next, double thr, int step, int* flag);

// TSFP2 pieces (stepping.cpp:106-117, 271-300)
void launch_osc_rotate(const LaunchCtx& L, size_t Nh, const double* w, const double* cw, const double* sw, double dt,
                       double2* uh, double2* vh);
// raise the dynamic shared-memory limit of the FFT kernels on the current device
void init_kernels();
void launch_tsfp2_kick(const LaunchCtx& L, size_t N, double tau, double kappa, int cubic, const double* u,
                       const double* pert, double* v, const int* guard = nullptr);
// unscaled inverse of one spectrum to reals (C2C axes 0..d-2 + C2R), in place on H
// guard (nullable): the final write of x is skipped when *guard != kNoBlowup (a blow-up was
// flagged earlier in the same multi-step enqueue: the state stays at the offending step)
void launch_irfft(const LaunchCtx& L, const GridGeom& g, double2* H, double* x, const int* guard = nullptr);
void launch_sup_check(const LaunchCtx& L, size_t N, const double* u, double thr, int step, int* flag);

// two-level integrators LFFP / CNFP (stepping.cpp:88-104, 170-264), fw_wave.cu
size_t wave_partials();
void launch_wave_start(const LaunchCtx& L, size_t N, double tau, double kappa, int cubic, const double* phi,
                       const double* psi, const double* lphi, double* u1);
void launch_lffp_update(const LaunchCtx& L, size_t N, double t2, double kappa, int cubic, const double* cur,
                        const double* prev, const double* lu, double* next, const int* flag);
void launch_cnfp_rhs0(const LaunchCtx& L, size_t N, double t2, double alpha, int cubic, const double* cur,
                      const double* prev, const double* lprev, double* rhs0);
void launch_cnfp_rhs(const LaunchCtx& L, size_t N, double t2, const double* rhs0, const double* w, double* rhs);
void launch_cg_apply_a(const LaunchCtx& L, size_t N, double alpha, const double* w, const double* lw,
                       const double* rhs, double* out);
void launch_cg_step(const LaunchCtx& L, size_t N, double a, const double* p, const double* ap, double* x, double* r);
void launch_cg_dir(const LaunchCtx& L, size_t N, double beta, const double* r, double* p);
// *out = sum a*b (mode 0) or sum (a-b)^2 (mode 1), deterministic order; partial: wave_partials() doubles
void launch_dot(const LaunchCtx& L, size_t N, int mode, const double* a, const double* b, double* partial,
                double* out);

// batched multi-field pipeline (many independent fields of one grid, e.g. configs[4]):
// per-field pointers of one kernel launch, indexed by blockIdx.z
struct BatchLine {
  const void* src;
  void* dst;
  const double* w;    // weights (already offset to the launch's first term)
  const double* aux;  // dev1 for the C2R recombination
  double* out;
};
// forward for F fields: tab[f] = {u_f, Uh_f}; tab is a DEVICE array of F entries
void launch_forward_batch(const LaunchCtx& L, const GridGeom& g, int F, const BatchLine* tab_r2c,
                          const BatchLine* tab_c2c, bool scale);
// inverse + recombination for F fields of one grid and term range:
// tab0[f] = {Uh_f, T_f, w_f + m_first Nh}, tab1[f] = {T_f, T_f} (axes 1..d-2), tab2[f] = {T_f, -, -, dev1_f, out_f}
// (resume: the terms before m_first were recombined into out_f by an earlier launch -- term
// chunks sized so that a chunk's spectra stay in L2 between the two kernels)
void launch_inverse_batch(const LaunchCtx& L, const GridGeom& g, int F, int m_first, int m_last,
                          const BatchLine* tab0, const BatchLine* tab1, const BatchLine* tab2,
                          const int* guard = nullptr, bool resume = false);

// fused transpose: the last pass of a line C2C writes output element j of line (o, in), term t
// to dst[q] + t tstride + (j - q blk) jstride + o ostride + in + base, q = j / blk -- the
// destination ranks' buffers (peer memory over NVLink), or local buffers (nq = 1 / tests)
constexpr int kMaxScatter = 8;
struct Scatter {
  double2* dst[kMaxScatter];
  long long blk, jstride, ostride, tstride, base;
  int nq;
  int lgblk;  // log2(blk) when blk is a power of two (32-bit shift / mask in the epilogue), else -1
};

// register-resident line FFTs (fw_lines.cu) for n in {256, 512, 1024}; false = not served
// (Sd: stride of the destination along the axis when it differs from the source's S -- the
// all-terms inverse of a 2D grid writes term spectra whose rows are padded to 128 B; 0 = S)
bool launch_lines(const LaunchCtx& L, int n, int dir, const double2* src, double2* dst, const double* w,
                  long long S, long long outer, long long inner, long long src_ts, long long dst_ts, long long w_ts,
                  int nterms, int nfields, double sc, bool scale, const BatchLine* bl,
                  const Scatter* scatter = nullptr, long long Sd = 0);

// register-resident row R2C (fw_lines.cu) for nl in {256, 512, 1024}
bool launch_rows_r2c(const LaunchCtx& L, int nl, const double* u, double2* Uh, long long rows, int nfields,
                     double sc, bool scale, const BatchLine* bl);
// register-resident row C2R + ascending-m recombination (fw_lines.cu) for nl in {256, 512, 1024}
// (xrs: row stride of src in complex elements, 0 = nl/2 + 1)
bool launch_rows_c2r(const LaunchCtx& L, int nl, const double2* src, long long src_ts, int m_first, int m_last,
                     const double* dev1, double* out, long long rows, int nfields, double* residue, const int* guard,
                     const BatchLine* bl, long long xrs = 0, int resume = 0);

// stage entry points (distributed orchestration on local sub-arrays)
void launch_stage_r2c(const LaunchCtx& L, const GridGeom& g, const double* u, double2* H, double scale, bool do_scale);
void launch_stage_c2c(const LaunchCtx& L, const GridGeom& g, int axis, int dir, const double2* src, double2* dst,
                      const double* w, long long src_ts, long long dst_ts, long long w_ts, int nterms, double scale,
                      bool do_scale);
void launch_stage_c2r(const LaunchCtx& L, const GridGeom& g, const double2* src, long long src_ts, int m_first,
                      int m_last, const double* dev1, double* out, double* residue);

}  // namespace fw
