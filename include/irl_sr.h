/*
 * irl_sr.h — C-ABI of the B200 (sm_100a) IRL stochastic-reconfiguration hot path.
 *
 * Drop-in boundary for the reference package `irlnqs` (arXiv 2601.01437,
 * /root/reference/pkg/src/irlnqs).  Every entry point replaces one reference
 * function on the hot path; the reference-side binding (ctypes) is shown in
 * INTEGRATION.md and implemented in paper_2601_01437_b200/_lib.py.
 *
 * Conventions:
 *   - all array pointers are DEVICE pointers owned by the caller; kernels never
 *     allocate, free or retain them past the call; inputs are const;
 *   - `stream` is a cudaStream_t passed as void* (the caller's current stream);
 *     every call is asynchronous on that stream and re-entrant;
 *   - O is row-major N x ld (ld >= P, from irl_padded_ld), padding columns zero;
 *     f64: ld doubles per row; c128: ld interleaved complex (re, im) per row;
 *   - P-length vectors are allocated with the padded length ld, padding zero;
 *   - complex vectors passed as *_re / *_im are PLANAR arrays of length ld;
 *     a NULL *_im means "imaginary part zero" (input) or "not wanted" (output);
 *   - workspace is caller-allocated, >= the matching *_workspace_bytes(), 256-B aligned;
 *   - return value: IRL_OK or an IRL_ERR_* code; irl_last_error() gives text
 *     (thread-local).  No exception or exit() crosses the ABI.
 */
#ifndef IRL_SR_H_
#define IRL_SR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define IRL_OK 0
#define IRL_ERR_ARG 1       /* bad shape / null pointer / bad mode */
#define IRL_ERR_ALIGN 2     /* pointer or ld not 16-byte aligned / padded */
#define IRL_ERR_WORKSPACE 3 /* workspace too small */
#define IRL_ERR_CUDA 4      /* CUDA runtime error (text in irl_last_error) */
#define IRL_ERR_DEVICE 5    /* no sm_100 device / unsupported plan */

#define IRL_MVP_AUTO 0      /* fused single pass when it fits, else two-pass */
#define IRL_MVP_FUSED 1     /* one HBM pass, column slices over a CTA cluster (DSMEM exchange) */
#define IRL_MVP_TWO_PASS 2  /* t = O v pass, then O^H y pass */
#define IRL_MVP_ROWS 3      /* one HBM pass, a warp per row (narrow rows: ld <= 512 16-byte units) */
#define IRL_MVP_WIDE 4      /* one HBM pass, persistent column-sliced grid, stages resident until their accumulate (very wide rows) */

#define IRL_MODEL_RBM 0
#define IRL_MODEL_MLP 1

/* Library identity / diagnostics. */
int irl_version(void);
const char* irl_last_error(void);

/* Development only: copies up to `bytes` of the wide-path trace (per-CTA,
 * per-block %globaltimer stamps recorded when IRL_WIDE_TRACE is set) to host
 * memory; returns the bytes copied (0 when tracing is off). */
size_t irl_debug_wide_trace(void* host, size_t bytes);

/* Padded leading dimension (in elements: doubles for f64, complex for c128) for
 * P parameters.  Rows are padded to whole 16-B units and to a multiple of 16
 * (64 for very wide rows) units so every column split is TMA-aligned. */
int64_t irl_padded_ld(int64_t p, int is_complex);

/* ---------------------------------------------------------------- A3 ----
 * estimate_energy (estimators.py:146-153) + centred coefficients (:166-168).
 * stats3 (device, 3 doubles) = {E = Re sum w e, Im sum w e, sum w |e - E|^2};
 * coeff[n] = w_n (e_n - E)  (c128 hermitian=1: w_n Re(e_n - E), imag 0).   */
int irl_energy_f64(const double* w, const double* e, int64_t n, double* stats3, double* coeff, void* stream);
int irl_energy_c128(const double* w, const double* e, int64_t n, int hermitian, double* stats3, double* coeff,
                    void* stream);

/* ------------------------------------------------------------- A4/A5 ----
 * Column statistics of a stored O: obar = w @ O (estimators.py:167) and
 * g = coeff @ conj(O)  (so F = 2 Re g reproduces energy_gradient, :156-163). */
size_t irl_colstats_workspace_bytes(int64_t n, int64_t ld, int is_complex);
int irl_colstats_f64(const double* O, int64_t n, int64_t ld, const double* w, const double* coeff, double* obar,
                     double* g, void* ws, size_t ws_bytes, void* stream);
int irl_colstats_c128(const double* O, int64_t n, int64_t ld, const double* w, const double* coeff, double* obar,
                      double* g, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- A2 ----
 * Batched log-derivative rows (role of ansatz.log_derivative, ansatz.py:249-290,
 * called per sample by build_batch, estimators.py:112-126) for the shallow NQS,
 * with the column statistics of A4/A5 fused into the same pass.
 *   x     : N x n_vis uint8 (0/1)
 *   theta : RBM [a (n), b (h), W (h x n)]  (c128: interleaved complex)
 *           MLP [W (h x n_in), b (h), u (h), c]
 *   hidden-unit activations are also returned: t (N x h, S-typed) and, MLP only,
 *   g = u (1 - t^2) (N x h f64), inside the workspace (see irl_hidden_*). */
size_t irl_obuild_workspace_bytes(int model, int64_t n, int n_vis, int hidden, int64_t ld, int is_complex);
int irl_obuild_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* O,
                       int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                       size_t ws_bytes, void* stream);
int irl_obuild_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* O,
                        int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                        size_t ws_bytes, void* stream);
int irl_obuild_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, double* O,
                       int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                       size_t ws_bytes, void* stream);
/* Hidden layer only: t = tanh(b + W x) (N x h), and MLP g = u (1 - t^2). */
int irl_hidden_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* t,
                       void* stream);
int irl_hidden_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* t,
                        void* stream);
int irl_hidden_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, double* t,
                       double* g, void* stream);

/* ------------------------------------------------------- A6/A7/A10 ----
 * Matrix-free centred product (heff_matvec, estimators.py:171-186; dense_qgt's
 * matrix-free form, :335-344) with the optional bordered row/column of the
 * optimizer's closure (optimizer.py:140-148):
 *   out = O_c^H (coeff * (O_c v))  (+ u0 * half_f)          O_c = O - obar
 *   out0 = half_f . v   (real part of half_f^H v for c128)
 * coeff = w (e - E) gives H_eff v ; coeff = w gives S v.
 * half_f / u0 / out0 may be NULL (plain product).  u0, out0 are device scalars. */
size_t irl_mvp_workspace_bytes(int64_t n, int64_t ld, int is_complex);
int irl_mvp_f64(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff,
                const double* v, double* out, const double* half_f, const double* u0, double* out0, int mode,
                void* ws, size_t ws_bytes, void* stream);
int irl_mvp_c128(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff,
                 const double* v_re, const double* v_im, double* out_re, double* out_im, const double* hf_re,
                 const double* hf_im, const double* u0, double* out0, int mode, void* ws, size_t ws_bytes,
                 void* stream);
/* Two centred products for the same v over one read of O (the GEVP form
 * H_eff v = lambda S v, PAPER Eq. 11, applies dense_heff's and dense_qgt's
 * operators, estimators.py:319-344, to every iterate):
 *   out_a = O_c^H (coeff_a * (O_c v)) (+ u0 * half_f), out0 = half_f . v
 *   out_b = O_c^H (coeff_b * (O_c v))
 * Rows on the single-CTA fused path stream O once for both; narrow (ROWS),
 * clustered and very wide (WIDE) rows run the two products one after the other. */
size_t irl_mvp2_workspace_bytes(int64_t n, int64_t ld, int is_complex);
int irl_mvp2_f64(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff_a,
                 const double* coeff_b, const double* v, double* out_a, double* out_b, const double* half_f,
                 const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream);
int irl_mvp2_c128(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff_a,
                  const double* coeff_b, const double* v_re, const double* v_im, double* outa_re, double* outa_im,
                  double* outb_re, double* outb_im, const double* hf_re, const double* hf_im, const double* u0,
                  double* out0, void* ws, size_t ws_bytes, void* stream);
/* Which path (IRL_MVP_FUSED / IRL_MVP_TWO_PASS / IRL_MVP_ROWS / IRL_MVP_WIDE) AUTO takes, and its launch
 * geometry (cluster size, units per slice, threads, rows per stage, stages,
 * row blocks); for benches and tests.  Returns IRL_OK or an error. */
int irl_mvp_plan(int64_t n, int64_t ld, int is_complex, int mode, int* out_path, int* out_geom7);

/* --------------------------------------------------------- K6 (cfg5) ----
 * On-the-fly O regeneration for the shallow MLP: O is never stored.  The same
 * products (heff_matvec / S v, estimators.py:171-186, bordered opt:140-148)
 * and column statistics (estimators.py:156-168) are regenerated from the
 * bit-packed inputs and the hidden activations t, g (N x h f64) with FP64
 * tensor-core GEMMs.  x bits: N x 2 uint64 (n_in <= 100).  Vectors use the
 * padded MLP layout [W (h x n_in), b, u, c] of length ld = irl_padded_ld(P). */
size_t irl_otf_workspace_bytes(int64_t n, int n_in, int hidden);
int irl_otf_prepare_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, uint64_t* xbits,
                            double* t, double* g, void* stream);
int irl_otf_colstats_mlp_f64(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in, int hidden,
                             int64_t ld, const double* w, const double* coeff, double* obar, double* grad, void* ws,
                             size_t ws_bytes, void* stream);
/* RBM (real theta) on-the-fly mode, layout [a (n), b (h), W (h x n)]: the same
 * products and statistics regenerated from the packed inputs and t = tanh(b + W x). */
int irl_otf_prepare_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, uint64_t* xbits,
                            double* t, void* stream);
int irl_otf_colstats_rbm_f64(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                             const double* w, const double* coeff, double* obar, double* grad, void* ws,
                             size_t ws_bytes, void* stream);
int irl_otf_mvp_rbm_f64(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                        const double* obar, const double* coeff, const double* v, double* out, const double* half_f,
                        const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream);
int irl_otf_mvp_mlp_f64(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in, int hidden,
                        int64_t ld, const double* obar, const double* coeff, const double* v, double* out,
                        const double* half_f, const double* u0, double* out0, void* ws, size_t ws_bytes,
                        void* stream);
/* Same product with G = u (1 - t^2) formed inside the GEMM kernels from t and
 * the output weights u (length hidden) instead of read from a stored G: half
 * the activation traffic per product (the small-n_in products are HBM-bound on
 * t and g).  Same arguments as irl_otf_mvp_mlp_f64 with u in place of g. */
int irl_otf_mvp_mlp_u_f64(const uint64_t* xbits, const double* t, const double* u, int64_t n, int n_in, int hidden,
                          int64_t ld, const double* obar, const double* coeff, const double* v, double* out,
                          const double* half_f, const double* u0, double* out0, void* ws, size_t ws_bytes,
                          void* stream);
/* Complex-theta RBM on the fly (hermitian kind, cfg4): t = tanh(b + W x) complex
 * (N x h interleaved c128), vectors in the planar real embedding of irl_mvp_c128
 * (ld = irl_padded_ld(P, 1)); obar, coeff, grad interleaved c128.  Statistics:
 * obar = sum w O, grad = sum c conj(O) (estimators.py:156-168); product as
 * irl_mvp_c128 with a real coeff stored as c128. */
size_t irl_otf_workspace_bytes_c128(int64_t n, int n_vis, int hidden);
int irl_otf_prepare_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta,
                             uint64_t* xbits, double* t, void* stream);
int irl_otf_colstats_rbm_c128(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                              const double* w, const double* coeff, double* obar, double* grad, void* ws,
                              size_t ws_bytes, void* stream);
int irl_otf_mvp_rbm_c128(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                         const double* obar, const double* coeff, const double* v_re, const double* v_im,
                         double* out_re, double* out_im, const double* half_f_re, const double* half_f_im,
                         const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------ A13 / A16 ----
 * IRL driver helpers.
 * irl_lanczos_step_small: one Lanczos step (krylov.py:96-116) on device scalars
 * for short vectors (L <= 4096): given W = A v_j, writes alpha_j, beta_j into
 * ab[j], ab[m + j], reorthogonalises W twice against V rows 0..j (ldv stride)
 * and stores V[j+1] = W / beta_j.  Single CTA, graph-capturable.
 * irl_host_qr_sweeps: HOST function; nshift implicit-shift QR bulge chases
 * (krylov.py:165-190, as applied by implicit_restart :225-227) on the dense
 * row-major m x m tridiagonal T, accumulating Q (both in/out, host memory). */
int irl_lanczos_step_small(double* V, int64_t ldv, double* W, int64_t L, int j, int m, double* ab, void* stream);
/* The same step on one thread-block cluster (2..16 CTAs, DSMEM reductions) for
 * medium L; j + 1 <= 64. */
int irl_lanczos_step_cluster(double* V, int64_t ldv, double* W, int64_t L, int j, int m, double* ab, void* stream);
int irl_host_qr_sweeps(int m, double* T, double* Q, const double* shifts, int nshift);

/* ------------------------------------------------ §8(f) 1: completion ----
 * Connected (two-configuration) product: heff_matvec + heff_offdiag_matvec
 * (estimators.py:171-186 + :254-294, summed as the optimizer closure does,
 * optimizer.py:144-147), with the optional bordered row/column of irl_mvp_*:
 *   out = O_c^H (w corr + coeff (O_c v))        (real / raw complex: real part)
 *   corr_n = sum_{e in seg(dist_index[n])} pcoeff_e (q_part[partner_row_e] - q_n)
 *   q = O_c v,  q_part = (partner_O - obar) v
 * The cache arrays mirror ConnectedCache (estimators.py:189-218): dist_index
 * (N, int64) indexes the CSR segments indptr (n_dist + 1, int64); partner_row
 * (nnz, int64) indexes rows of partner_O (n_partner x ld, padded like O);
 * pcoeff (nnz, S) = <x|H|y> psi(y)/psi(x) (f64: its real part, which is exact
 * for real O).  coeff may be NULL: the completion alone (heff_offdiag_matvec).
 * All indices must be in range (the Python wrapper validates once per cache). */
size_t irl_connected_workspace_bytes(int64_t n, int64_t n_partner, int64_t ld, int is_complex);
int irl_connected_mvp_f64(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* w,
                          const double* coeff, const int64_t* dist_index, const int64_t* indptr,
                          const int64_t* partner_row, const double* pcoeff, const double* partner_O,
                          int64_t n_partner, const double* v, double* out, const double* half_f, const double* u0,
                          double* out0, int mode, void* ws, size_t ws_bytes, void* stream);
int irl_connected_mvp_c128(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* w,
                           const double* coeff, const int64_t* dist_index, const int64_t* indptr,
                           const int64_t* partner_row, const double* pcoeff, const double* partner_O,
                           int64_t n_partner, const double* v_re, const double* v_im, double* out_re,
                           double* out_im, const double* hf_re, const double* hf_im, const double* u0, double* out0,
                           int mode, void* ws, size_t ws_bytes, void* stream);

/* Batched log psi of the shallow NQS (role of ansatz.log_amplitude,
 * ansatz.py:200-247, for the BASELINE RBM / MLP), for the partner amplitude
 * ratios psi(y)/psi(x) of the connected cache (estimators.py:248-252):
 *   RBM  log psi = a.x + sum_j log cosh(b_j + W_j.x)   (c128: complex theta, complex out)
 *   MLP  log psi = u.tanh(b + W x) + c
 * x: N x n_vis uint8 (0/1); logpsi: N doubles (c128: N interleaved complex). */
size_t irl_logamp_workspace_bytes(int64_t n, int hidden, int is_complex);
int irl_logamp_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* logpsi,
                       void* ws, size_t ws_bytes, void* stream);
int irl_logamp_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* logpsi,
                        void* ws, size_t ws_bytes, void* stream);
int irl_logamp_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, double* logpsi,
                       void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------- §8(f) 2: local energies ----
 * Molecular Hamiltonian from FCIDUMP integrals (hamiltonian.py): samples are
 * bitmasks over M = 2 n_spatial <= 64 spin-orbitals (blocked: spin up first,
 * hilbert.py:1-5); h1 (n_spatial^2) and g2 (n_spatial^4, chemists' (ij|kl), 8-fold
 * symmetry expanded) are device arrays; theta is the shallow-NQS parameter
 * vector (model IRL_MODEL_RBM / IRL_MODEL_MLP, layouts as irl_obuild_*).
 *   irl_ham_local_energy     E_loc(x) = sum_y <x|H|y> psi(y)/psi(x)       (ham:290-302)
 *   irl_ham_connected_count  number of kept off-diagonal partners per sample
 *   irl_ham_connected_fill   their bitmasks, elements <y|H|x> and coefficients
 *                            element * psi(y)/psi(x) at offsets[n]        (ham:238-287, est:243-249)
 * Spin-conserving singles and doubles with the Slater-Condon rules and the
 * fermionic sign of classify_excitation (ham:180-235, hilbert.py:137-158);
 * |element| <= drop is dropped (ham:282-285).  eloc / coeff: double (c128:
 * interleaved complex).  Workspace: irl_ham_workspace_bytes. */
size_t irl_ham_workspace_bytes(int n_spatial, int hidden, int is_complex);
int irl_ham_local_energy(int model, int is_complex, const uint64_t* xbits, int64_t n, int n_spatial, double e_core,
                         const double* h1, const double* g2, double drop, int hidden, const double* theta,
                         double* eloc, void* ws, size_t ws_bytes, void* stream);
int irl_ham_connected_count(int model, int is_complex, const uint64_t* xbits, int64_t n, int n_spatial, double e_core,
                            const double* h1, const double* g2, double drop, int hidden, const double* theta,
                            int64_t* counts, void* ws, size_t ws_bytes, void* stream);
int irl_ham_connected_fill(int model, int is_complex, const uint64_t* xbits, int64_t n, int n_spatial, double e_core,
                           const double* h1, const double* g2, double drop, int hidden, const double* theta,
                           const int64_t* offsets, uint64_t* partner_bits, double* elements, double* coeff, void* ws,
                           size_t ws_bytes, void* stream);

/* ------------------------------- §8(f) 4: the reference's own ansatz ----
 * Autoregressive NQS of ansatz.py (ans:1-290), flat theta in the reference
 * layout [W1 (h x 2M), b1, W2 (2 x h), b2, Wp (h x M), bp, up, w_lin, c];
 * configurations are uint64 bitmasks in the sector (n_up, n_down); h <= 64.
 *   irl_ar_logamp  ln psi = (ln p / 2, phase) per configuration, -inf outside
 *                  the sector (log_amplitude, ans:229-247); logpsi interleaved c128
 *   irl_ar_rows    O rows d ln psi / d theta into N x ld complex (log_derivative,
 *                  ans:249-290; *error = 1 for a configuration outside the sector)
 *   irl_ar_sample  exact ancestral sampling (sample, ans:215-236): rng_states
 *                  (n x 4 uint64: state hi, lo, inc hi, lo) are numpy PCG64
 *                  streams of SeedSequence(seed).spawn(n), replayed bit for bit
 * Local energies with this ansatz (ham:290-302) combine the Hamiltonian-only
 * enumeration (irl_ham_diagonal_and_count, irl_ham_partners_fill: <x|H|x>,
 * kept partners and elements), irl_ar_logamp on the partners, and
 * irl_eloc_combine: E_loc = diag + sum element exp(ln psi(y) - ln psi(x)). */
int irl_ar_logamp(const uint64_t* xbits, int64_t n, int n_orbitals, int hidden, int n_up, int n_down,
                  const double* theta, double* logpsi, int* error, void* stream);
int irl_ar_rows(const uint64_t* xbits, int64_t n, int n_orbitals, int hidden, int n_up, int n_down,
                const double* theta, double* O, int64_t ld, int* error, void* stream);
int irl_ar_sample(const uint64_t* rng_states, int64_t n, int n_orbitals, int hidden, int n_up, int n_down,
                  const double* theta, uint64_t* out_bits, int* error, void* stream);
int irl_ham_diagonal_and_count(const uint64_t* xbits, int64_t n, int n_spatial, double e_core, const double* h1,
                               const double* g2, double drop, double* diag, int64_t* counts, void* stream);
int irl_ham_partners_fill(const uint64_t* xbits, int64_t n, int n_spatial, double e_core, const double* h1,
                          const double* g2, double drop, const int64_t* offsets, uint64_t* partner_bits,
                          double* elements, void* stream);
int irl_eloc_combine(const int64_t* indptr, const double* elements, const double* logpsi_partner,
                     const double* logpsi_x, const double* diag, int64_t n, double* eloc, void* stream);
/* Binary search of queries in ascending keys: out = index or -1 (partner rows
 * that are batch rows reuse the batch's O, est:236-242's o_row table). */
int irl_sorted_lookup(const uint64_t* keys, int64_t n_keys, const uint64_t* queries, int64_t n_queries, int64_t* out,
                      void* stream);

/* Connected completion on an on-the-fly batch (O never stored; the products of
 * irl_otf_mvp_*): the same cache arrays as irl_connected_mvp_*; partner_O
 * holds stored partner rows (n_partner x ld), or is NULL when partner_row
 * indexes the batch's own rows (exact mode: the partner dots are the batch's
 * centred dots of the same product).  Real models may instead pass the
 * partners' packed inputs and hidden activations (partner_xbits, partner_t,
 * MLP partner_g from irl_otf_prepare_*): the partner dots are then regenerated
 * by the same DMMA GEMM, no partner O is stored.  coeff may be NULL
 * (completion only). */
size_t irl_otf_connected_workspace_bytes(int model, int64_t n, int64_t n_partner, int n_in, int hidden, int64_t ld,
                                         int is_complex);
int irl_otf_connected_mvp_rbm_f64(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden,
                                  int64_t ld, const double* obar, const double* w, const double* coeff,
                                  const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                                  const double* pcoeff, const double* partner_O, const uint64_t* partner_xbits,
                                  const double* partner_t, const double* partner_g, int64_t n_partner, const double* v,
                                  double* out, const double* half_f, const double* u0, double* out0, void* ws,
                                  size_t ws_bytes, void* stream);
int irl_otf_connected_mvp_mlp_f64(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in,
                                  int hidden, int64_t ld, const double* obar, const double* w, const double* coeff,
                                  const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                                  const double* pcoeff, const double* partner_O, const uint64_t* partner_xbits,
                                  const double* partner_t, const double* partner_g, int64_t n_partner, const double* v,
                                  double* out, const double* half_f, const double* u0, double* out0, void* ws,
                                  size_t ws_bytes, void* stream);
int irl_otf_connected_mvp_rbm_c128(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden,
                                   int64_t ld, const double* obar, const double* w, const double* coeff,
                                   const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                                   const double* pcoeff, const double* partner_O, int64_t n_partner,
                                   const double* v_re, const double* v_im, double* out_re, double* out_im,
                                   const double* hf_re, const double* hf_im, const double* u0, double* out0, void* ws,
                                   size_t ws_bytes, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* IRL_SR_H_ */
