/*
 * sfseg.h -- C ABI of the B200-native SFSeg / SFSeg++ power-iteration hot path.
 *
 * The method (arxiv 2212.08058, /root/reference/PAPER.md, "P:<lines>"):
 *   principal eigenvector of the implicit space-time pixel graph
 *   M_ij = F_i F_j G(i - j)        (Eq.1/2, unary-only case p = 1,
 *                                   constant pairwise map -- SURVEY.md §8(c) A3)
 *   by power iteration in 3D-filtering form (Eq.4/7/8):
 *   y_k = F . (G_3D * (F . x_{k-1})),   x_k = y_k / ||y_k||_2,
 *   with F the learned channel combine of Eq.9 and G_3D the
 *   separable Gaussian of P:319 (normalised 1D taps, radius ceil(3 sigma),
 *   zero padding -- readings A5, A6, A8).
 *
 * Conventions (all entry points):
 *   - Every pointer is a DEVICE pointer unless its name ends in _host.
 *   - Dense layouts: channels [B][C][T][H][W] fp32, volumes [B][T][H][W] fp32,
 *     masks [B][T][H][W] uint8; W fastest, no padding, C order.
 *   - The caller owns all memory (PyTorch allocates); the solve entry points
 *     never allocate or free device memory and never synchronise unless stated.
 *     No call changes process-wide behaviour: the path choice and the optional
 *     event timing are per-call arguments (sfseg_options).  The only process-
 *     wide state is read-only caches: the TMA-encode driver entry point, the SM
 *     count per device and the shared-memory attribute per (kernel, device).
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it.
 *     Entry points do NOT synchronise unless stated ("syncs").
 *   - Validation first: every argument is checked before any launch; on a
 *     validation error nothing is written and nothing is launched.
 *   - Device-detected errors (zero norm, non-finite norm) are recorded in the
 *     workspace's error word and reported by sfseg_sync_status().  The word is
 *     STICKY: later calls on the same workspace do not clear it (the first error
 *     wins); only sfseg_sync_status reads and clears it.  A freshly allocated
 *     workspace must be reset once with sfseg_workspace_reset before its first use.
 *   - No C++ exception crosses the ABI.
 *   - Results are bitwise reproducible for a fixed (shape, build, GPU model):
 *     all reductions are fixed-order (fp32 within a CTA, fp64 across CTAs).
 */
#ifndef SFSEG_H_
#define SFSEG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFSEG_ABI_VERSION 1

typedef enum {
  SFSEG_OK = 0,
  SFSEG_ERR_INVALID_ARGUMENT = 1, /* null pointer, C<1, K<1, sigma<=0, tau non-finite, bad enum */
  SFSEG_ERR_SHAPE = 2,            /* B,T,H,W < 1; radius above the compiled maximum */
  SFSEG_ERR_WORKSPACE = 3,        /* workspace too small or not 256-byte aligned */
  SFSEG_ERR_DEGENERATE = 4,       /* some ||y_k|| == 0 (e.g. F == 0); device-detected */
  SFSEG_ERR_NONFINITE = 5,        /* NaN/Inf reached a norm; device-detected */
  SFSEG_ERR_CUDA = 6,             /* a CUDA runtime / driver call failed */
  SFSEG_ERR_NCCL = 7,             /* a NCCL call failed (multi-GPU) */
  SFSEG_ERR_UNSUPPORTED = 8       /* feature not available in this build */
} sfseg_status;

/* Dense volume shape.  When time-sharded, T is the LOCAL slab length. */
typedef struct { int64_t B, T, H, W; } sfseg_shape;

/* Separable Gaussian G_3D.  radius < 0 => ceil(3 sigma) (reading A5).
 * 1D taps g[k] = exp(-k^2/(2 sigma^2)) / sum_{|j|<=r} exp(-j^2/(2 sigma^2))
 * (reading A6); the same sigma_s / radius_s is used for the y and x axes. */
typedef struct { double sigma_t, sigma_s; int32_t radius_t, radius_s; } sfseg_gauss;

typedef enum { SFSEG_ACT_IDENTITY = 0, SFSEG_ACT_SIGMOID = 1 } sfseg_act;
typedef enum {
  SFSEG_THR_PER_FRAME_MAX = 0,  /* mask = x > tau * max_frame(x)   (reading A12, default) */
  SFSEG_THR_GLOBAL_MAX = 1,     /* mask = x > tau * max_volume(x) */
  SFSEG_THR_ABSOLUTE = 2        /* mask = x > tau */
} sfseg_thr_mode;

/* Multi-GPU time-slab sharding.  NULL => single GPU. */
typedef struct sfseg_comm sfseg_comm;
typedef struct {
  sfseg_comm* comm;   /* from sfseg_comm_create */
  int64_t T_global;   /* frames of the whole volume */
  int64_t t_offset;   /* first global frame of this rank's slab */
} sfseg_dist;

/* Per-iteration statistics written by sfseg_power_iterate (DEVICE memory,
 * double [B][K][3]):  [..][k][0] = nu_k  = ||y_k||_2 (normaliser of Eq.8)
 *                      [..][k][1] = gain n_k = nu_k / ||x_{k-1}||_2 (x_0 not unit; A10)
 *                      [..][k][2] = Rayleigh quotient x_{k-1}^T M x_{k-1} / ||x_{k-1}||^2
 *                                   (Eq.3; only when want_rayleigh != 0, else 0). */
#define SFSEG_STATS_PER_ITER 3

const char* sfseg_status_string(sfseg_status s);
int32_t sfseg_abi_version(void);
/* Text of the last CUDA error seen by this thread inside the library (for SFSEG_ERR_CUDA). */
const char* sfseg_last_cuda_error(void);

/* ---- per-call options (no process-global switches) ----
 * algo selects the forward path (all compute the same operator, Eq.7 with p = 1,
 * up to fp32 rounding order):
 *   SFSEG_ALGO_AUTO: the fused single-pass 3D kernel (one HBM read of p_{k-1} and F,
 *     one write of p_k per voxel-iteration) when the compiled radii allow it
 *     (r_t <= 3, r_s <= 8; PAPER.md:319's 3x7x7 support is such a case), otherwise
 *     one temporal pass + one fused spatial pass per iteration.
 *   SFSEG_ALGO_TWO_PASS: always the two-pass iteration.  Its spatial pass runs on the
 *     tensor pipe for compiled spatial radii 8..48: each operand and tap split into two
 *     fp16 planes (22 significant bits; the data scaled per volume by a power of two into
 *     fp16's range) and three products per tap, fp32 accumulation: fp32-class arithmetic
 *     (A25; x_K error within 2x the FP32-FMA pass's).  The same for the two-pass
 *     fallback of SFSEG_ALGO_AUTO.
 *   SFSEG_ALGO_TWO_PASS_FP32: the two-pass iteration with the FP32-FMA spatial pass.
 * profiler: NULL, or a sfseg_profiler that records CUDA events around every pass launch
 * (benchmark instrumentation).
 * binarize: NULL, or the soft-binarisation of Alg.1 STEP 3 (SURVEY §8(f) row f2,
 * reading A21): after the normalisation of every iteration k > n_cont,
 *   x_k <- sigma(kappa_k (x_k - theta_k)),  theta_k = mean of the positive entries of x_k,
 *   kappa_k = kappa0 * growth^(k - n_cont - 1),
 * and the binarised x_k is the next iterate as is (not renormalised).  When K > n_cont the
 * output x_out is the last binarised iterate (values in (0,1), not unit norm).  With a tape,
 * sfseg_power_iterate_backward_ex (same options) differentiates through it ("trainable by
 * using a soft-binarization between iterations").  Forces the two-pass iteration. */
#define SFSEG_ALGO_AUTO 0
#define SFSEG_ALGO_TWO_PASS 1
#define SFSEG_ALGO_TWO_PASS_FP32 3
/* the two-pass iteration with the warp-level (mma.sync) tensor-core spatial pass in three bf16
 * planes and six products per tap (|a - a1 - a2 - a3| <= 2^-27 |a|; A23) */
#define SFSEG_ALGO_TWO_PASS_MMA_SYNC 4
/* the two-pass iteration with the tcgen05 / TMEM spatial pass (spatial radii <= 24; else as TWO_PASS) */
#define SFSEG_ALGO_TWO_PASS_TCGEN05 5
/* the two-pass iteration with the mma.sync spatial pass in two fp16 planes and three products
 * per tap (22 significant bits per operand; A25): half the tensor work of the
 * bf16 format (what SFSEG_ALGO_TWO_PASS runs).  The forward temporal pass records max |v| per volume, and the data are
 * scaled by a power of two into fp16's normal range; entries below 2^-24 of a volume's
 * max |v| lose relative precision (absolute error <= 2^-39 max |v|). */
#define SFSEG_ALGO_TWO_PASS_MMA_F16 6
typedef struct sfseg_profiler sfseg_profiler;
typedef struct {
  int32_t n_cont;   /* continuous iterations before binarisation starts (>= 0) */
  float kappa0;     /* steepness of the first binarised iteration (> 0) */
  float growth;     /* geometric growth of the steepness per iteration (> 0) */
} sfseg_binarize;
/* slab_schedule (time slabs, a sfseg_dist or sfseg_power_iterate_slabs):
 *   SFSEG_SLAB_OVERLAP (0): per iteration the spatial pass computes the r_t boundary frames
 *     first; the halo exchange runs on a second stream (the communicator's, or one the
 *     emulation creates for the call) while the interior frames are computed, and the norm
 *     allreduce + finalize run there while the next temporal pass runs (the normalisation
 *     s_k is applied by the next spatial pass instead of the temporal pass).
 *   SFSEG_SLAB_SERIAL (1): the same kernels in the same order on the caller's stream only
 *     (bitwise the same results; for checking the overlapped schedule). */
#define SFSEG_SLAB_OVERLAP 0
#define SFSEG_SLAB_SERIAL 1
typedef struct {
  int32_t algo;
  sfseg_profiler* profiler;
  const sfseg_binarize* binarize;
  int32_t slab_schedule;
} sfseg_options;

/* Per-kernel timing object (owned by the caller).  sfseg_profiler_read syncs the
 * recorded events and returns, per category [0]=temporal pass, [1]=spatial pass,
 * [2]=once-per-solve kernels, [3]=backward passes, [4]=fused single-pass 3D
 * iteration, [5]=reserved, the summed milliseconds and launch counts, then resets. */
sfseg_status sfseg_profiler_create(sfseg_profiler** out);
sfseg_status sfseg_profiler_destroy(sfseg_profiler* p);
sfseg_status sfseg_profiler_read(sfseg_profiler* p, double* ms_host /*[6]*/, int64_t* count_host /*[6]*/);

/* Zero the header (error word, counters) of a freshly allocated workspace (async on stream). */
sfseg_status sfseg_workspace_reset(void* ws, void* stream);

/* Largest radii compiled into this build (spatial, temporal). */
void sfseg_max_radii(int32_t* radius_s_max_host, int32_t* radius_t_max_host);

/* Workspace needed by sfseg_power_iterate / sfseg_power_iterate_backward for
 * this problem (want_tape != 0: also the bytes of the tape buffer that a
 * forward must record for a later backward).  Host outputs; no GPU work. */
sfseg_status sfseg_workspace_bytes(sfseg_shape shape, int32_t C, sfseg_gauss gauss, int32_t K,
                                   int32_t want_tape, const sfseg_dist* dist_or_null,
                                   size_t* ws_bytes_host, size_t* tape_bytes_host);

/* Eq.9 / Alg.1 lines 1-2:
 *   F = act(sum_c w_c ch_c + b), act = identity (single channel "without the
 *   sigmoid") or sigmoid 1/(1+e^{-z}) (the printed e^{x} is a typo, A1).
 * ch [B][C][T][H][W] -> F [B][T][H][W].  w_host: C floats in host memory. */
sfseg_status sfseg_combine_channels(const float* ch, int32_t C, sfseg_shape shape,
                                    const float* w_host, float b, int32_t act,
                                    float* F, void* stream);

/* K power iterations (Eq.4/7/8, Alg.1 Step 2 + normalise)
 * from x_0 = F (Alg.1 line 3) or from x0_or_null ([B][T][H][W]).
 *   ch/C/w_host/b/act: as sfseg_combine_channels (combine fused into the solve).
 *   x_out  [B][T][H][W]: x_K, unit L2 norm per volume (reading A9).
 *   F_out_or_null [B][T][H][W]: the combined F (needed by a later backward).
 *   stats_or_null: DEVICE double [B][K][3] (see SFSEG_STATS_PER_ITER).
 *   want_rayleigh: also compute the Rayleigh quotient (+4 B/voxel/iteration).
 *   tape_or_null: if non-NULL (size from sfseg_workspace_bytes with want_tape),
 *     records what sfseg_power_iterate_backward needs.
 *   ws / ws_bytes: device workspace, 256-byte aligned, >= sfseg_workspace_bytes.
 *   dist_or_null: time-slab sharding; NULL => whole volume on this GPU.
 * Asynchronous; call sfseg_sync_status(ws, stream) to learn device errors. */
sfseg_status sfseg_power_iterate(const float* ch, int32_t C, const float* w_host, float b,
                                 int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                 const float* x0_or_null, float* x_out, float* F_out_or_null,
                                 double* stats_or_null, int32_t want_rayleigh, void* tape_or_null,
                                 void* ws, size_t ws_bytes, const sfseg_dist* dist_or_null,
                                 void* stream);
/* Same, with per-call options (NULL == {SFSEG_ALGO_AUTO, NULL}).  With dist_or_null the
 * call validates its arguments on every rank and agrees on the outcome (one int
 * allreduce, one stream sync) before the first data-path collective: a rank's invalid
 * argument makes every rank return an error instead of blocking its peers. */
sfseg_status sfseg_power_iterate_ex(const float* ch, int32_t C, const float* w_host, float b,
                                    int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                    const float* x0_or_null, float* x_out, float* F_out_or_null,
                                    double* stats_or_null, int32_t want_rayleigh, void* tape_or_null,
                                    void* ws, size_t ws_bytes, const sfseg_dist* dist_or_null,
                                    const sfseg_options* opt_or_null, void* stream);

/* Gradient of L(x_K) w.r.t. the channel weights and bias through the K
 * unrolled iterations ("through the full spectral algorithm", P:42, P:212-213,
 * P:232); recursion of SURVEY.md Appendix A.  Inputs are those of the forward
 * call that wrote `tape` (same ch, w, b, act, shape, gauss, K, x0).
 *   dL_dx [B][T][H][W]: dL/dx_K supplied by the caller (the loss is not in the ABI).
 *   dL_dw_host: C doubles; dL_db_host: 1 double (host memory).
 * Syncs `stream` once at the end (host outputs); returns device errors too. */
sfseg_status sfseg_power_iterate_backward(const float* ch, int32_t C, const float* w_host,
                                          float b, int32_t act, sfseg_shape shape,
                                          sfseg_gauss gauss, int32_t K,
                                          const float* x0_or_null, const void* tape,
                                          const float* dL_dx, double* dL_dw_host,
                                          double* dL_db_host, void* ws, size_t ws_bytes,
                                          const sfseg_dist* dist_or_null, void* stream);
sfseg_status sfseg_power_iterate_backward_ex(const float* ch, int32_t C, const float* w_host,
                                             float b, int32_t act, sfseg_shape shape,
                                             sfseg_gauss gauss, int32_t K,
                                             const float* x0_or_null, const void* tape,
                                             const float* dL_dx, double* dL_dw_host,
                                             double* dL_db_host, void* ws, size_t ws_bytes,
                                             const sfseg_dist* dist_or_null,
                                             const sfseg_options* opt_or_null, void* stream);

/* ---- full SFSeg / SFSeg++ operator ----
 * The general power iteration of Eq.7 / Eq.10: a unary
 * map S with exponent p and a pairwise map F with the first-order Taylor
 * bracket of Eq.2,
 *   X_crt = S^p [ (alpha^-1 - F^2) G*(S^p X) - G*(F^2 S^p X) + 2 F G*(F S^p X) ],
 *   X_{k+1} = X_crt / ||X_crt||_2                                   (Eq.8 / Eq.11)
 * i.e. M_ij = s_i^p s_j^p [alpha^-1 - (f_i - f_j)^2] G_ij.  S and F come from
 * their own channel stacks by Eq.9 (act as in sfseg_combine_channels);
 * x_0 = S (Alg.1 line 3) or x0_or_null.  No clamping (reading A18): with S, F in
 * [0,1] and alpha <= 1 the operator is non-negative.  S^p needs S >= 0 (A19): a
 * negative S gives NaN, reported as SFSEG_ERR_NONFINITE by sfseg_sync_status.
 *   s_ch [B][Cs][T][H][W], f_ch [B][Cf][T][H][W]; ws_host / wf_host: Cs / Cf floats (host).
 *   p > 0, alpha > 0 (finite), else SFSEG_ERR_INVALID_ARGUMENT.
 *   stats_or_null: DEVICE double [B][K][3] as sfseg_power_iterate (Rayleigh slot = 0).
 *   bin_or_null: soft-binarisation (Alg.1 STEP 3): after the
 *     normalisation of every iteration k > n_cont, x_k <- sigma(kappa_k (x_k - theta_k)) with
 *     theta_k = mean of the positive entries of x_k and kappa_k = kappa0 * growth^(k-n_cont-1)
 *     (reading A21); the binarised x_k is the next iterate as is, and when
 *     K > n_cont x_out is the last binarised iterate (values in (0,1), not unit norm; hard
 *     mask: sfseg_threshold with SFSEG_THR_ABSOLUTE, tau = 0.5).  NULL: no binarisation.
 *   ws: >= sfseg_workspace_bytes_full(...), 256-byte aligned.  Asynchronous. */
sfseg_status sfseg_workspace_bytes_full(sfseg_shape shape, int32_t Cs, int32_t Cf, sfseg_gauss gauss,
                                        int32_t K, size_t* ws_bytes_host);
sfseg_status sfseg_power_iterate_full(const float* s_ch, int32_t Cs, const float* ws_host, float bs,
                                      int32_t act_s, const float* f_ch, int32_t Cf,
                                      const float* wf_host, float bf, int32_t act_f, double p,
                                      double alpha, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                      const float* x0_or_null, float* x_out, double* stats_or_null,
                                      const sfseg_binarize* bin_or_null, void* ws, size_t ws_bytes,
                                      const sfseg_options* opt_or_null, void* stream);

/* ---- online / sub-window mode ----
 * PAPER.md:367-387 (Fig. offline_online): the power iteration runs on
 * q-frame sub-windows sliding by `stride` frames (starts 0, stride, ... while
 * start + q < T, then T - q; q >= T is the offline solve), each window the
 * offline iteration of sfseg_power_iterate (zero padding at the window ends,
 * normalisation per window), warm-started on the frames it shares with the
 * previous window from that window's solution, rescaled per volume to the L2
 * norm of F on those frames (reading A20), and from F elsewhere (Alg.1 line 3).
 * x_out [B][T][H][W]: per frame the result of the LAST window covering it (each
 * window's result is unit-norm over that window).  Combine as
 * sfseg_power_iterate; device errors of every window via sfseg_sync_status(ws, stream).
 * 1 <= stride <= q when q < T (else SFSEG_ERR_INVALID_ARGUMENT: frames would be skipped).
 * ws: >= sfseg_workspace_bytes_online(...).  Asynchronous. */
sfseg_status sfseg_workspace_bytes_online(sfseg_shape shape, int32_t C, sfseg_gauss gauss, int32_t K,
                                          int32_t q, size_t* ws_bytes_host);
sfseg_status sfseg_power_iterate_online(const float* ch, int32_t C, const float* w_host, float b,
                                        int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                        int32_t q, int32_t stride, float* x_out, void* ws,
                                        size_t ws_bytes, void* stream);

/* Hard threshold ("simply obtained by thresholding"): uint8 mask.
 * Mode per sfseg_thr_mode; strict '>' in fp32 against tau*max; a frame (or
 * volume) whose max is <= 0 yields zeros.  ws: >= sfseg_threshold_ws_bytes. */
size_t sfseg_threshold_ws_bytes(sfseg_shape shape);
sfseg_status sfseg_threshold(const float* x, sfseg_shape shape, float tau, int32_t mode,
                             uint8_t* mask, void* ws, size_t ws_bytes, void* stream);

/* Synchronise `stream`, then read and clear the device error word in `ws`.
 * Returns SFSEG_OK, SFSEG_ERR_DEGENERATE, SFSEG_ERR_NONFINITE or SFSEG_ERR_CUDA. */
sfseg_status sfseg_sync_status(void* ws, void* stream);

/* End-to-end convenience over HOST buffers (used for the e2e measurement):
 * H2D of ch_host (pinned or pageable) into d_ch, sfseg_power_iterate, then
 * sfseg_threshold, then D2H of x and mask into x_out_host / mask_out_host
 * (either may be NULL), then sync.  Device buffers d_ch ([B][C][T][H][W]),
 * d_x ([B][T][H][W]) and d_mask are caller-owned scratch.  Syncs. */
sfseg_status sfseg_solve_host(const float* ch_host, int32_t C, const float* w_host, float b,
                              int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                              float tau, int32_t thr_mode, float* d_ch, float* d_x,
                              uint8_t* d_mask, float* x_out_host, uint8_t* mask_out_host,
                              void* ws, size_t ws_bytes, void* stream);

/* End-to-end over a BATCH of host volumes, pipelined inside the library: the H2D copy of
 * volume i+1 (stream_h2d) and the D2H copy of volume i-1 (stream_d2h) overlap the solve and
 * threshold of volume i (stream), one cudaMemcpyAsync per copy, two device slots ordered by
 * events (created and destroyed inside the call).  ch_host[i]: [B][C][T][H][W] (pinned for
 * overlap); x_out_host[i] / mask_out_host[i] (either array or entry may be NULL).  d_ch
 * [2][B][C][T][H][W], d_x [2][B][T][H][W], d_mask [2][B][T][H][W]: caller-owned device slots.
 * Streams are the caller's.  Syncs; returns the first device error of any volume. */
sfseg_status sfseg_solve_host_batch(const float* const* ch_host, int32_t n, int32_t C, const float* w_host,
                                    float b, int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                    float tau, int32_t thr_mode, float* d_ch, float* d_x, uint8_t* d_mask,
                                    float* const* x_out_host, uint8_t* const* mask_out_host, void* ws,
                                    size_t ws_bytes, void* stream, void* stream_h2d, void* stream_d2h);

/* ---- plan introspection ----
 * The forward path sfseg_power_iterate_ex takes for this shape, Gaussian and algo on
 * one GPU without a tape (a tape forces the two-pass iteration): info_host[0] =
 * SFSEG_PATH_*, [1] = compiled temporal radius, [2] = compiled spatial radius.  Host
 * only, no device work.  Errors: SFSEG_ERR_INVALID_ARGUMENT / SFSEG_ERR_SHAPE. */
#define SFSEG_PATH_TWO_PASS_FP32 0
#define SFSEG_PATH_TWO_PASS_TC 1
#define SFSEG_PATH_FUSED_3D 2
#define SFSEG_PATH_TWO_PASS_TCGEN05 4
#define SFSEG_PATH_TWO_PASS_TC_F16 5
sfseg_status sfseg_forward_path(sfseg_shape shape, sfseg_gauss gauss, int32_t algo, int32_t* info_host /*[3]*/);

/* ---- multi-GPU communicator (NCCL, loaded at run time with dlopen) ---- */
/* Multi-GPU solve: call sfseg_power_iterate with dist_or_null = {comm, T_global,
 * t_offset} on every rank (one process per GPU, ranks own consecutive slabs
 * in rank order, each slab >= the compiled temporal radius); ch / x0 / x_out
 * are the rank's LOCAL slab [B][C][T_local][H][W] / [B][T_local][H][W].
 * Workspace from sfseg_workspace_bytes(..., dist, ...).  Every iteration:
 * r_t-frame halo send/recv with ranks +-1 and an fp64 allreduce of the norm
 * partials (NCCL, enqueued on `stream`).  With a tape (each rank its own: nu_k global, u_k of
 * its frames) sfseg_power_iterate_backward with the same sfseg_dist runs the time-slab backward
 * (halo of F y_bar_k per step, allreduces of the step scalars and of dw, db; x_0 = F, no
 * binarisation).  F_out / binarisation: SFSEG_ERR_UNSUPPORTED.
 * 128-byte NCCL unique id into id_host (call on rank 0, broadcast it). */
sfseg_status sfseg_get_unique_id(uint8_t id_host[128]);
sfseg_status sfseg_comm_create(const uint8_t id_host[128], int32_t nranks, int32_t rank,
                               int32_t device, sfseg_comm** out);
sfseg_status sfseg_comm_destroy(sfseg_comm* comm);

/* ---- time-slab decomposition emulated on ONE GPU (validation of the sharded path) ----
 * Splits every volume's T frames into nslabs consecutive slabs (slab i covers
 * frames [i*T/n, (i+1)*T/n)) and runs the exact per-rank phases of the
 * multi-GPU solve for all slabs on `stream`: halo frames are
 * copied device-to-device and the norm partials summed in rank order.  Same
 * arguments/outputs as sfseg_power_iterate on the full dense volume (no tape). */
/* Host only (no device work): the spatial-pass launches of one time-slab iteration of the
 * overlapped schedule (SFSEG_SLAB_OVERLAP) for a slab of T frames with compiled
 * temporal radius radius_t and the given neighbours, as (first frame, frame count) pairs in
 * launch order in ranges_host[0 .. 2 n_ranges): the boundary ranges the neighbours need
 * first (*n_boundary_host of them; the halo exchange is enqueued after these), then the
 * interior.  The ranges tile [0, T) exactly.  Errors: SFSEG_ERR_INVALID_ARGUMENT. */
sfseg_status sfseg_slab_launch_ranges(int32_t T, int32_t radius_t, int32_t has_lo, int32_t has_hi,
                                      int32_t* ranges_host /*[6]*/, int32_t* n_ranges_host,
                                      int32_t* n_boundary_host);
sfseg_status sfseg_slabs_workspace_bytes(sfseg_shape shape, int32_t C, sfseg_gauss gauss, int32_t K,
                                         int32_t nslabs, size_t* ws_bytes_host);
sfseg_status sfseg_power_iterate_slabs(const float* ch, int32_t C, const float* w_host, float b,
                                       int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                       int32_t nslabs, const float* x0_or_null, float* x_out,
                                       double* stats_or_null, int32_t want_rayleigh,
                                       void* tape_or_null, void* ws, size_t ws_bytes,
                                       const sfseg_options* opt_or_null, void* stream);
/* Tape of the emulated slabs (one per slab, concatenated) and the time-slab BACKWARD emulated
 * the same way (per step an r_t-frame halo of F y_bar_k exchanged with
 * the neighbour slabs, an allreduce of <x_{k-1}, x_bar_{k-1}>, and a final allreduce of the C + 1
 * weight-gradient sums): the per-rank phases of sfseg_power_iterate_backward with a
 * sfseg_dist.  x_0 = F only, no binarisation (SFSEG_ERR_UNSUPPORTED).  Syncs (host outputs). */
sfseg_status sfseg_slabs_tape_bytes(sfseg_shape shape, int32_t C, sfseg_gauss gauss, int32_t K, int32_t nslabs,
                                    size_t* tape_bytes_host);
sfseg_status sfseg_power_iterate_slabs_backward(const float* ch, int32_t C, const float* w_host, float b,
                                                int32_t act, sfseg_shape shape, sfseg_gauss gauss, int32_t K,
                                                int32_t nslabs, const void* tape, const float* dL_dx,
                                                double* dL_dw_host, double* dL_db_host, void* ws,
                                                size_t ws_bytes, const sfseg_options* opt_or_null,
                                                void* stream);
/* Syncs `stream`; returns the first device-detected error of any slab. */
sfseg_status sfseg_slabs_sync_status(sfseg_shape shape, int32_t C, sfseg_gauss gauss, int32_t K,
                                     int32_t nslabs, void* ws, void* stream);

/* ---- learning loop ----
 * One optimizer step of Eq.13, AdamW, with AMSGrad ("AdamW optimizer
 * with AMSGrad") when amsgrad != 0:
 *   m_t = b1 m + (1 - b1) g;  v_t = b2 v + (1 - b2) g^2;  vmax_t = max(vmax, v_t)
 *   w  <- w - lr ( m_t/(1 - b1^t) / (sqrt(vmax_t (or v_t))/sqrt(1 - b2^t) + eps) + weight_decay w )
 * (alpha = 1, eta_t = lr: the decoupled weight decay of AdamW, reading A22).
 * w [n], grad [n], state [3][n] (m, v, vmax; zero before step 1): DEVICE doubles, updated in
 * place; t >= 1 is the step number.  Asynchronous on stream. */
typedef struct { double lr, beta1, beta2, eps, weight_decay; int32_t amsgrad; } sfseg_adamw;
sfseg_status sfseg_adamw_step(double* w, const double* grad, double* state, int32_t n, int64_t t,
                              const sfseg_adamw* hp, void* stream);

/* Focal-Dice loss of Eq.12 (reading A24) and its gradient, on the device:
 * per training frame i = (volume, frame) the soft Dice overlap
 *   D_i = 2 sum(x t) / (sum(x) + sum(t))
 * of the prediction x (e.g. the soft-binarised output of sfseg_power_iterate_ex) and the binary
 * ground truth t (mask: uint8 0/1), J = sum_i (1 - D_i)^gamma (gamma = 0.75 in the paper),
 * dL_dx = dJ/dx.  x, dL_dx [B][T][H][W] fp32, mask [B][T][H][W] uint8; loss: ONE DEVICE double.
 * A frame with sum(x) + sum(t) == 0 contributes 0.  Sums in fp64, fixed order (deterministic).
 * ws: >= sfseg_focal_dice_ws_bytes(shape), 256-byte aligned.  Asynchronous. */
size_t sfseg_focal_dice_ws_bytes(sfseg_shape shape);
sfseg_status sfseg_focal_dice(const float* x, const uint8_t* mask, sfseg_shape shape, double gamma,
                              double* loss, float* dL_dx, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SFSEG_H_ */
