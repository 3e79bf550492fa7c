// Host side of libsfseg.so: argument validation, workspace carve-up, radius
// dispatch, TMA descriptor construction and launch sequencing of the
// sm_100a kernels.  C ABI declared in include/sfseg.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/sfseg.h"
#include "common.cuh"
#include "misc.cuh"
#include "spass.cuh"
#include "tpass.cuh"
#include "comm.cuh"
#include "full.cuh"
#include "online.cuh"
#include "bwd.cuh"
#include "learn.cuh"
#include "launch.h"
#include "spass_tc6.cuh"

using namespace sfseg;

namespace sfseg {
cudaError_t set_smem_attr_once(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find({kernel, dev});
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[{kernel, dev}] = smem;
  return e;
}
}  // namespace sfseg

namespace {

#define SF_CUDA(call)                                                   \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) {                                            \
      last_cuda_error() = e_;                                           \
      return SFSEG_ERR_CUDA;                                            \
    }                                                                   \
  } while (0)

cudaError_t& last_cuda_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}

// Debug builds only (-DSFSEG_DEBUG_SYNC): synchronise after every launch and name the
// failing kernel.  The release library never synchronises inside an asynchronous call.
cudaError_t after_launch(const char* name, cudaStream_t st) {
  cudaError_t e = cudaGetLastError();
#ifdef SFSEG_DEBUG_SYNC
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) fprintf(stderr, "[sfseg] kernel %s failed: %s\n", name, cudaGetErrorString(e));
#else
  (void)name;
  (void)st;
#endif
  return e;
}

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }
inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------ radius dispatch tables
constexpr int kSpatialRadii[] = {1, 2, 3, 4, 5, 6, 8, 9, 12, 16, 18, 24, 32, 36, 48};
constexpr int kTemporalRadii[] = {0, 1, 2, 3, 4, 5, 6, 8, 9, 12, 16};

int pick_spatial(int r) {
  for (int R : kSpatialRadii)
    if (R >= r) return R;
  return -1;
}
int pick_temporal(int r) {
  for (int R : kTemporalRadii)
    if (R >= r) return R;
  return -1;
}

int resolve_radius(double sigma, int32_t r) { return r >= 0 ? r : (int)std::ceil(3.0 * sigma - 1e-12); }

void gauss_taps(double sigma, int r, int Rpad, float* out /* 2*Rpad+1 */) {
  std::vector<double> g(2 * r + 1);
  double s = 0.0;
  for (int k = -r; k <= r; ++k) {
    g[k + r] = std::exp(-(double)k * k / (2.0 * sigma * sigma));
    s += g[k + r];
  }
  for (int i = 0; i < 2 * Rpad + 1; ++i) {
    const int k = i - Rpad;
    out[i] = (std::abs(k) <= r) ? (float)(g[k + r] / s) : 0.f;
  }
}

// SM count of the CURRENT device (cached per device id: plans are made per call on the
// caller's current device).
int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  std::atomic<int>& c = cache[dev & 63];
  int n = c.load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    c.store(n, std::memory_order_relaxed);
  }
  return n;
}

// ------------------------------------------------------------------ TMA descriptor encode (driver entry point)
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// The two fp16 planes of v for the tcgen05 spatial pass: dims {W, H, 2 BT} (plane-frames
// [bt][plane]), box {64, 128, 2} = both planes of a 128-row x 64-column tile, SWIZZLE_128B (the
// MMA's K-major B operand layout); columns >= W and rows outside [0, H) read as zero.
bool make_planes_tmap(CUtensorMap* map, const void* base, int64_t W, int64_t H, int64_t BT, int64_t Wp) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)(2 * BT)};
  cuuint64_t strides[2] = {(cuuint64_t)(Wp * 2), (cuuint64_t)(H * Wp * 2)};
  cuuint32_t box[3] = {(cuuint32_t)k6BoxW, (cuuint32_t)k6XN, 2u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_volume_tmap(CUtensorMap* map, const float* base, int64_t W, int64_t H, int64_t BT, int64_t Wp, int boxw,
                      int boxh = kM) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)BT};
  cuuint64_t strides[2] = {(cuuint64_t)(Wp * 4), (cuuint64_t)(H * Wp * 4)};
  cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)boxh, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int spass_occupancy(int R) {
  switch (R) {
#define OC(r) \
  case r:     \
    return spass_ctas_per_sm(r);
    OC(1) OC(2) OC(3) OC(4) OC(5) OC(6) OC(8) OC(9) OC(12) OC(16) OC(18) OC(24) OC(32) OC(36) OC(48)
#undef OC
    default:
      return 1;
  }
}

}  // namespace
// ------------------------------------------------------------------ optional per-kernel event timing
// (bench instrumentation: a caller-owned sfseg_profiler passed in sfseg_options)
struct ProfRec {
  int cat;
  cudaEvent_t a, b;
};
struct sfseg_profiler {
  std::mutex mu;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
namespace {
using Profiler = sfseg_profiler;
enum ProfCat { PC_TPASS = 0, PC_SPASS = 1, PC_ONCE = 2, PC_BWD = 3, PC_F3D = 4, PC_MK = 5, PC_N = 6 };

// RAII scope that brackets a launch with events when profiling is on.
struct ProfScope {
  Profiler* p;
  cudaStream_t st;
  int cat;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(Profiler* prof, cudaStream_t s, int c) : p(prof), st(s), cat(c) {
    if (!p) return;
    std::lock_guard<std::mutex> g(p->mu);
    a = p->get();
    b = p->get();
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> g(p->mu);
    p->recs.push_back({cat, a, b});
  }
};

// Blocks per frame for the row-parallel streaming kernels (misc.cuh): enough
// CTAs in total to fill 148 SMs several times over, at most one per kRows rows.
int ew_gx(int64_t H, int64_t BT) {
  const int64_t want = (8 * (int64_t)num_sms() + BT - 1) / BT;
  const int64_t rows = (H + kRows - 1) / kRows;
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, rows), 16));
}

// ------------------------------------------------------------------ problem plan
struct Plan {
  int64_t B, T, H, W, Wp, BT;
  int C, K;
  int rt, rs;      // requested radii
  int RT, RS;      // compiled radii (>= requested; extra taps are zero)
  float gt[2 * kMaxRT + 1];
  float gs[2 * kMaxRS + 1];
  int64_t vol_elems;  // B*T*H*Wp
  int S;              // strips
  int NB;             // 32-row blocks per column
  int64_t U;          // spass block units
  int G;              // spass grid
  bool tc;            // forward spatial pass on the tensor cores (spass_tc_kernel)
  bool f16;           // ... in the two-plane fp16 format (fmt 1; temporal pass records max |v|)
  int Gtc;            // its grid
  int Gcap, Gcap_tc;  // resident-CTA caps of the FP32 / tensor-core passes (grids of frame-range launches)
  bool tc6;           // ... on tcgen05 / TMEM (spass_tc6_kernel, hot forward only): 128-column strips,
                      //   v written by the temporal pass as two fp16 planes (TP_FWD16)
  int S6;             // its strips
  int NB6;            // its 64-row y-blocks per column
  int64_t U6;         // its units = BT * S6 * NB6
  int G6;             // its grid (one CTA per SM: all 512 TMEM columns)
  int gx;             // elementwise grid.x per frame
  bool f3d;           // single-pass fused 3D kernel (small radii) for the single-GPU forward
  int TX, TY;         // f3d tiles per frame (64 columns x f3d_th(RS) rows)
  int64_t U3;         // f3d units = B * TY * TX * T
  int G3;             // f3d grid
  int algo;           // SFSEG_ALGO_* of this call (sfseg_options; no process-global switch)
  Profiler* prof;     // per-launch event timing (nullable)
  bool bin;           // soft-binarisation (row f2) of iterations k > binv.n_cont
  sfseg_binarize binv;
  // workspace offsets
  size_t off_sc, off_part, off_out, off_F, off_p, off_v, off_p2, off_xbar, off_Fbar, off_x0p, ws_fwd, ws_bwd;
  size_t n_part;
  size_t tape_nu_bytes, tape_hdr_bytes, tape_bytes;  // tape: nu [B][K], bin stats [B][K][2], K x u
  float kappa(int k) const {  // steepness of iteration k (1-based); 0 when not binarised
    if (!bin || k <= binv.n_cont) return 0.f;
    return (float)(binv.kappa0 * std::pow((double)binv.growth, (double)(k - binv.n_cont - 1)));
  }
};

bool valid_algo(int32_t algo) {
  return algo == SFSEG_ALGO_AUTO || algo == SFSEG_ALGO_TWO_PASS || algo == SFSEG_ALGO_TWO_PASS_FP32 ||
         algo == SFSEG_ALGO_TWO_PASS_MMA_SYNC || algo == SFSEG_ALGO_TWO_PASS_TCGEN05 ||
         algo == SFSEG_ALGO_TWO_PASS_MMA_F16;
}

// Grid of the tcgen05 spatial pass over U units of B volumes x S strips: one CTA per SM; a
// multiple of B x S when that fits, so CTA ranges align with strips (spass_tc6.cuh).
int tc6_grid(int64_t B, int64_t S, int64_t U) {
  const int64_t bs = B * S, sms = num_sms();
  const int64_t g = bs <= sms ? bs * (sms / bs) : sms;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, U));
}

sfseg_status make_plan(sfseg_shape sh, int32_t C, sfseg_gauss g, int32_t K, Plan* P,
                       const sfseg_options* opt = nullptr) {
  const int algo = opt ? opt->algo : SFSEG_ALGO_AUTO;
  if (!valid_algo(algo)) return SFSEG_ERR_INVALID_ARGUMENT;
  P->algo = algo;
  P->prof = opt ? opt->profiler : nullptr;
  P->bin = opt && opt->binarize;
  if (P->bin) {
    const sfseg_binarize& bz = *opt->binarize;
    if (bz.n_cont < 0 || !(bz.kappa0 > 0.f) || !std::isfinite(bz.kappa0) || !(bz.growth > 0.f) ||
        !std::isfinite(bz.growth))
      return SFSEG_ERR_INVALID_ARGUMENT;
    P->binv = bz;
  }
  if (C < 1 || C > kMaxC) return C < 1 ? SFSEG_ERR_INVALID_ARGUMENT : SFSEG_ERR_UNSUPPORTED;
  if (K < 1) return SFSEG_ERR_INVALID_ARGUMENT;
  if (!(g.sigma_t > 0.0) || !(g.sigma_s > 0.0) || !std::isfinite(g.sigma_t) || !std::isfinite(g.sigma_s))
    return SFSEG_ERR_INVALID_ARGUMENT;
  if (sh.B < 1 || sh.T < 1 || sh.H < 1 || sh.W < 1) return SFSEG_ERR_SHAPE;
  if (sh.H > (1 << 24) || sh.W > (1 << 24) || sh.B * sh.T > (1 << 30)) return SFSEG_ERR_SHAPE;
  P->B = sh.B;
  P->T = sh.T;
  P->H = sh.H;
  P->W = sh.W;
  P->BT = sh.B * sh.T;
  P->Wp = round_up(sh.W, 8);
  P->C = C;
  P->K = K;
  P->rt = resolve_radius(g.sigma_t, g.radius_t);
  P->rs = resolve_radius(g.sigma_s, g.radius_s);
  P->RT = pick_temporal(P->rt);
  P->RS = pick_spatial(std::max(P->rs, 1));
  if (P->RT < 0 || P->RS < 0) return SFSEG_ERR_SHAPE;
  gauss_taps(g.sigma_t, P->rt, P->RT, P->gt);
  gauss_taps(g.sigma_s, P->rs, P->RS, P->gs);
  P->vol_elems = P->BT * P->H * P->Wp;
  P->S = (int)((sh.W + kTW - 1) / kTW);
  P->NB = (int)((sh.H + kM - 1) / kM);
  P->U = P->BT * P->S * P->NB;
  const int64_t cap = (int64_t)num_sms() * spass_occupancy(P->RS);
  P->G = (int)std::max<int64_t>(1, std::min<int64_t>(cap, P->U / 4));
  P->Gcap = (int)cap;
  P->gx = ew_gx(P->H, P->BT);
  P->tc = algo != SFSEG_ALGO_TWO_PASS_FP32 && spass_tc_supported(P->RS);
  // the hot forward's default spatial pass (r_s in 8..36, no soft-binarisation; single GPU and time slabs): tcgen05 / TMEM
  P->tc6 = P->tc && spass_tc6_supported(P->RS) && !P->bin &&
           (algo == SFSEG_ALGO_AUTO || algo == SFSEG_ALGO_TWO_PASS || algo == SFSEG_ALGO_TWO_PASS_TCGEN05);
  // the forward's default tensor-core format is two fp16 planes (A25); SFSEG_ALGO_TWO_PASS_MMA_SYNC
  // selects the three-plane bf16 one (A23)
  P->f16 = P->tc && (algo == SFSEG_ALGO_AUTO || algo == SFSEG_ALGO_TWO_PASS || algo == SFSEG_ALGO_TWO_PASS_MMA_F16);
  P->S6 = (int)((sh.W + k6M - 1) / k6M);
  P->NB6 = (int)((sh.H + k6YN - 1) / k6YN);
  P->U6 = P->BT * P->S6 * P->NB6;
  P->G6 = tc6_grid(P->B, P->S6, P->U6);
  P->Gcap_tc = num_sms() * spass_tc_occupancy(P->RS, P->f16 ? 1 : 0);
  P->Gtc = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)P->Gcap_tc, P->U / 4));
  P->f3d = algo == SFSEG_ALGO_AUTO && !P->bin && f3d_supported(P->RT, P->RS);
  P->TX = (int)((sh.W + kF3dTW - 1) / kF3dTW);
  P->TY = (int)((sh.H + f3d_th(std::min(P->RS, kF3dMaxR)) - 1) / f3d_th(std::min(P->RS, kF3dMaxR)));
  P->U3 = P->B * P->TY * P->TX * P->T;
  P->G3 = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms() * f3d_occupancy(P->RT, P->RS), P->U3 / 4));
  // partials: spass [2][B][G], combine/init [B][T*gx], contraction [G2][C+1]
  size_t n_part = std::max<size_t>(2 * (size_t)P->B * std::max({(size_t)P->G * kSpassPartSlots, (size_t)P->Gtc, (size_t)P->G3 * kF3dCW, (size_t)P->G6}),
                                   2 * (size_t)P->BT * P->gx);
  {  // backward contraction: one (C_pad + 1)-vector per (frame, block)
    const int cpad = C <= 1 ? 1 : C <= 2 ? 2 : C <= 4 ? 4 : C <= 8 ? 8 : C <= 16 ? 16 : kMaxC;
    n_part = std::max<size_t>(n_part, (size_t)P->BT * P->gx * (cpad + 1));
  }
  P->n_part = n_part;
  size_t off = align_up(sizeof(WsHeader));
  P->off_sc = off;
  off += align_up(sizeof(double) * kScal * P->B);
  P->off_part = off;
  off += align_up(sizeof(double) * n_part);
  P->off_out = off;
  off += align_up(sizeof(double) * (kMaxC + 1));
  const size_t vb = align_up(sizeof(float) * (size_t)P->vol_elems);
  P->off_F = off;
  off += vb;
  P->off_p = off;
  off += vb;
  P->off_v = off;
  off += vb;
  P->off_p2 = off;  // scratch volume (backward: u = G_xy * v of the tensor-core plain pass)
  off += vb;
  P->ws_fwd = off;
  P->off_xbar = off;
  off += vb;
  P->off_Fbar = off;
  off += vb;
  P->off_x0p = off;
  off += vb;
  P->ws_bwd = off;
  P->tape_nu_bytes = align_up(sizeof(double) * P->B * K);
  P->tape_hdr_bytes = P->tape_nu_bytes + align_up(sizeof(double) * 2 * P->B * K);
  P->tape_bytes = P->tape_hdr_bytes + (size_t)K * vb;
  return SFSEG_OK;
}

// Zero the per-call part of the workspace (counters, per-volume scalars) but NOT the error
// word: device errors are sticky across calls on one workspace until sfseg_sync_status reads
// and clears them (online windows, pipelined solves).  A fresh workspace's header is zeroed
// once by sfseg_workspace_reset.
cudaError_t clear_header(void* ws, size_t bytes, cudaStream_t st) {
  static_assert(offsetof(WsHeader, err) == 0, "error word first");
  return cudaMemsetAsync(static_cast<char*>(ws) + sizeof(unsigned), 0, bytes - sizeof(unsigned), st);
}

template <class T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

sfseg_status check_ws(const void* ws, size_t ws_bytes, size_t need) {
  if (!ws) return SFSEG_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(ws) % kAlign) != 0 || ws_bytes < need) return SFSEG_ERR_WORKSPACE;
  return SFSEG_OK;
}

sfseg_status map_cuda(cudaError_t e) {
  if (e == cudaSuccess) return SFSEG_OK;
  last_cuda_error() = e;
  return SFSEG_ERR_CUDA;
}

void fill_combine(CombineParams& cp, const Plan& P, const float* ch, const float* w_host, float b, int act, void* ws) {
  std::memset(&cp, 0, sizeof(cp));
  cp.ch = ch;
  cp.sc = at<double>(ws, P.off_sc);
  cp.partials = at<double>(ws, P.off_part);
  cp.counter = &at<WsHeader>(ws, 0)->counter[1];
  cp.err = &at<WsHeader>(ws, 0)->err;
  cp.B = (int)P.B;
  cp.C = P.C;
  cp.T = (int)P.T;
  cp.H = (int)P.H;
  cp.W = (int)P.W;
  cp.Wp = (int)P.Wp;
  cp.act = act;
  cp.gx = P.gx;
  cp.in_T = (int)P.T;
  cp.in_t0 = 0;
  cp.bias = b;
  for (int c = 0; c < P.C; ++c) cp.w[c] = w_host[c];
}

void fill_spass_common(SpassParams& sp, const Plan& P, void* ws) {
  sp.F = at<float>(ws, P.off_F);
  sp.sc = at<double>(ws, P.off_sc);
  sp.partials = at<double>(ws, P.off_part);
  sp.counter = &at<WsHeader>(ws, 0)->counter[0];
  sp.err = &at<WsHeader>(ws, 0)->err;
  sp.U = P.U;
  sp.B = (int)P.B;
  sp.T = (int)P.T;
  sp.H = (int)P.H;
  sp.W = (int)P.W;
  sp.Wp = (int)P.Wp;
  sp.S = P.S;
  sp.NB = P.NB;
  sp.G = P.G;
  sp.K = P.K;
  for (int d = 0; d <= P.RS; ++d) sp.g[d] = P.gs[P.RS + d];
}

// Forward spatial pass: the tensor-core kernel when the plan selected it, else the FP32 one.
// Input descriptor of the forward spatial pass over v (box width of the selected kernel).
bool make_spass_fwd_tmap(CUtensorMap* map, const Plan& P, const float* v) {
  return make_volume_tmap(map, v, P.W, P.H, P.BT, P.Wp, P.tc ? spass_tc_boxw(P.RS) : spass_boxw(P.RS));
}
cudaError_t launch_spass_forward(const Plan& P, SpassParams& sp, cudaStream_t st) {
  if (sp.t_cnt > 0) {  // frame-range launch (time-slab schedule): its own unit count and grid
    sp.U = (int64_t)P.B * sp.t_cnt * P.S * P.NB;
    sp.G = (int)std::max<int64_t>(1, std::min<int64_t>(P.tc ? P.Gcap_tc : P.Gcap, sp.U / 4));
  } else {
    sp.U = P.U;
    sp.G = P.tc ? P.Gtc : P.G;
  }
  if (P.tc) return launch_spass_tc(P.RS, sp, sp.G, P.f16 ? 1 : 0, st);
  return launch_spass_fwd(P.RS, sp, sp.G, st);
}

// Temporal pass j of a sequence of (temporal, spatial) pass pairs records max |v| per volume
// for the fp16 spatial pass (slot SC_VMAX + (j & 1); that spatial pass zeroes the other slot).
// Every pair whose spatial pass runs in the fp16 format must go through this.
void set_vslot(TpassParams& tp, SpassParams* sp, const Plan& P, void* ws, int j) {
  tp.vmax = P.f16 ? reinterpret_cast<unsigned*>(at<double>(ws, P.off_sc) + SC_VMAX + (j & 1)) : nullptr;
  if (sp) {
    sp->vslot = j & 1;
    sp->vzero = ((j & 1) ^ 1) + 1;
  }
}

void fill_tpass_common(TpassParams& tp, const Plan& P, void* ws) {
  tp.sc = at<double>(ws, P.off_sc);
  tp.frame4 = P.H * P.Wp / 4;
  tp.T = (int)P.T;
  for (int i = 0; i < 2 * P.RT + 1; ++i) {
    tp.g[i] = P.gt[i];
    uint32_t b;
    std::memcpy(&b, &P.gt[i], 4);
    tp.g2[i] = (unsigned long long)b | ((unsigned long long)b << 32);
  }
}

bool validate_act(int act) { return act == SFSEG_ACT_IDENTITY || act == SFSEG_ACT_SIGMOID; }

bool finite_weights(const float* w, int C, float b) {
  if (!std::isfinite(b)) return false;
  for (int c = 0; c < C; ++c)
    if (!std::isfinite(w[c])) return false;
  return true;
}

// ====================================================================== time-slab sharding
// (SURVEY.md §8(e)).  Each rank owns T_r consecutive frames of every volume.
// Per iteration only the temporal pass reads neighbour frames: the r_t
// boundary frames of the iterate p are exchanged with ranks +-1 after every
// spatial pass, and the per-volume norm partials are summed across ranks
// (fp64) before the scalar finalize.  The same phase functions drive both the
// NCCL transport (one rank per GPU) and an in-process emulation of n ranks on
// one GPU (halo copies + a rank-ordered reduction kernel) used to test the
// decomposition on a single device.
struct SlabOffsets {
  size_t off_hlo, off_hhi, off_slo, off_shi, off_loc, off_glob, total;
};
// after the single-GPU backward region (x_bar, F_bar, x_0): receive halos, send halos (backward),
// local / global sums (2 per volume, or the C + 1 weight-gradient sums)
SlabOffsets slab_offsets(const Plan& P) {
  SlabOffsets o;
  size_t off = P.ws_bwd;
  const size_t hb = align_up(sizeof(float) * (size_t)P.B * P.RT * P.H * P.Wp);
  o.off_hlo = off;
  off += hb;
  o.off_hhi = off;
  off += hb;
  o.off_slo = off;
  off += hb;
  o.off_shi = off;
  off += hb;
  const size_t lb = align_up(sizeof(double) * std::max<size_t>(2 * (size_t)P.B, (size_t)kMaxC + 1));
  o.off_loc = off;
  off += lb;
  o.off_glob = off;
  off += lb;
  o.total = off;
  return o;
}

struct Rank {
  Plan P;
  const float* ch = nullptr;
  const float* x0 = nullptr;
  int in_T = 0, in_t0 = 0;  // channel / x0 buffer frames and this slab's first frame in it
  float* x_out = nullptr;
  int out_T = 0, out_t0 = 0;
  double* stats = nullptr;
  int rayleigh = 0;
  void* tape = nullptr;     // this rank's tape (nu_k global, u_k local frames) or null
  void* ws = nullptr;
  SlabOffsets so;
  bool has_lo = false, has_hi = false;
  float *F = nullptr, *p = nullptr, *v = nullptr, *hlo = nullptr, *hhi = nullptr;
  double *loc = nullptr, *glob = nullptr;
  SpassParams sp;
  TpassParams tp;
};

sfseg_status rank_setup(Rank& r, cudaStream_t st) {
  const Plan& P = r.P;
  r.so = slab_offsets(P);
  r.F = at<float>(r.ws, P.off_F);
  r.p = at<float>(r.ws, P.off_p);
  r.v = at<float>(r.ws, P.off_v);
  r.hlo = at<float>(r.ws, r.so.off_hlo);
  r.hhi = at<float>(r.ws, r.so.off_hhi);
  r.loc = at<double>(r.ws, r.so.off_loc);
  r.glob = at<double>(r.ws, r.so.off_glob);
  SF_CUDA(clear_header(r.ws, P.off_part, st));
  std::memset(&r.sp, 0, sizeof(r.sp));
  // the slab runs the single-GPU plan's spatial pass: tcgen05 (v as fp16 planes, F by TMA) when the
  // plan says so, else the mma.sync / FP32 pass
  if (!(P.tc6 ? make_planes_tmap(&r.sp.tmap, r.v, P.W, P.H, P.BT, P.Wp) : make_spass_fwd_tmap(&r.sp.tmap, P, r.v)))
    return SFSEG_ERR_CUDA;
  if (P.tc6 && !make_volume_tmap(&r.sp.fmap, r.F, P.W, P.H, P.BT, P.Wp, k6M, k6YN)) return SFSEG_ERR_CUDA;
  fill_spass_common(r.sp, P, r.ws);
  if (P.tc6) {
    r.sp.S = P.S6;
    r.sp.NB = P.NB6;
  }
  r.sp.stats = r.stats;
  r.sp.loc = r.loc;
  r.sp.tape_nu = nullptr;   // nu_k is written by the post-allreduce finalize
  std::memset(&r.tp, 0, sizeof(r.tp));
  fill_tpass_common(r.tp, P, r.ws);
  r.tp.src = r.p;
  r.tp.out = r.v;
  r.tp.halo_lo = r.has_lo ? r.hlo : nullptr;
  r.tp.halo_hi = r.has_hi ? r.hhi : nullptr;
  r.tp.lag = 1;   // lagged normalisation (slab_iterations)
  r.sp.lag = 1;
  if (P.tc6) {
    float gsum = 0.f;
    for (int i = 0; i < 2 * P.RT + 1; ++i) gsum += std::fabs(P.gt[i]);
    r.tp.gsum = gsum * (1.f + 1e-5f);   // |v| <= gsum max |p| over the slab's frames and its halos
    r.tp.vexp_out = at<double>(r.ws, P.off_sc) + SC_VEXP;
  }
  return SFSEG_OK;
}

sfseg_status ph_combine(Rank& r, const float* w_host, float b, int act, cudaStream_t st) {
  CombineParams cp;
  fill_combine(cp, r.P, r.ch, w_host, b, act, r.ws);
  cp.x0 = r.x0;
  cp.F = r.F;
  cp.p0 = r.p;
  cp.loc = r.loc;
  cp.in_T = r.in_T;
  cp.in_t0 = r.in_t0;
  if (r.P.tc6) cp.pmax = reinterpret_cast<unsigned*>(at<double>(r.ws, r.P.off_sc) + SC_VMAX);   // max |p_0|
  combine_kernel<<<dim3(r.P.gx, (unsigned)r.P.BT), kEwThreads, 0, st>>>(cp);
  SF_CUDA(after_launch("combine(slab)", st));
  return SFSEG_OK;
}

sfseg_status ph_finalize(Rank& r, int k, cudaStream_t st) {
  FinParams fp;
  fp.glob = r.glob;
  fp.sc = at<double>(r.ws, r.P.off_sc);
  fp.stats = r.stats;
  fp.tape_nu = (k >= 1 && r.tape) ? static_cast<double*>(r.tape) : nullptr;
  fp.err = &at<WsHeader>(r.ws, 0)->err;
  fp.B = (int)r.P.B;
  fp.K = r.P.K;
  fp.k = k;
  fp.rayleigh = r.rayleigh;
  finalize_kernel<<<(unsigned)((r.P.B + 127) / 128), 128, 0, st>>>(fp);
  SF_CUDA(after_launch("finalize(slab)", st));
  return SFSEG_OK;
}

sfseg_status ph_T(Rank& r, int k, cudaStream_t st) {
  const Plan& P = r.P;
  if (P.tc6) {
    // v as two fp16 planes of v 2^e: e from max |p_{k-1}| over the slab's own frames (slot (k-1) & 1,
    // written by the combine / the spatial pass's range launches) and the received halo frames
    double* const scv = at<double>(r.ws, P.off_sc);
    unsigned* const pin = reinterpret_cast<unsigned*>(scv + SC_VMAX + ((k - 1) & 1));
    if (r.tp.halo_lo || r.tp.halo_hi) {
      const long n4 = (long)P.RT * P.H * P.Wp / 4;
      const unsigned gx = (unsigned)std::max<long>(1, std::min<long>(64, n4 / (4 * kEwThreads)));
      halo_absmax_kernel<<<dim3(gx, (unsigned)P.B, 2), kEwThreads, 0, st>>>(
          reinterpret_cast<const float4*>(r.tp.halo_lo), reinterpret_cast<const float4*>(r.tp.halo_hi), n4, pin);
      SF_CUDA(after_launch("halo_absmax(slab)", st));
    }
    r.tp.pmax_in = pin;
    r.tp.pmax_zero = reinterpret_cast<unsigned*>(scv + SC_VMAX + (k & 1));
    ProfScope ps(P.prof, st, PC_TPASS);
    SF_CUDA(launch_tpass_fwd16(P.RT, r.tp, (int)P.B, st));
    SF_CUDA(after_launch("tpass16(slab)", st));
    return SFSEG_OK;
  }
  set_vslot(r.tp, &r.sp, P, r.ws, k);
  ProfScope ps(P.prof, st, PC_TPASS);
  SF_CUDA(launch_tpass_fwd(P.RT, r.tp, (int)P.B, st));
  SF_CUDA(after_launch("tpass(slab)", st));
  return SFSEG_OK;
}

// The spatial-pass launches of one slab iteration as (first frame, count) pairs in launch
// order: the boundary ranges the neighbours need (the first r_t frames when there is a lower
// neighbour, the last r_t when there is an upper one), then the interior.  With no neighbour,
// or a slab too thin for disjoint boundary ranges, one launch covers the slab (counted as
// boundary: the exchange waits for it).  Returns the number of ranges; *n_boundary of them
// precede the halo exchange.
int slab_ranges(int T, int RT, bool has_lo, bool has_hi, int32_t out[6], int32_t* n_boundary) {
  const int lo = has_lo ? RT : 0, hi = has_hi ? RT : 0;
  int n = 0;
  if (lo + hi == 0 || lo + hi >= T) {
    out[0] = 0;
    out[1] = T;
    *n_boundary = 1;
    return 1;
  }
  if (lo > 0) {
    out[2 * n] = 0;
    out[2 * n + 1] = lo;
    ++n;
  }
  if (hi > 0) {
    out[2 * n] = T - hi;
    out[2 * n + 1] = hi;
    ++n;
  }
  *n_boundary = n;
  out[2 * n] = lo;
  out[2 * n + 1] = T - lo - hi;
  return n + 1;
}

// Spatial pass of iteration k over frames [t_lo, t_lo + t_cnt) of every volume; acc: add the
// launch's norm sums to loc (the later launches of one iteration, in a fixed order).
sfseg_status ph_S_range(Rank& r, int k, int t_lo, int t_cnt, int acc, cudaStream_t st) {
  r.sp.out = r.p;
  r.sp.pprev = r.rayleigh ? r.p : nullptr;
  r.sp.tape_u = r.tape ? reinterpret_cast<float*>(static_cast<char*>(r.tape) + r.P.tape_hdr_bytes +
                                                 (size_t)(k - 1) * align_up(sizeof(float) * (size_t)r.P.vol_elems))
                       : nullptr;
  r.sp.k = k;
  r.sp.last = (k == r.P.K) ? 1 : 0;
  r.sp.t_lo = t_lo;
  r.sp.t_cnt = t_cnt;
  r.sp.loc_acc = acc;
  ProfScope ps(r.P.prof, st, PC_SPASS);
  if (r.P.tc6) {
    r.sp.pslot = r.sp.last ? 0 : (k & 1) + 1;   // max |p_k| of the range for the next temporal pass
    r.sp.U = r.P.B * (int64_t)t_cnt * r.P.S6 * r.P.NB6;
    r.sp.G = tc6_grid(r.P.B, r.P.S6, r.sp.U);
    SF_CUDA(launch_spass_tc6(r.P.RS, r.sp, r.sp.G, st));
  } else {
    SF_CUDA(launch_spass_forward(r.P, r.sp, st));
  }
  SF_CUDA(after_launch("spass(slab)", st));
  return SFSEG_OK;
}

// The frames a rank's neighbours need (its r_t boundary frames) are computed first, so the
// halo transfer can run while the interior frames are computed (slab_ranges, exported as
// sfseg_slab_launch_ranges for the host-logic tests).
sfseg_status ph_S_boundary(Rank& r, int k, cudaStream_t st) {
  int32_t rg[6], nb = 0;
  slab_ranges((int)r.P.T, r.P.RT, r.has_lo, r.has_hi, rg, &nb);
  sfseg_status s = SFSEG_OK;
  for (int i = 0; i < nb && s == SFSEG_OK; ++i) s = ph_S_range(r, k, rg[2 * i], rg[2 * i + 1], i > 0 ? 1 : 0, st);
  return s;
}
sfseg_status ph_S_interior(Rank& r, int k, cudaStream_t st) {
  int32_t rg[6], nb = 0;
  const int n = slab_ranges((int)r.P.T, r.P.RT, r.has_lo, r.has_hi, rg, &nb);
  return n > nb ? ph_S_range(r, k, rg[2 * nb], rg[2 * nb + 1], 1, st) : SFSEG_OK;
}

// The comm stream gets the highest priority: the spatial pass fills every SM with one wave
// of CTAs, so the transfer kernels must be placed first when CTA slots free up (between the
// boundary and interior launches) rather than queue behind the interior wave.
cudaError_t create_comm_stream(cudaStream_t* s) {
  int lo = 0, hi = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (e != cudaSuccess) return e;
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, hi);
}

// Streams and events of the overlapped time-slab schedule.  Compute (st): temporal pass,
// boundary spatial pass, interior spatial pass.  Comm (cs): the halo exchange (after the
// boundary pass, overlapping the interior pass) and the norm allreduce + finalize (after
// the interior pass, overlapping the next temporal pass, which does not need s_k: the
// normalisation is lagged into the next spatial pass, TpassParams::lag / SpassParams::lag).
// serial: cs == st and no events (the same kernels in the same per-stream order: bitwise
// the same results).
struct SlabSched {
  cudaStream_t st = nullptr, cs = nullptr;
  cudaEvent_t ev[4] = {};
  bool ovl = false;
  bool own = false;  // stream / events created for this call (single-GPU emulation)
  enum { EV_B = 0, EV_H = 1, EV_I = 2, EV_F = 3 };
  cudaError_t rec(int e, cudaStream_t s) { return ovl ? cudaEventRecord(ev[e], s) : cudaSuccess; }
  cudaError_t wait(cudaStream_t s, int e) { return ovl ? cudaStreamWaitEvent(s, ev[e], 0) : cudaSuccess; }
  cudaError_t init_own(cudaStream_t compute, bool overlap) {
    st = cs = compute;
    ovl = overlap;
    if (!overlap) return cudaSuccess;
    own = true;
    cudaError_t e = create_comm_stream(&cs);
    for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    return e;
  }
  ~SlabSched() {
    if (!own) return;
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
  }
};

// The K iterations of the time-slab forward for the ranks in R (one per process with NCCL,
// all of them in the single-GPU emulation); exch / reduce enqueue the halo exchange and the
// norm allreduce on a stream.  Entered after the combine, its reduction and the first halo
// exchange (all on st); returns with st after the last finalize.
template <class Exch, class Reduce>
sfseg_status slab_iterations(std::vector<Rank*>& R, SlabSched& S, Exch&& exch, Reduce&& reduce) {
  const int K = R[0]->P.K;
  sfseg_status s = SFSEG_OK;
  for (int k = 1; k <= K; ++k) {
    if (k > 1) SF_CUDA(S.wait(S.st, SlabSched::EV_H));  // halos of p_{k-1}
    for (Rank* r : R)
      if ((s = ph_T(*r, k, S.st)) != SFSEG_OK) return s;
    if (k > 1) SF_CUDA(S.wait(S.st, SlabSched::EV_F));  // s_{k-1} for the spatial pass
    for (Rank* r : R)
      if ((s = ph_S_boundary(*r, k, S.st)) != SFSEG_OK) return s;
    if (k < K) {
      SF_CUDA(S.rec(SlabSched::EV_B, S.st));
      SF_CUDA(S.wait(S.cs, SlabSched::EV_B));
      if ((s = exch(S.cs)) != SFSEG_OK) return s;
      SF_CUDA(S.rec(SlabSched::EV_H, S.cs));
    }
    for (Rank* r : R)
      if ((s = ph_S_interior(*r, k, S.st)) != SFSEG_OK) return s;
    SF_CUDA(S.rec(SlabSched::EV_I, S.st));
    SF_CUDA(S.wait(S.cs, SlabSched::EV_I));
    if ((s = reduce(S.cs)) != SFSEG_OK) return s;
    for (Rank* r : R)
      if ((s = ph_finalize(*r, k, S.cs)) != SFSEG_OK) return s;
    SF_CUDA(S.rec(SlabSched::EV_F, S.cs));
  }
  SF_CUDA(S.wait(S.st, SlabSched::EV_F));
  return SFSEG_OK;
}

sfseg_status ph_final(Rank& r, cudaStream_t st) {
  const Plan& P = r.P;
  dim3 grid((unsigned)P.gx, (unsigned)P.BT);
  final_scale_kernel<<<grid, kEwThreads, 0, st>>>(r.p, r.x_out, at<double>(r.ws, P.off_sc), (int)P.T, (int)P.H,
                                                  (int)P.W, (int)P.Wp, r.out_T, r.out_t0);
  SF_CUDA(after_launch("final_scale(slab)", st));
  return SFSEG_OK;
}

// The r_t boundary frames of p with ranks +-1; with_allreduce: the norm partials' fp64
// allreduce goes into the SAME NCCL group (both depend only on the spatial pass just run):
// one grouped launch per iteration instead of two, the sends overlapping the reduction.
sfseg_status nccl_exchange(Rank& r, sfseg_comm* c, cudaStream_t st, bool with_allreduce = false) {
  NcclApi& api = nccl();
  const Plan& P = r.P;
  const size_t fr = (size_t)P.H * P.Wp, n = (size_t)P.RT * fr;
  if (n == 0 && !with_allreduce) return SFSEG_OK;
  if (api.GroupStart() != ncclSuccess) return SFSEG_ERR_NCCL;
  if (with_allreduce &&
      api.AllReduce(r.loc, r.glob, 2 * (size_t)P.B, ncclFloat64, ncclSum, c->comm, st) != ncclSuccess)
    return SFSEG_ERR_NCCL;
  for (int64_t b = 0; b < P.B && n > 0; ++b) {
    float* base = r.p + (size_t)b * P.T * fr;
    if (r.has_lo) {
      if (api.Send(base, n, ncclFloat32, c->rank - 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
      if (api.Recv(r.hlo + b * n, n, ncclFloat32, c->rank - 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
    }
    if (r.has_hi) {
      if (api.Send(base + (P.T - P.RT) * fr, n, ncclFloat32, c->rank + 1, c->comm, st) != ncclSuccess)
        return SFSEG_ERR_NCCL;
      if (api.Recv(r.hhi + b * n, n, ncclFloat32, c->rank + 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
    }
  }
  if (api.GroupEnd() != ncclSuccess) return SFSEG_ERR_NCCL;
  return SFSEG_OK;
}

sfseg_status nccl_allreduce(Rank& r, sfseg_comm* c, cudaStream_t st, size_t n = 0) {
  if (nccl().AllReduce(r.loc, r.glob, n ? n : 2 * (size_t)r.P.B, ncclFloat64, ncclSum, c->comm, st) != ncclSuccess)
    return SFSEG_ERR_NCCL;
  return SFSEG_OK;
}

sfseg_status local_exchange(std::vector<Rank>& R, cudaStream_t st) {
  const int n = (int)R.size();
  for (int i = 0; i < n; ++i) {
    const Plan& P = R[i].P;
    const size_t fr = (size_t)P.H * P.Wp, cnt = (size_t)P.RT * fr;
    for (int64_t b = 0; b < P.B; ++b) {
      if (R[i].has_lo) {
        const Plan& Q = R[i - 1].P;
        SF_CUDA(cudaMemcpyAsync(R[i].hlo + b * cnt, R[i - 1].p + ((size_t)b * Q.T + (Q.T - Q.RT)) * fr,
                                cnt * sizeof(float), cudaMemcpyDeviceToDevice, st));
      }
      if (R[i].has_hi) {
        const Plan& Q = R[i + 1].P;
        SF_CUDA(cudaMemcpyAsync(R[i].hhi + b * cnt, R[i + 1].p + (size_t)b * Q.T * fr, cnt * sizeof(float),
                                cudaMemcpyDeviceToDevice, st));
      }
    }
  }
  return SFSEG_OK;
}

sfseg_status local_allreduce(std::vector<Rank>& R, cudaStream_t st, int n = 0) {
  LocalReduceParams lp;
  std::memset(&lp, 0, sizeof(lp));
  lp.nranks = (int)R.size();
  lp.n = n ? n : 2 * (int)R[0].P.B;
  for (int i = 0; i < lp.nranks; ++i) {
    lp.loc[i] = R[i].loc;
    lp.glob[i] = R[i].glob;
  }
  local_allreduce_kernel<<<(unsigned)((lp.n + 127) / 128), 128, 0, st>>>(lp);
  SF_CUDA(after_launch("local_allreduce", st));
  return SFSEG_OK;
}

// ---------------------------------------------------------------------- time-slab backward
// (SURVEY.md §8(e) c2/c3 row): the single-GPU backward's steps (Appendix A) per slab, with
// (1) the backward temporal pass's r_t-frame halos of F y_bar_k exchanged with ranks +-1
// before every step (bwd_halo_kernel fills the send buffers), (2) the per-step scalars
// <x_{k-1}, x_bar_{k-1}> (and the binarisation sums) allreduced before their finalize, and
// (3) the C + 1 weight-gradient sums allreduced at the end.
struct BwdRank {
  Rank* r = nullptr;
  const float* g = nullptr;   // dL/dx buffer [B][g_T][H][W]
  int g_T = 0, g_t0 = 0;
  float* xbar = nullptr;
  float* Fbar = nullptr;
  float* ubuf = nullptr;
  float* slo = nullptr;
  float* shi = nullptr;
  SpassParams sp;
  TpassParams tp;
  BwdEpiParams be;
};

const float* slab_tape_u(const Rank& r, int i) {
  return reinterpret_cast<const float*>(static_cast<const char*>(r.tape) + r.P.tape_hdr_bytes +
                                        (size_t)i * align_up(sizeof(float) * (size_t)r.P.vol_elems));
}

sfseg_status bw_setup(BwdRank& q, cudaStream_t st) {
  Rank& r = *q.r;
  const Plan& P = r.P;
  q.xbar = at<float>(r.ws, P.off_xbar);
  q.Fbar = at<float>(r.ws, P.off_Fbar);
  q.ubuf = at<float>(r.ws, P.off_p2);
  q.slo = at<float>(r.ws, r.so.off_slo);
  q.shi = at<float>(r.ws, r.so.off_shi);
  std::memset(&q.sp, 0, sizeof(q.sp));
  if (!make_spass_fwd_tmap(&q.sp.tmap, P, r.v)) return SFSEG_ERR_CUDA;
  fill_spass_common(q.sp, P, r.ws);
  q.sp.plain = 1;
  q.sp.out = q.ubuf;
  std::memset(&q.tp, 0, sizeof(q.tp));
  fill_tpass_common(q.tp, P, r.ws);
  q.tp.src = q.xbar;
  q.tp.F = r.F;
  q.tp.out = r.v;
  q.tp.halo_lo = r.has_lo ? r.hlo : nullptr;
  q.tp.halo_hi = r.has_hi ? r.hhi : nullptr;
  std::memset(&q.be, 0, sizeof(q.be));
  q.be.u = q.ubuf;
  q.be.F = r.F;
  q.be.xbar = q.xbar;
  q.be.Fbar = q.Fbar;
  q.be.sc = at<double>(r.ws, P.off_sc);
  q.be.tape_nu = static_cast<const double*>(r.tape);
  q.be.tape_bin = reinterpret_cast<const double*>(static_cast<const char*>(r.tape) + P.tape_nu_bytes);
  q.be.partials = at<double>(r.ws, P.off_part);
  q.be.counter = &at<WsHeader>(r.ws, 0)->counter[0];
  q.be.loc = r.loc;
  q.be.B = (int)P.B;
  q.be.T = (int)P.T;
  q.be.H = (int)P.H;
  q.be.W = (int)P.W;
  q.be.Wp = (int)P.Wp;
  q.be.gx = P.gx;
  q.be.K = P.K;
  return SFSEG_OK;
}

sfseg_status bw_init(BwdRank& q, cudaStream_t st) {
  Rank& r = *q.r;
  const Plan& P = r.P;
  BwdInitParams ip;
  std::memset(&ip, 0, sizeof(ip));
  ip.g = q.g;
  ip.F = r.F;
  ip.uK1 = slab_tape_u(r, P.K - 1);
  ip.xbar = q.xbar;
  ip.Fbar = q.Fbar;
  ip.tape_nu = static_cast<const double*>(r.tape);
  ip.tape_bin = q.be.tape_bin;
  ip.sc = at<double>(r.ws, P.off_sc);
  ip.partials = at<double>(r.ws, P.off_part);
  ip.counter = &at<WsHeader>(r.ws, 0)->counter[2];
  ip.loc = r.loc;
  ip.B = (int)P.B;
  ip.T = (int)P.T;
  ip.H = (int)P.H;
  ip.W = (int)P.W;
  ip.Wp = (int)P.Wp;
  ip.K = P.K;
  ip.gx = P.gx;
  ip.g_T = q.g_T;
  ip.g_t0 = q.g_t0;
  bwd_init_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(ip);
  SF_CUDA(after_launch("bwd_init(slab)", st));
  return SFSEG_OK;
}

sfseg_status bw_init_fin(BwdRank& q, cudaStream_t st) {
  Rank& r = *q.r;
  BwdInitFinParams fp;
  fp.glob = r.glob;
  fp.sc = at<double>(r.ws, r.P.off_sc);
  fp.tape_nu = static_cast<const double*>(r.tape);
  fp.tape_bin = q.be.tape_bin;
  fp.kappa = 0.f;
  fp.B = (int)r.P.B;
  fp.K = r.P.K;
  bwd_init_finalize_kernel<<<(unsigned)((r.P.B + 127) / 128), 128, 0, st>>>(fp);
  SF_CUDA(after_launch("bwd_init_finalize", st));
  return SFSEG_OK;
}

sfseg_status bw_halo(BwdRank& q, int k, cudaStream_t st) {
  Rank& r = *q.r;
  const Plan& P = r.P;
  if (!(r.has_lo || r.has_hi) || P.RT == 0) return SFSEG_OK;
  BwdHaloParams hp;
  hp.xbar = q.xbar;
  hp.F = r.F;
  hp.u1 = slab_tape_u(r, k - 1);
  hp.sc = at<double>(r.ws, P.off_sc);
  hp.send_lo = q.slo;
  hp.send_hi = q.shi;
  hp.frame = P.H * P.Wp;
  hp.T = (int)P.T;
  hp.RT = P.RT;
  bwd_halo_kernel<<<dim3(8, (unsigned)(2 * P.RT), (unsigned)P.B), kEwThreads, 0, st>>>(hp);
  SF_CUDA(after_launch("bwd_halo", st));
  return SFSEG_OK;
}

sfseg_status bw_step(BwdRank& q, int k, cudaStream_t st) {
  Rank& r = *q.r;
  const Plan& P = r.P;
  q.tp.u1 = slab_tape_u(r, k - 1);
  set_vslot(q.tp, &q.sp, P, r.ws, k);
  {
    ProfScope ps(P.prof, st, PC_BWD);
    SF_CUDA(launch_tpass_bwd(P.RT, q.tp, (int)P.B, st));
    SF_CUDA(after_launch("tpass_bwd(slab)", st));
  }
  q.sp.k = k;
  {
    ProfScope ps(P.prof, st, PC_BWD);
    SF_CUDA(launch_spass_forward(P, q.sp, st));
    SF_CUDA(after_launch("spass(plain, slab bwd)", st));
  }
  q.be.u1 = slab_tape_u(r, k - 1);
  q.be.u2 = k >= 2 ? slab_tape_u(r, k - 2) : nullptr;
  q.be.k = k;
  q.be.kappa_prev = 0.f;
  {
    ProfScope ps(P.prof, st, PC_BWD);
    bwd_epi_kernel<<<dim3((unsigned)P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(q.be);
    SF_CUDA(after_launch("bwd_epi(slab)", st));
  }
  return SFSEG_OK;
}

sfseg_status bw_step_fin(BwdRank& q, int k, cudaStream_t st) {
  Rank& r = *q.r;
  BwdStepFinParams fp;
  fp.glob = r.glob;
  fp.sc = at<double>(r.ws, r.P.off_sc);
  fp.tape_nu = static_cast<const double*>(r.tape);
  fp.tape_bin = q.be.tape_bin;
  fp.kappa_prev = 0.f;
  fp.B = (int)r.P.B;
  fp.K = r.P.K;
  fp.k = k;
  bwd_step_finalize_kernel<<<(unsigned)((r.P.B + 127) / 128), 128, 0, st>>>(fp);
  SF_CUDA(after_launch("bwd_step_finalize", st));
  return SFSEG_OK;
}

// dw, db of this slab into loc[0..C] (the caller allreduces them into glob)
sfseg_status bw_contract(BwdRank& q, const float* w_host, float b, int act, cudaStream_t st) {
  Rank& r = *q.r;
  const Plan& P = r.P;
  ContractParams cc;
  std::memset(&cc, 0, sizeof(cc));
  cc.ch = r.ch;
  cc.Fbar = q.Fbar;
  cc.xbar0 = q.xbar;   // x_0 = F
  cc.partials = at<double>(r.ws, P.off_part);
  cc.out = r.loc;
  cc.counter = &at<WsHeader>(r.ws, 0)->counter[3];
  cc.B = (int)P.B;
  cc.C = P.C;
  cc.T = (int)P.T;
  cc.H = (int)P.H;
  cc.W = (int)P.W;
  cc.Wp = (int)P.Wp;
  cc.in_T = r.in_T;
  cc.in_t0 = r.in_t0;
  cc.act = act;
  cc.bias = b;
  for (int c = 0; c < P.C; ++c) cc.w[c] = w_host[c];
  const dim3 G2((unsigned)P.gx, (unsigned)P.BT);
  const int C = P.C;
  if (C <= 1) contract_kernel<1><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 2) contract_kernel<2><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 4) contract_kernel<4><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 8) contract_kernel<8><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 16) contract_kernel<16><<<G2, kEwThreads, 0, st>>>(cc);
  else contract_kernel<kMaxC><<<G2, kEwThreads, 0, st>>>(cc);
  SF_CUDA(after_launch("contract(slab)", st));
  return SFSEG_OK;
}

// in-process halo exchange of the backward send buffers (emulated ranks)
sfseg_status local_bwd_exchange(std::vector<Rank>& R, std::vector<BwdRank>& Q, cudaStream_t st) {
  for (size_t i = 0; i < R.size(); ++i) {
    const Plan& P = R[i].P;
    const size_t n = sizeof(float) * (size_t)P.B * P.RT * P.H * P.Wp;
    if (R[i].has_lo) SF_CUDA(cudaMemcpyAsync(R[i].hlo, Q[i - 1].shi, n, cudaMemcpyDeviceToDevice, st));
    if (R[i].has_hi) SF_CUDA(cudaMemcpyAsync(R[i].hhi, Q[i + 1].slo, n, cudaMemcpyDeviceToDevice, st));
  }
  return SFSEG_OK;
}

sfseg_status nccl_bwd_exchange(Rank& r, BwdRank& q, sfseg_comm* c, cudaStream_t st) {
  NcclApi& api = nccl();
  const Plan& P = r.P;
  const size_t n = (size_t)P.B * P.RT * P.H * P.Wp;
  if (n == 0) return SFSEG_OK;
  if (api.GroupStart() != ncclSuccess) return SFSEG_ERR_NCCL;
  if (r.has_lo) {
    if (api.Send(q.slo, n, ncclFloat32, c->rank - 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
    if (api.Recv(r.hlo, n, ncclFloat32, c->rank - 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
  }
  if (r.has_hi) {
    if (api.Send(q.shi, n, ncclFloat32, c->rank + 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
    if (api.Recv(r.hhi, n, ncclFloat32, c->rank + 1, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
  }
  if (api.GroupEnd() != ncclSuccess) return SFSEG_ERR_NCCL;
  return SFSEG_OK;
}

// Every rank's argument check ends in one agreement allreduce (max of the status codes,
// on the communicator's own device word) BEFORE the first data-path collective, so a rank
// that fails validation cannot leave its peers blocked in ncclAllReduce / ncclSend.
// Syncs `st` once (the host needs the agreed status).
sfseg_status dist_agree(sfseg_comm* c, sfseg_status mine, cudaStream_t st) {
  NcclApi& api = nccl();
  if (!api.ok || !c->flag) return SFSEG_ERR_NCCL;
  int32_t h = (int32_t)mine;
  SF_CUDA(cudaMemcpyAsync(c->flag, &h, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  if (api.AllReduce(c->flag, c->flag, 1, ncclInt32, ncclMax, c->comm, st) != ncclSuccess) return SFSEG_ERR_NCCL;
  SF_CUDA(cudaMemcpyAsync(&h, c->flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  return (sfseg_status)h;
}

// One rank of an NCCL-connected time-slab solve.
sfseg_status dist_power_iterate(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                sfseg_shape sh, sfseg_gauss gauss, int32_t K, const float* x0, float* x_out,
                                float* F_out, double* stats, int32_t want_rayleigh, void* tape, void* ws,
                                size_t ws_bytes, const sfseg_dist* dist, const sfseg_options* opt, void* stream) {
  if (!dist->comm || !dist->comm->comm) return SFSEG_ERR_INVALID_ARGUMENT;  // no communicator to agree on
  sfseg_comm* c = dist->comm;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // ---- local validation: no early return before the agreement
  Plan P;
  sfseg_status s = SFSEG_OK;
  if (!ch || !w_host || !x_out || !validate_act(act)) s = SFSEG_ERR_INVALID_ARGUMENT;
  else if ((s = make_plan(sh, C, gauss, K, &P, opt)) != SFSEG_OK) {
  } else if (!finite_weights(w_host, C, b)) s = SFSEG_ERR_INVALID_ARGUMENT;
  else if (F_out || P.bin) s = SFSEG_ERR_UNSUPPORTED;  // F export / binarisation: single-GPU only
  else if (tape && (reinterpret_cast<uintptr_t>(tape) % kAlign) != 0) s = SFSEG_ERR_WORKSPACE;
  else if (dist->t_offset < 0 || dist->t_offset + P.T > dist->T_global) s = SFSEG_ERR_SHAPE;
  else if (c->nranks > 1 && P.T < P.RT) s = SFSEG_ERR_SHAPE;  // the halo must come from one neighbour
  else s = check_ws(ws, ws_bytes, slab_offsets(P).total);
  const sfseg_status agreed = dist_agree(c, s, st);
  if (s != SFSEG_OK) return s;
  if (agreed != SFSEG_OK) return agreed;  // a peer failed its validation: nobody starts the solve
  Rank r;
  r.P = P;
  r.ch = ch;
  r.x0 = x0;
  r.in_T = (int)P.T;
  r.x_out = x_out;
  r.out_T = (int)P.T;
  r.stats = stats;
  r.rayleigh = want_rayleigh;
  r.ws = ws;
  r.tape = tape;
  r.has_lo = dist->t_offset > 0 && c->rank > 0;
  r.has_hi = dist->t_offset + P.T < dist->T_global && c->rank < c->nranks - 1;
  if ((s = rank_setup(r, st)) != SFSEG_OK) return s;
  if ((s = ph_combine(r, w_host, b, act, st)) != SFSEG_OK) return s;
  if ((s = nccl_allreduce(r, c, st)) != SFSEG_OK) return s;
  if ((s = ph_finalize(r, 0, st)) != SFSEG_OK) return s;
  if ((s = nccl_exchange(r, c, st)) != SFSEG_OK) return s;
  SlabSched S;
  S.st = S.cs = st;
  if (!(opt && opt->slab_schedule == SFSEG_SLAB_SERIAL) && c->cs) {  // overlapped on the comm's stream
    S.cs = c->cs;
    S.ovl = true;
    for (int i = 0; i < 4; ++i) S.ev[i] = c->ev[i];
  }
  std::vector<Rank*> R{&r};
  if ((s = slab_iterations(
           R, S, [&](cudaStream_t q) { return nccl_exchange(r, c, q); },
           [&](cudaStream_t q) { return nccl_allreduce(r, c, q); })) != SFSEG_OK)
    return s;
  return ph_final(r, st);
}

// One rank of an NCCL-connected time-slab backward (the tape from a dist forward).
sfseg_status dist_power_iterate_backward(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                         sfseg_shape sh, sfseg_gauss gauss, int32_t K, const float* x0,
                                         const void* tape, const float* dL_dx, double* dL_dw_host,
                                         double* dL_db_host, void* ws, size_t ws_bytes, const sfseg_dist* dist,
                                         const sfseg_options* opt, void* stream) {
  if (!dist->comm || !dist->comm->comm) return SFSEG_ERR_INVALID_ARGUMENT;
  sfseg_comm* c = dist->comm;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Plan P;
  sfseg_status s = SFSEG_OK;
  if (!ch || !w_host || !tape || !dL_dx || !dL_dw_host || !validate_act(act)) s = SFSEG_ERR_INVALID_ARGUMENT;
  else if ((s = make_plan(sh, C, gauss, K, &P, opt)) != SFSEG_OK) {
  } else if (!finite_weights(w_host, C, b)) s = SFSEG_ERR_INVALID_ARGUMENT;
  else if (x0 || P.bin) s = SFSEG_ERR_UNSUPPORTED;   // user x_0 / binarisation: single-GPU backward only
  else if (dist->t_offset < 0 || dist->t_offset + P.T > dist->T_global) s = SFSEG_ERR_SHAPE;
  else if (c->nranks > 1 && P.T < P.RT) s = SFSEG_ERR_SHAPE;
  else if ((reinterpret_cast<uintptr_t>(tape) % kAlign) != 0) s = SFSEG_ERR_WORKSPACE;
  else s = check_ws(ws, ws_bytes, slab_offsets(P).total);
  const sfseg_status agreed = dist_agree(c, s, st);
  if (s != SFSEG_OK) return s;
  if (agreed != SFSEG_OK) return agreed;
  Rank r;
  r.P = P;
  r.ch = ch;
  r.in_T = (int)P.T;
  r.ws = ws;
  r.tape = const_cast<void*>(tape);
  r.has_lo = dist->t_offset > 0 && c->rank > 0;
  r.has_hi = dist->t_offset + P.T < dist->T_global && c->rank < c->nranks - 1;
  if ((s = rank_setup(r, st)) != SFSEG_OK) return s;
  BwdRank q;
  q.r = &r;
  q.g = dL_dx;
  q.g_T = (int)P.T;
  if ((s = bw_setup(q, st)) != SFSEG_OK) return s;
  if ((s = ph_combine(r, w_host, b, act, st)) != SFSEG_OK) return s;
  if ((s = bw_init(q, st)) != SFSEG_OK) return s;
  if ((s = nccl_allreduce(r, c, st)) != SFSEG_OK) return s;
  if ((s = bw_init_fin(q, st)) != SFSEG_OK) return s;
  for (int k = K; k >= 1; --k) {
    if ((s = bw_halo(q, k, st)) != SFSEG_OK) return s;
    if ((s = nccl_bwd_exchange(r, q, c, st)) != SFSEG_OK) return s;
    if ((s = bw_step(q, k, st)) != SFSEG_OK) return s;
    if ((s = nccl_allreduce(r, c, st)) != SFSEG_OK) return s;
    if ((s = bw_step_fin(q, k, st)) != SFSEG_OK) return s;
  }
  if ((s = bw_contract(q, w_host, b, act, st)) != SFSEG_OK) return s;
  if ((s = nccl_allreduce(r, c, st, (size_t)C + 1)) != SFSEG_OK) return s;
  std::vector<double> out(C + 1);
  SF_CUDA(cudaMemcpyAsync(out.data(), r.glob, sizeof(double) * (C + 1), cudaMemcpyDeviceToHost, st));
  s = sfseg_sync_status(ws, stream);
  for (int i = 0; i < C; ++i) dL_dw_host[i] = out[i];
  if (dL_db_host) *dL_db_host = out[C];
  return s;
}

// Slab boundaries: slab i of n covers frames [i*T/n, (i+1)*T/n) (uneven when n does not divide T).
inline int64_t slab_start(int64_t T, int n, int i) { return (T * i) / n; }

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* sfseg_status_string(sfseg_status s) {
  switch (s) {
    case SFSEG_OK: return "ok";
    case SFSEG_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SFSEG_ERR_SHAPE: return "invalid shape or radius";
    case SFSEG_ERR_WORKSPACE: return "workspace too small or misaligned";
    case SFSEG_ERR_DEGENERATE: return "degenerate iterate (zero norm)";
    case SFSEG_ERR_NONFINITE: return "non-finite value reached a norm";
    case SFSEG_ERR_CUDA: return "CUDA error";
    case SFSEG_ERR_NCCL: return "NCCL error";
    case SFSEG_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

int32_t sfseg_abi_version(void) { return SFSEG_ABI_VERSION; }

const char* sfseg_last_cuda_error(void) { return cudaGetErrorString(last_cuda_error()); }

sfseg_status sfseg_forward_path(sfseg_shape sh, sfseg_gauss g, int32_t algo, int32_t* info) {
  if (!info) return SFSEG_ERR_INVALID_ARGUMENT;
  Plan P;
  const sfseg_options opt{algo, nullptr};
  sfseg_status s = make_plan(sh, 1, g, 1, &P, &opt);
  if (s != SFSEG_OK) return s;
  info[0] = P.f3d ? SFSEG_PATH_FUSED_3D
            : P.tc6 ? SFSEG_PATH_TWO_PASS_TCGEN05
            : P.f16 ? SFSEG_PATH_TWO_PASS_TC_F16
            : P.tc  ? SFSEG_PATH_TWO_PASS_TC
                    : SFSEG_PATH_TWO_PASS_FP32;
  info[1] = P.RT;
  info[2] = P.RS;
  return SFSEG_OK;
}


void sfseg_max_radii(int32_t* rs, int32_t* rt) {
  if (rs) *rs = kMaxRS;
  if (rt) *rt = kMaxRT;
}

sfseg_status sfseg_workspace_bytes(sfseg_shape shape, int32_t C, sfseg_gauss gauss, int32_t K, int32_t want_tape,
                                   const sfseg_dist* dist, size_t* ws_bytes, size_t* tape_bytes) {
  if (!ws_bytes) return SFSEG_ERR_INVALID_ARGUMENT;
  Plan P;
  sfseg_status st = make_plan(shape, C, gauss, K, &P);
  if (st != SFSEG_OK) return st;
  *ws_bytes = dist ? slab_offsets(P).total : (want_tape ? P.ws_bwd : P.ws_fwd);
  if (tape_bytes) *tape_bytes = want_tape ? P.tape_bytes : 0;
  return SFSEG_OK;
}

sfseg_status sfseg_combine_channels(const float* ch, int32_t C, sfseg_shape sh, const float* w_host, float b,
                                    int32_t act, float* F, void* stream) {
  if (!ch || !w_host || !F || C < 1 || !validate_act(act)) return SFSEG_ERR_INVALID_ARGUMENT;
  if (C > kMaxC) return SFSEG_ERR_UNSUPPORTED;
  if (sh.B < 1 || sh.T < 1 || sh.H < 1 || sh.W < 1) return SFSEG_ERR_SHAPE;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  // Dense-to-dense combine: reuse the combine kernel with Wp = W and no side outputs.
  CombineParams cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.ch = ch;
  cp.F = F;
  cp.B = (int)sh.B;
  cp.C = C;
  cp.T = (int)sh.T;
  cp.H = (int)sh.H;
  cp.W = (int)sh.W;
  cp.Wp = (int)sh.W;
  cp.act = act;
  cp.in_T = (int)sh.T;
  cp.in_t0 = 0;
  cp.bias = b;
  for (int c = 0; c < C; ++c) cp.w[c] = w_host[c];
  cp.gx = ew_gx(sh.H, sh.B * sh.T);
  cp.partials = nullptr;  // no ||x_0|| reduction for the standalone combine
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  combine_kernel<<<dim3(cp.gx, (unsigned)(sh.B * sh.T)), kEwThreads, 0, st>>>(cp);
  return map_cuda(cudaGetLastError());
}

sfseg_status sfseg_power_iterate(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                 sfseg_shape sh, sfseg_gauss gauss, int32_t K, const float* x0, float* x_out,
                                 float* F_out, double* stats, int32_t want_rayleigh, void* tape, void* ws,
                                 size_t ws_bytes, const sfseg_dist* dist, void* stream) {
  return sfseg_power_iterate_ex(ch, C, w_host, b, act, sh, gauss, K, x0, x_out, F_out, stats, want_rayleigh, tape,
                                ws, ws_bytes, dist, nullptr, stream);
}

sfseg_status sfseg_power_iterate_ex(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                    sfseg_shape sh, sfseg_gauss gauss, int32_t K, const float* x0, float* x_out,
                                    float* F_out, double* stats, int32_t want_rayleigh, void* tape, void* ws,
                                    size_t ws_bytes, const sfseg_dist* dist, const sfseg_options* opt,
                                    void* stream) {
  if (dist) return dist_power_iterate(ch, C, w_host, b, act, sh, gauss, K, x0, x_out, F_out, stats, want_rayleigh,
                                      tape, ws, ws_bytes, dist, opt, stream);
  if (!ch || !w_host || !x_out || !validate_act(act)) return SFSEG_ERR_INVALID_ARGUMENT;
  Plan P;
  sfseg_status s = make_plan(sh, C, gauss, K, &P, opt);
  if (s != SFSEG_OK) return s;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  if ((s = check_ws(ws, ws_bytes, P.ws_fwd)) != SFSEG_OK) return s;
  if (tape && (reinterpret_cast<uintptr_t>(tape) % kAlign) != 0) return SFSEG_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  // header + per-volume scalars start from zero
  SF_CUDA(clear_header(ws, P.off_part, st));

  float* F = at<float>(ws, P.off_F);
  float* p = at<float>(ws, P.off_p);
  float* v = at<float>(ws, P.off_v);
  double* tape_nu = tape ? static_cast<double*>(tape) : nullptr;
  auto tape_u = [&](int i) -> float* {
    return reinterpret_cast<float*>(static_cast<char*>(tape) + P.tape_hdr_bytes +
                                    (size_t)i * align_up(sizeof(float) * (size_t)P.vol_elems));
  };

  // (a1) combine -> F, p_0 = F * x_0, ||x_0||
  CombineParams cp;
  fill_combine(cp, P, ch, w_host, b, act, ws);
  cp.x0 = x0;
  cp.F = F;
  cp.p0 = p;
  cp.F_out = F_out;
  if (P.tc6) cp.pmax = reinterpret_cast<unsigned*>(at<double>(ws, P.off_sc) + SC_VMAX);   // max |p_0|
  {
    ProfScope ps(P.prof, st, PC_ONCE);
    combine_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(cp);
    SF_CUDA(after_launch("combine", st));
  }

  if (P.f3d) {
    // single-pass fused 3D iteration: p_{k-1} -> p_k ping-pong between the p and v buffers
    F3dParams fp;
    std::memset(&fp, 0, sizeof(fp));
    CUtensorMap map_p, map_v;
    if (!make_volume_tmap(&map_p, p, P.W, P.H, P.BT, P.Wp, f3d_boxw(P.RS))) return SFSEG_ERR_CUDA;
    if (!make_volume_tmap(&map_v, v, P.W, P.H, P.BT, P.Wp, f3d_boxw(P.RS))) return SFSEG_ERR_CUDA;
    if (!make_volume_tmap(&fp.fmap, F, P.W, P.H, P.BT, P.Wp, kF3dTW, f3d_th(P.RS))) return SFSEG_ERR_CUDA;
    fp.F = F;
    fp.sc = at<double>(ws, P.off_sc);
    fp.partials = at<double>(ws, P.off_part);
    fp.counter = &at<WsHeader>(ws, 0)->counter[0];
    fp.err = &at<WsHeader>(ws, 0)->err;
    fp.stats = stats;
    fp.tape_nu = tape_nu;
    fp.U = P.U3;
    fp.B = (int)P.B;
    fp.T = (int)P.T;
    fp.H = (int)P.H;
    fp.W = (int)P.W;
    fp.Wp = (int)P.Wp;
    fp.TX = P.TX;
    fp.TY = P.TY;
    fp.G = P.G3;
    fp.K = K;
    fp.rayleigh = want_rayleigh ? 1 : 0;
    for (int i = 0; i < 2 * P.RT + 1; ++i) fp.gt[i] = P.gt[i];
    for (int d = 0; d <= P.RS; ++d) fp.gs[d] = P.gs[P.RS + d];
    float* last_out = p;
    for (int k = 1; k <= K; ++k) {
      const bool odd = (k & 1) != 0;
      fp.tmap = odd ? map_p : map_v;
      fp.out = odd ? v : p;
      fp.tape_u = tape ? tape_u(k - 1) : nullptr;
      fp.k = k;
      fp.last = (k == K) ? 1 : 0;
      ProfScope ps(P.prof, st, PC_F3D);
      SF_CUDA(launch_f3d(P.RT, P.RS, fp, P.G3, st));
      SF_CUDA(after_launch("f3d", st));
      last_out = fp.out;
    }
    dim3 grid((unsigned)P.gx, (unsigned)P.BT);
    final_scale_kernel<<<grid, kEwThreads, 0, st>>>(last_out, x_out, at<double>(ws, P.off_sc), (int)P.T, (int)P.H,
                                                    (int)P.W, (int)P.Wp, (int)P.T, 0);
    SF_CUDA(after_launch("final_scale", st));
    return SFSEG_OK;
  }

  SpassParams sp;
  std::memset(&sp, 0, sizeof(sp));
  if (!(P.tc6 ? make_planes_tmap(&sp.tmap, v, P.W, P.H, P.BT, P.Wp) : make_spass_fwd_tmap(&sp.tmap, P, v)))
    return SFSEG_ERR_CUDA;
  if (P.tc6 && !make_volume_tmap(&sp.fmap, F, P.W, P.H, P.BT, P.Wp, k6M, k6YN)) return SFSEG_ERR_CUDA;
  fill_spass_common(sp, P, ws);
  sp.stats = stats;
  sp.tape_nu = tape_nu;
  TpassParams tp;
  std::memset(&tp, 0, sizeof(tp));
  fill_tpass_common(tp, P, ws);
  tp.src = p;
  tp.out = v;
  double* const scv = at<double>(ws, P.off_sc);
  auto pmax_slot = [&](int j) { return reinterpret_cast<unsigned*>(scv + SC_VMAX + (j & 1)); };
  if (P.tc6) {
    float gsum = 0.f;
    for (int i = 0; i < 2 * P.RT + 1; ++i) gsum += std::fabs(P.gt[i]);
    tp.gsum = gsum * (1.f + 1e-5f);   // |v| <= s gsum max |p| with margin for rounding
    tp.vexp_out = scv + SC_VEXP;
    sp.S = P.S6;
    sp.NB = P.NB6;
    sp.U = P.U6;
    sp.G = P.G6;
  }

  for (int k = 1; k <= K; ++k) {
    // (a2)+(a3) v = s_{k-1} * G_t * p_{k-1}
    if (P.tc6) {   // as two fp16 planes of v 2^e (e from max |p_{k-1}|, slot (k-1) & 1)
      tp.pmax_in = pmax_slot(k - 1);
      tp.pmax_zero = pmax_slot(k);
      ProfScope ps(P.prof, st, PC_TPASS);
      SF_CUDA(launch_tpass_fwd16(P.RT, tp, (int)P.B, st));
      SF_CUDA(after_launch("tpass_fwd16", st));
    } else {
      set_vslot(tp, &sp, P, ws, k);
      ProfScope ps(P.prof, st, PC_TPASS);
      SF_CUDA(launch_tpass_fwd(P.RT, tp, (int)P.B, st));
      SF_CUDA(after_launch("tpass_fwd", st));
    }
    // (a4)-(a7) u = G_y G_x v ; y_k = F u ; p_k = F y_k ; ||y_k||, <p_{k-1}, u>
    const float kap = P.kappa(k);
    sp.out = p;
    sp.pprev = want_rayleigh ? p : nullptr;
    sp.tape_u = tape ? tape_u(k - 1) : nullptr;
    sp.k = k;
    sp.last = (k == K || kap > 0.f) ? 1 : 0;   // a binarised iteration stores y_k itself
    if (P.tc6) {
      sp.pslot = sp.last ? 0 : (k & 1) + 1;   // max |p_k| for the next temporal pass
      ProfScope ps(P.prof, st, PC_SPASS);
      SF_CUDA(launch_spass_tc6(P.RS, sp, P.G6, st));
      SF_CUDA(after_launch("spass_tc6", st));
    } else {
      ProfScope ps(P.prof, st, PC_SPASS);
      SF_CUDA(launch_spass_forward(P, sp, st));
      SF_CUDA(after_launch("spass_fwd", st));
    }
    if (kap > 0.f) {
      // Alg.1 STEP 3 (row f2): theta_k, then x_k = sigma(kappa (y_k / nu_k - theta_k)) and the
      // next stored iterate p_k = F x_k (scale 1); the output itself after the last iteration
      BinParams bp;
      std::memset(&bp, 0, sizeof(bp));
      bp.y = p;
      bp.U = F;
      bp.a = (k == K) ? nullptr : p;
      bp.x_dense = (k == K) ? x_out : nullptr;
      bp.sc = at<double>(ws, P.off_sc);
      bp.partials = at<double>(ws, P.off_part);
      bp.counter = &at<WsHeader>(ws, 0)->counter[1];
      bp.err = &at<WsHeader>(ws, 0)->err;
      bp.B = (int)P.B;
      bp.T = (int)P.T;
      bp.H = (int)P.H;
      bp.W = (int)P.W;
      bp.Wp = (int)P.Wp;
      bp.gx = P.gx;
      bp.kappa = kap;
      bp.tape_bin = tape ? reinterpret_cast<double*>(static_cast<char*>(tape) + P.tape_nu_bytes) : nullptr;
      bp.K = K;
      bp.k = k;
      ProfScope ps(P.prof, st, PC_ONCE);
      pos_stats_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(bp);
      SF_CUDA(after_launch("pos_stats", st));
      binarize_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(bp);
      SF_CUDA(after_launch("binarize", st));
    }
  }
  if (P.kappa(K) > 0.f) return SFSEG_OK;   // x_out = the last binarised iterate (values in (0,1))
  // (a8) x_K = y_K / nu_K (dense output)
  {
    ProfScope ps(P.prof, st, PC_ONCE);
    dim3 grid((unsigned)P.gx, (unsigned)P.BT);
    final_scale_kernel<<<grid, kEwThreads, 0, st>>>(p, x_out, at<double>(ws, P.off_sc), (int)P.T, (int)P.H, (int)P.W,
                                                    (int)P.Wp, (int)P.T, 0);
    SF_CUDA(after_launch("final_scale", st));
  }
  return SFSEG_OK;
}

sfseg_status sfseg_power_iterate_backward(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                          sfseg_shape sh, sfseg_gauss gauss, int32_t K, const float* x0,
                                          const void* tape, const float* dL_dx, double* dL_dw_host,
                                          double* dL_db_host, void* ws, size_t ws_bytes, const sfseg_dist* dist,
                                          void* stream) {
  return sfseg_power_iterate_backward_ex(ch, C, w_host, b, act, sh, gauss, K, x0, tape, dL_dx, dL_dw_host,
                                         dL_db_host, ws, ws_bytes, dist, nullptr, stream);
}

sfseg_status sfseg_power_iterate_backward_ex(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                             sfseg_shape sh, sfseg_gauss gauss, int32_t K, const float* x0,
                                             const void* tape, const float* dL_dx, double* dL_dw_host,
                                             double* dL_db_host, void* ws, size_t ws_bytes, const sfseg_dist* dist,
                                             const sfseg_options* opt, void* stream) {
  if (dist) return dist_power_iterate_backward(ch, C, w_host, b, act, sh, gauss, K, x0, tape, dL_dx, dL_dw_host,
                                               dL_db_host, ws, ws_bytes, dist, opt, stream);
  if (!ch || !w_host || !tape || !dL_dx || !dL_dw_host || !validate_act(act)) return SFSEG_ERR_INVALID_ARGUMENT;
  Plan P;
  sfseg_status s = make_plan(sh, C, gauss, K, &P, opt);
  if (s != SFSEG_OK) return s;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  if ((s = check_ws(ws, ws_bytes, P.ws_bwd)) != SFSEG_OK) return s;
  if ((reinterpret_cast<uintptr_t>(tape) % kAlign) != 0) return SFSEG_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SF_CUDA(clear_header(ws, P.off_part, st));

  float* F = at<float>(ws, P.off_F);
  float* v = at<float>(ws, P.off_v);
  float* xbar = at<float>(ws, P.off_xbar);
  float* Fbar = at<float>(ws, P.off_Fbar);
  float* x0p = x0 ? at<float>(ws, P.off_x0p) : nullptr;
  const double* tape_nu = static_cast<const double*>(tape);
  auto tape_u = [&](int i) -> const float* {
    return reinterpret_cast<const float*>(static_cast<const char*>(tape) + P.tape_hdr_bytes +
                                          (size_t)i * align_up(sizeof(float) * (size_t)P.vol_elems));
  };

  // tcgen05 plain passes (the forward's plan): the temporal pass writes fp16 planes with an exponent
  // from the range bound of A26; slots SC_VMAX + (k & 1): max |x_bar_k|; + 3: max |F|; + 4: max |F x_0|
  const bool t6 = P.tc6;
  double* const scb = at<double>(ws, P.off_sc);
  auto bslot = [&](int j) { return reinterpret_cast<unsigned*>(scb + SC_VMAX + j); };
  CombineParams cp;
  fill_combine(cp, P, ch, w_host, b, act, ws);
  cp.x0 = x0;
  cp.F = F;
  cp.x0p = x0p;
  if (t6) {
    cp.fmax = bslot(3);
    cp.pmax = bslot(4);
  }
  combine_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(cp);
  SF_CUDA(after_launch("combine", st));

  BwdInitParams ip;
  std::memset(&ip, 0, sizeof(ip));
  ip.g = dL_dx;
  ip.F = F;
  ip.uK1 = tape_u(K - 1);
  ip.xbar = xbar;
  ip.Fbar = Fbar;
  ip.tape_nu = tape_nu;
  ip.sc = at<double>(ws, P.off_sc);
  ip.partials = at<double>(ws, P.off_part);
  ip.counter = &at<WsHeader>(ws, 0)->counter[2];
  ip.tape_bin = reinterpret_cast<const double*>(static_cast<const char*>(tape) + P.tape_nu_bytes);
  ip.kappa = P.kappa(K);
  ip.B = (int)P.B;
  ip.T = (int)P.T;
  ip.H = (int)P.H;
  ip.W = (int)P.W;
  ip.Wp = (int)P.Wp;
  ip.K = K;
  ip.g_T = (int)P.T;
  ip.g_t0 = 0;
  ip.gx = P.gx;
  if (t6) ip.xbmax = bslot(K & 1);
  bwd_init_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(ip);
  SF_CUDA(after_launch("bwd_init", st));

  SpassParams sp;
  std::memset(&sp, 0, sizeof(sp));
  // spatial part of a backward step: on the tensor-core plan, u = G_xy * v by the
  // tensor-core pass in plain mode into a scratch volume, then the streaming epilogue
  // (bwd_epi_kernel); otherwise the FP32 pass with the fused epilogue (SP_BWD)
  if (!(t6     ? make_planes_tmap(&sp.tmap, v, P.W, P.H, P.BT, P.Wp)
         : P.tc ? make_spass_fwd_tmap(&sp.tmap, P, v)
                : make_volume_tmap(&sp.tmap, v, P.W, P.H, P.BT, P.Wp, spass_boxw(P.RS))))
    return SFSEG_ERR_CUDA;
  fill_spass_common(sp, P, ws);
  sp.tape_nu = const_cast<double*>(tape_nu);
  sp.out = xbar;
  sp.Fbar = Fbar;
  sp.x0p = x0p;
  float* ubuf = at<float>(ws, P.off_p2);
  BwdEpiParams be;
  std::memset(&be, 0, sizeof(be));
  be.u = ubuf;
  be.F = F;
  be.xbar = xbar;
  be.x0p = x0p;
  be.Fbar = Fbar;
  be.sc = at<double>(ws, P.off_sc);
  be.tape_nu = tape_nu;
  be.partials = at<double>(ws, P.off_part);
  be.counter = &at<WsHeader>(ws, 0)->counter[0];
  be.B = (int)P.B;
  be.T = (int)P.T;
  be.H = (int)P.H;
  be.W = (int)P.W;
  be.Wp = (int)P.Wp;
  be.gx = P.gx;
  be.K = K;
  be.tape_bin = ip.tape_bin;
  TpassParams tp;
  std::memset(&tp, 0, sizeof(tp));
  fill_tpass_common(tp, P, ws);
  tp.src = xbar;
  tp.F = F;
  tp.out = v;
  if (t6) {
    float gt = 0.f, gs = 0.f;
    for (int i = 0; i < 2 * P.RT + 1; ++i) gt += std::fabs(P.gt[i]);
    for (int i = 0; i < 2 * P.RS + 1; ++i) gs += std::fabs(P.gs[i]);
    tp.gsum = gt * (1.f + 1e-4f);
    tp.gs3 = gt * gs * gs * (1.f + 1e-4f);
    tp.fmax_in = bslot(3);
    tp.vexp_out = scb + SC_VEXP;
  }
  for (int k = K; k >= 1; --k) {
    tp.u1 = tape_u(k - 1);
    if (t6) {
      tp.vmax = nullptr;
      tp.pmax_in = bslot(k & 1);          // max |x_bar_k|
      tp.pmax_zero = bslot((k - 1) & 1);  // for bwd_epi's max |x_bar_{k-1}|
      tp.umax_in = bslot(k == 1 ? 4 : 3); // |u_1| <= gs3 max|F x_0|, |u_k| <= gs3 max|F| (x_{k-1} unit norm)
      be.xbmax = bslot((k - 1) & 1);
      ProfScope ps(P.prof, st, PC_BWD);
      SF_CUDA(launch_tpass_bwd16(P.RT, tp, (int)P.B, st));
      SF_CUDA(after_launch("tpass_bwd16", st));
    } else {
      set_vslot(tp, &sp, P, ws, k);
      ProfScope ps(P.prof, st, PC_BWD);
      SF_CUDA(launch_tpass_bwd(P.RT, tp, (int)P.B, st));
      SF_CUDA(after_launch("tpass_bwd", st));
    }
    sp.u1 = tape_u(k - 1);
    sp.u2 = (k >= 2) ? tape_u(k - 2) : nullptr;
    sp.k = k;
    // plain spatial pass + streaming epilogue: always with the tensor-core pass, and on the FP32
    // plan when an iteration is binarised (the fused FP32 epilogue has no binarisation adjoint)
    if (P.tc || P.bin) {
      SpassParams pl = sp;
      pl.plain = 1;
      pl.out = ubuf;
      if (t6) {
        pl.S = P.S6;
        pl.NB = P.NB6;
        pl.U = P.U6;
        pl.G = P.G6;
        pl.eslot = 0;
        ProfScope ps(P.prof, st, PC_BWD);
        SF_CUDA(launch_spass_tc6(P.RS, pl, P.G6, st));
        SF_CUDA(after_launch("spass_tc6(plain, bwd)", st));
      } else {
        ProfScope ps(P.prof, st, PC_BWD);
        SF_CUDA(launch_spass_forward(P, pl, st));
        SF_CUDA(after_launch("spass_tc(plain, bwd)", st));
      }
      be.u1 = sp.u1;
      be.u2 = sp.u2;
      be.k = k;
      be.kappa_prev = P.kappa(k - 1);
      {
        ProfScope ps(P.prof, st, PC_BWD);
        bwd_epi_kernel<<<dim3((unsigned)P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(be);
        SF_CUDA(after_launch("bwd_epi", st));
      }
    } else {
      ProfScope ps(P.prof, st, PC_BWD);
      SF_CUDA(launch_spass_bwd(P.RS, sp, P.G, st));
      SF_CUDA(after_launch("spass_bwd", st));
    }
  }

  ContractParams cc;
  std::memset(&cc, 0, sizeof(cc));
  cc.ch = ch;
  cc.Fbar = Fbar;
  cc.xbar0 = x0 ? nullptr : xbar;
  cc.partials = at<double>(ws, P.off_part);
  cc.out = at<double>(ws, P.off_out);
  cc.counter = &at<WsHeader>(ws, 0)->counter[3];
  cc.B = (int)P.B;
  cc.C = C;
  cc.T = (int)P.T;
  cc.H = (int)P.H;
  cc.W = (int)P.W;
  cc.Wp = (int)P.Wp;
  cc.in_T = (int)P.T;
  cc.in_t0 = 0;
  cc.act = act;
  cc.bias = b;
  for (int c = 0; c < C; ++c) cc.w[c] = w_host[c];
  const dim3 G2((unsigned)P.gx, (unsigned)P.BT);  // partials: BT * gx * (C+1) <= n_part (checked in make_plan)
  if (C <= 1) contract_kernel<1><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 2) contract_kernel<2><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 4) contract_kernel<4><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 8) contract_kernel<8><<<G2, kEwThreads, 0, st>>>(cc);
  else if (C <= 16) contract_kernel<16><<<G2, kEwThreads, 0, st>>>(cc);
  else contract_kernel<kMaxC><<<G2, kEwThreads, 0, st>>>(cc);
  SF_CUDA(after_launch("contract", st));
  std::vector<double> out(C + 1);
  SF_CUDA(cudaMemcpyAsync(out.data(), cc.out, sizeof(double) * (C + 1), cudaMemcpyDeviceToHost, st));
  s = sfseg_sync_status(ws, stream);
  for (int c = 0; c < C; ++c) dL_dw_host[c] = out[c];
  if (dL_db_host) *dL_db_host = out[C];
  return s;
}

// ====================================================================== full SFSeg operator
namespace {
struct FullLayout {
  size_t off_U, off_F, off_a, off_v, off_ua, off_ub, off_uc, total;
};
FullLayout full_layout(const Plan& P) {
  FullLayout L;
  const size_t vb = align_up(sizeof(float) * (size_t)P.vol_elems);
  size_t off = P.off_F;  // header, scalars, partials and the reduction output block as in the hot path
  L.off_U = off;
  off += vb;
  L.off_F = off;
  off += vb;
  L.off_a = off;
  off += vb;
  L.off_v = off;
  off += vb;
  L.off_ua = off;
  off += vb;
  L.off_ub = off;
  off += vb;
  L.off_uc = off;
  off += vb;
  L.total = off;
  return L;
}
sfseg_status full_check(int32_t Cs, int32_t Cf, double p, double alpha) {
  if (Cs < 1 || Cf < 1) return SFSEG_ERR_INVALID_ARGUMENT;
  if (Cs > kMaxC || Cf > kMaxC) return SFSEG_ERR_UNSUPPORTED;
  if (!(p > 0.0) || !std::isfinite(p) || !(alpha > 0.0) || !std::isfinite(alpha)) return SFSEG_ERR_INVALID_ARGUMENT;
  return SFSEG_OK;
}
}  // namespace

sfseg_status sfseg_workspace_bytes_full(sfseg_shape sh, int32_t Cs, int32_t Cf, sfseg_gauss gauss, int32_t K,
                                        size_t* ws_bytes_host) {
  if (!ws_bytes_host) return SFSEG_ERR_INVALID_ARGUMENT;
  sfseg_status s = full_check(Cs, Cf, 1.0, 1.0);
  if (s != SFSEG_OK) return s;
  Plan P;
  if ((s = make_plan(sh, std::max(Cs, Cf), gauss, K, &P)) != SFSEG_OK) return s;
  *ws_bytes_host = full_layout(P).total;
  return SFSEG_OK;
}

sfseg_status sfseg_power_iterate_full(const float* s_ch, int32_t Cs, const float* ws_host, float bs, int32_t act_s,
                                      const float* f_ch, int32_t Cf, const float* wf_host, float bf, int32_t act_f,
                                      double p, double alpha, sfseg_shape sh, sfseg_gauss gauss, int32_t K,
                                      const float* x0, float* x_out, double* stats, const sfseg_binarize* bin,
                                      void* ws, size_t ws_bytes, const sfseg_options* opt, void* stream) {
  if (!s_ch || !f_ch || !ws_host || !wf_host || !x_out || !validate_act(act_s) || !validate_act(act_f))
    return SFSEG_ERR_INVALID_ARGUMENT;
  if (bin && (bin->n_cont < 0 || !(bin->kappa0 > 0.f) || !std::isfinite(bin->kappa0) || !(bin->growth > 0.f) ||
              !std::isfinite(bin->growth)))
    return SFSEG_ERR_INVALID_ARGUMENT;
  sfseg_status s = full_check(Cs, Cf, p, alpha);
  if (s != SFSEG_OK) return s;
  Plan P;
  if ((s = make_plan(sh, std::max(Cs, Cf), gauss, K, &P, opt)) != SFSEG_OK) return s;
  if (!finite_weights(ws_host, Cs, bs) || !finite_weights(wf_host, Cf, bf)) return SFSEG_ERR_INVALID_ARGUMENT;
  const FullLayout L = full_layout(P);
  if ((s = check_ws(ws, ws_bytes, L.total)) != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SF_CUDA(clear_header(ws, P.off_part, st));
  float* U = at<float>(ws, L.off_U);
  float* F = at<float>(ws, L.off_F);
  float* a = at<float>(ws, L.off_a);
  // four volumes for the three temporal outputs v_c and spatial outputs u_c: each spatial
  // pass writes over a v already consumed (buffers 0..3 = off_v, off_ua, off_ub, off_uc)
  float* buf[4] = {at<float>(ws, L.off_v), at<float>(ws, L.off_ua), at<float>(ws, L.off_ub),
                   at<float>(ws, L.off_uc)};
  float* vin[3] = {buf[0], buf[2], buf[3]};   // G_t*(a), G_t*(F^2 a), G_t*(F a)
  float* uo[3] = {buf[1], buf[0], buf[2]};    // u_a over a free buffer, u_b over v_a, u_c over v_b

  // Eq.9 for S and F, U = S^p, a_0 = U x_0, ||x_0||
  CombineFullParams cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.s_ch = s_ch;
  cp.f_ch = f_ch;
  cp.x0 = x0;
  cp.U = U;
  cp.F = F;
  cp.a0 = a;
  cp.sc = at<double>(ws, P.off_sc);
  cp.partials = at<double>(ws, P.off_part);
  cp.counter = &at<WsHeader>(ws, 0)->counter[1];
  cp.err = &at<WsHeader>(ws, 0)->err;
  cp.B = (int)P.B;
  cp.Cs = Cs;
  cp.Cf = Cf;
  cp.T = (int)P.T;
  cp.H = (int)P.H;
  cp.W = (int)P.W;
  cp.Wp = (int)P.Wp;
  cp.act_s = act_s;
  cp.act_f = act_f;
  cp.gx = P.gx;
  cp.bs = bs;
  cp.bf = bf;
  cp.p = (float)p;
  for (int c = 0; c < Cs; ++c) cp.ws[c] = ws_host[c];
  for (int c = 0; c < Cf; ++c) cp.wf[c] = wf_host[c];
  // tcgen05 plain passes (no soft-binarisation): the stacked temporal pass writes fp16 planes with
  // exponents from max |a| (slot SC_VMAX + (k & 1)) and max |F| (SC_VMAX + 5); e_c in SC_VMAX + 2 + c
  const bool t6 = P.tc6 && !bin;
  double* const scf = at<double>(ws, P.off_sc);
  auto uslot = [&](int j) { return reinterpret_cast<unsigned*>(scf + SC_VMAX + j); };
  if (t6) {
    cp.amax = uslot(0);
    cp.fmax = uslot(5);
  }
  combine_full_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(cp);
  SF_CUDA(after_launch("combine_full", st));

  SpassParams sp;
  std::memset(&sp, 0, sizeof(sp));
  CUtensorMap vmap[3];
  for (int c = 0; c < 3; ++c)
    if (!(t6 ? make_planes_tmap(&vmap[c], vin[c], P.W, P.H, P.BT, P.Wp) : make_spass_fwd_tmap(&vmap[c], P, vin[c])))
      return SFSEG_ERR_CUDA;
  fill_spass_common(sp, P, ws);
  sp.plain = 1;
  sp.F = F;            // the full layout's pairwise map (fill_spass_common points at the hot path's F slot)
  sp.ua = uo[0];       // the fused combination's operands (third pass, EPI_FULL)
  sp.ub = uo[1];
  sp.Ufull = U;
  sp.inv_alpha = (float)(1.0 / alpha);
  sp.stats = stats;
  Tpass3Params tp;
  std::memset(&tp, 0, sizeof(tp));
  tp.a = a;
  tp.F = F;
  for (int c = 0; c < 3; ++c) tp.out[c] = vin[c];
  tp.sc = at<double>(ws, P.off_sc);
  tp.frame2 = P.H * P.Wp / 2;
  tp.T = (int)P.T;
  for (int i = 0; i < 2 * P.RT + 1; ++i) {
    tp.g[i] = P.gt[i];
    uint32_t gb;
    std::memcpy(&gb, &P.gt[i], 4);
    tp.g2[i] = (unsigned long long)gb | ((unsigned long long)gb << 32);
  }
  if (t6) {
    float gsum = 0.f;
    for (int i = 0; i < 2 * P.RT + 1; ++i) gsum += std::fabs(P.gt[i]);
    tp.gsum = gsum * (1.f + 1e-5f);
    tp.fmax_in = uslot(5);
    tp.vexp_out = scf + SC_VMAX + 2;
    sp.S = P.S6;
    sp.NB = P.NB6;
    sp.U = P.U6;
    sp.G = P.G6;
  }
  FullEpiParams ep;
  std::memset(&ep, 0, sizeof(ep));
  ep.ua = uo[0];
  ep.ub = uo[1];
  ep.uc = uo[2];
  ep.U = U;
  ep.F = F;
  ep.out = a;
  ep.sc = at<double>(ws, P.off_sc);
  ep.partials = at<double>(ws, P.off_part);
  ep.counter = &at<WsHeader>(ws, 0)->counter[1];
  ep.err = &at<WsHeader>(ws, 0)->err;
  ep.stats = stats;
  ep.B = (int)P.B;
  ep.T = (int)P.T;
  ep.H = (int)P.H;
  ep.Wp = (int)P.Wp;
  ep.W = (int)P.W;
  ep.K = K;
  ep.gx = P.gx;
  ep.inv_alpha = (float)(1.0 / alpha);
  // SFSEG_FULL_FUSE (A/B, measured slower): the combination fused into the third
  // spatial pass (spass_tc EPI_FULL) instead of full_epilogue_kernel
#ifndef SFSEG_FULL_FUSE
#define SFSEG_FULL_FUSE 0
#endif
  const bool fuse = SFSEG_FULL_FUSE && P.tc && !t6;
  for (int k = 1; k <= K; ++k) {
    const bool bink = bin && k > bin->n_cont;  // Alg.1 STEP 3 after this iteration
    const int last = (k == K || bink) ? 1 : 0; // store y_k itself when it is binarised next
    // max |v| slots of this iteration's three inputs: 3 (k & 1) + c; each spatial pass zeroes
    // its input's slot of the other parity (last read by the previous iteration)
    const int base = 3 * (k & 1), other = 3 * ((k + 1) & 1);
    for (int c = 0; c < 3; ++c)
      tp.vmax[c] = (P.f16 && !t6) ? reinterpret_cast<unsigned*>(at<double>(ws, P.off_sc) + SC_VMAX + base + c) : nullptr;
    if (t6) {
      tp.amax_in = uslot((k - 1) & 1);
      tp.amax_zero = uslot(k & 1);
    }
    {  // G_t*(S^p X), G_t*(F^2 S^p X), G_t*(F S^p X) in one pass over a and F
      ProfScope ps(P.prof, st, PC_TPASS);
      SF_CUDA(launch_tpass3(P.RT, tp, (int)P.B, st, t6));
      SF_CUDA(after_launch("tpass3_full", st));
    }
    for (int c = 0; c < 3 && t6; ++c) {   // u_c = G_xy v_c on the tcgen05 pass (plain epilogue)
      sp.tmap = vmap[c];
      sp.eslot = SC_VMAX + 2 + c;
      sp.out = uo[c];
      sp.k = k;
      sp.plain = 1;
      sp.full_epi = 0;
      sp.last = last;
      ProfScope ps(P.prof, st, PC_SPASS);
      SF_CUDA(launch_spass_tc6(P.RS, sp, P.G6, st));
      SF_CUDA(after_launch("spass_tc6_plain", st));
    }
    for (int c = 0; c < 3 && !t6; ++c) {
      const bool fc = fuse && c == 2;
      sp.tmap = vmap[c];
      sp.vslot = base + c;
      sp.vzero = other + c + 1;
      sp.out = fc ? a : uo[c];
      sp.k = k;
      sp.plain = fc ? 0 : 1;
      sp.full_epi = fc ? 1 : 0;
      sp.last = last;
      {
        ProfScope ps(P.prof, st, PC_SPASS);
        SF_CUDA(launch_spass_forward(P, sp, st));
        SF_CUDA(after_launch(fc ? "spass_full" : "spass_plain", st));
      }
    }
    if (!fuse) {
      ep.k = k;
      ep.last = last;
      ep.amax = (t6 && !last) ? uslot(k & 1) : nullptr;
      full_epilogue_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(ep);
      SF_CUDA(after_launch("full_epilogue", st));
    }
    if (bink) {
      BinParams bp;
      std::memset(&bp, 0, sizeof(bp));
      bp.y = a;
      bp.U = U;
      bp.a = (k == K) ? nullptr : a;   // in place: each element of y_k becomes U x_k
      bp.x_dense = (k == K) ? x_out : nullptr;
      bp.sc = at<double>(ws, P.off_sc);
      bp.partials = at<double>(ws, P.off_part);
      bp.counter = &at<WsHeader>(ws, 0)->counter[1];
      bp.err = &at<WsHeader>(ws, 0)->err;
      bp.B = (int)P.B;
      bp.T = (int)P.T;
      bp.H = (int)P.H;
      bp.W = (int)P.W;
      bp.Wp = (int)P.Wp;
      bp.gx = P.gx;
      bp.kappa = (float)(bin->kappa0 * std::pow((double)bin->growth, (double)(k - bin->n_cont - 1)));
      pos_stats_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(bp);
      SF_CUDA(after_launch("pos_stats", st));
      binarize_kernel<<<dim3(P.gx, (unsigned)P.BT), kEwThreads, 0, st>>>(bp);
      SF_CUDA(after_launch("binarize", st));
    }
  }
  if (bin && K > bin->n_cont) return SFSEG_OK;  // x_out = the last binarised iterate (values in (0,1))
  dim3 grid((unsigned)P.gx, (unsigned)P.BT);
  final_scale_kernel<<<grid, kEwThreads, 0, st>>>(a, x_out, at<double>(ws, P.off_sc), (int)P.T, (int)P.H, (int)P.W,
                                                  (int)P.Wp, (int)P.T, 0);
  SF_CUDA(after_launch("final_scale", st));
  return SFSEG_OK;
}

// ====================================================================== online / sub-window mode (§8(f) f3)
namespace {
struct OnlineLayout {
  size_t inner, off_F, off_Fw, off_x0, off_xa, off_xb, off_fac, total;
};
sfseg_status online_layout(sfseg_shape sh, int32_t C, sfseg_gauss g, int32_t K, int32_t q, OnlineLayout* L) {
  if (q < 1) return SFSEG_ERR_INVALID_ARGUMENT;
  const int64_t qq = std::min<int64_t>(q, sh.T);
  Plan P;
  sfseg_status s = make_plan(sfseg_shape{sh.B, qq, sh.H, sh.W}, 1, g, K, &P);
  if (s != SFSEG_OK) return s;
  Plan Pc;
  if ((s = make_plan(sh, C, g, K, &Pc)) != SFSEG_OK) return s;  // validates C
  L->inner = align_up(P.ws_fwd + sfseg_threshold_ws_bytes(sfseg_shape{sh.B, qq, sh.H, sh.W}));
  const size_t full = align_up(sizeof(float) * (size_t)(sh.B * sh.T * sh.H * sh.W));
  const size_t win = align_up(sizeof(float) * (size_t)(sh.B * qq * sh.H * sh.W));
  size_t off = L->inner;
  L->off_F = off;
  off += full;
  L->off_Fw = off;
  off += win;
  L->off_x0 = off;
  off += win;
  L->off_xa = off;
  off += win;
  L->off_xb = off;
  off += win;
  L->off_fac = off;
  off += align_up(sizeof(double) * (size_t)sh.B);
  L->total = off;
  return SFSEG_OK;
}
// window starts: 0, stride, 2 stride, ... while start + q < T, then T - q (oracle/online.py)
std::vector<int64_t> window_starts(int64_t T, int64_t q, int64_t stride) {
  std::vector<int64_t> st;
  if (q >= T) return {0};
  for (int64_t s = 0; s + q < T; s += stride) st.push_back(s);
  if (st.empty() || st.back() + q < T) st.push_back(T - q);
  return st;
}
// copy frames [t0, t0 + n) of every volume between a [B][Ta][HW] and a [B][Tb][HW] buffer
cudaError_t copy_frames(float* dst, int64_t Td, int64_t td0, const float* src, int64_t Ts, int64_t ts0, int64_t n,
                        int64_t B, int64_t HW, cudaStream_t st) {
  return cudaMemcpy2DAsync(dst + td0 * HW, sizeof(float) * Td * HW, src + ts0 * HW, sizeof(float) * Ts * HW,
                           sizeof(float) * n * HW, B, cudaMemcpyDeviceToDevice, st);
}
}  // namespace

sfseg_status sfseg_workspace_bytes_online(sfseg_shape sh, int32_t C, sfseg_gauss gauss, int32_t K, int32_t q,
                                          size_t* ws_bytes_host) {
  if (!ws_bytes_host) return SFSEG_ERR_INVALID_ARGUMENT;
  OnlineLayout L;
  sfseg_status s = online_layout(sh, C, gauss, K, q, &L);
  if (s != SFSEG_OK) return s;
  *ws_bytes_host = L.total;
  return SFSEG_OK;
}

sfseg_status sfseg_power_iterate_online(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                        sfseg_shape sh, sfseg_gauss gauss, int32_t K, int32_t q, int32_t stride,
                                        float* x_out, void* ws, size_t ws_bytes, void* stream) {
  if (!ch || !w_host || !x_out || !validate_act(act) || stride < 1) return SFSEG_ERR_INVALID_ARGUMENT;
  // windows must tile the video: a stride longer than the window would leave frames unwritten
  if (q < sh.T && stride > q) return SFSEG_ERR_INVALID_ARGUMENT;
  OnlineLayout L;
  sfseg_status s = online_layout(sh, C, gauss, K, q, &L);
  if (s != SFSEG_OK) return s;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  if ((s = check_ws(ws, ws_bytes, L.total)) != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t T = sh.T, B = sh.B, HW = sh.H * sh.W, qq = std::min<int64_t>(q, T);
  char* base = static_cast<char*>(ws);
  float* Ffull = reinterpret_cast<float*>(base + L.off_F);
  float* Fw = reinterpret_cast<float*>(base + L.off_Fw);
  float* x0 = reinterpret_cast<float*>(base + L.off_x0);
  float* xcur = reinterpret_cast<float*>(base + L.off_xa);
  float* xprev = reinterpret_cast<float*>(base + L.off_xb);
  double* fac = reinterpret_cast<double*>(base + L.off_fac);
  // F once for the whole video (Eq.9); every window then solves with C = 1, identity
  if ((s = sfseg_combine_channels(ch, C, sh, w_host, b, act, Ffull, stream)) != SFSEG_OK) return s;
  const float one = 1.0f;
  const sfseg_shape ws_shape{B, qq, sh.H, sh.W};
  int64_t prev = -1;
  for (const int64_t s0 : window_starts(T, qq, stride)) {
    SF_CUDA(copy_frames(Fw, qq, 0, Ffull, T, s0, qq, B, HW, st));
    SF_CUDA(cudaMemcpyAsync(x0, Fw, sizeof(float) * (size_t)(B * qq * HW), cudaMemcpyDeviceToDevice, st));
    if (prev >= 0 && prev + qq > s0) {  // overlap frames [s0, prev + qq): warm start (reading A20)
      OnlineParams op;
      op.xprev = xprev;
      op.Fw = Fw;
      op.x0 = x0;
      op.factor = fac;
      op.counter = &at<WsHeader>(ws, 0)->counter[2];
      op.HW = HW;
      op.B = (int)B;
      op.q = (int)qq;
      op.nov = (int)(prev + qq - s0);
      op.po = (int)(s0 - prev);
      Plan P;  // the inner solve's partials region holds >= 2 * B * q * gx doubles
      make_plan(ws_shape, 1, gauss, K, &P);
      op.gx = P.gx;
      op.partials = at<double>(ws, P.off_part);
      online_norms_kernel<<<dim3(op.gx, (unsigned)(B * op.nov)), kEwThreads, 0, st>>>(op);
      SF_CUDA(after_launch("online_norms", st));
      online_warm_kernel<<<dim3(op.gx, (unsigned)(B * op.nov)), kEwThreads, 0, st>>>(op);
      SF_CUDA(after_launch("online_warm", st));
    }
    s = sfseg_power_iterate(Fw, 1, &one, 0.f, SFSEG_ACT_IDENTITY, ws_shape, gauss, K, x0, xcur, nullptr, nullptr, 0,
                            nullptr, ws, L.inner, nullptr, stream);
    if (s != SFSEG_OK) return s;
    SF_CUDA(copy_frames(x_out, T, s0, xcur, qq, 0, qq, B, HW, st));
    std::swap(xcur, xprev);
    prev = s0;
  }
  return SFSEG_OK;
}

size_t sfseg_threshold_ws_bytes(sfseg_shape sh) {
  if (sh.B < 1 || sh.T < 1) return 0;
  return align_up(sizeof(float) * (size_t)(sh.B * sh.T) * kThrGx);
}

sfseg_status sfseg_threshold(const float* x, sfseg_shape sh, float tau, int32_t mode, uint8_t* mask, void* ws,
                             size_t ws_bytes, void* stream) {
  if (!x || !mask || !std::isfinite(tau)) return SFSEG_ERR_INVALID_ARGUMENT;
  if (mode < 0 || mode > 2) return SFSEG_ERR_INVALID_ARGUMENT;
  if (sh.B < 1 || sh.T < 1 || sh.H < 1 || sh.W < 1) return SFSEG_ERR_SHAPE;
  sfseg_status s = check_ws(ws, ws_bytes, sfseg_threshold_ws_bytes(sh));
  if (s != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long HW = (long)(sh.H * sh.W);
  float* part = static_cast<float*>(ws);
  const unsigned BT = (unsigned)(sh.B * sh.T);
  const int gx = ew_gx(sh.H * sh.W / 1024 + 1, sh.B * sh.T);
  if (mode != SFSEG_THR_ABSOLUTE) {
    frame_max_kernel<<<dim3(kThrGx, BT), kEwThreads, 0, st>>>(x, part, HW);
    SF_CUDA(cudaGetLastError());
  }
  threshold_kernel<<<dim3(gx, BT), kEwThreads, 0, st>>>(x, mask, part, kThrGx, (int)sh.T, HW, tau, mode);
  return map_cuda(cudaGetLastError());
}

sfseg_status sfseg_workspace_reset(void* ws, void* stream) {
  if (!ws) return SFSEG_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return SFSEG_ERR_WORKSPACE;
  SF_CUDA(cudaMemsetAsync(ws, 0, align_up(sizeof(WsHeader)), static_cast<cudaStream_t>(stream)));
  return SFSEG_OK;
}

sfseg_status sfseg_sync_status(void* ws, void* stream) {
  if (!ws) return SFSEG_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned err = 0;
  SF_CUDA(cudaMemcpyAsync(&err, &at<WsHeader>(ws, 0)->err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  if (err) {
    unsigned zero = 0;
    SF_CUDA(cudaMemcpyAsync(&at<WsHeader>(ws, 0)->err, &zero, sizeof(unsigned), cudaMemcpyHostToDevice, st));
    SF_CUDA(cudaStreamSynchronize(st));
  }
  if (err & ERR_NONFINITE) return SFSEG_ERR_NONFINITE;
  if (err & ERR_DEGENERATE) return SFSEG_ERR_DEGENERATE;
  return SFSEG_OK;
}

sfseg_status sfseg_solve_host(const float* ch_host, int32_t C, const float* w_host, float b, int32_t act,
                              sfseg_shape sh, sfseg_gauss gauss, int32_t K, float tau, int32_t thr_mode, float* d_ch,
                              float* d_x, uint8_t* d_mask, float* x_out_host, uint8_t* mask_out_host, void* ws,
                              size_t ws_bytes, void* stream) {
  if (!ch_host || !d_ch || !d_x || !d_mask) return SFSEG_ERR_INVALID_ARGUMENT;
  Plan P;
  sfseg_status s = make_plan(sh, C, gauss, K, &P);
  if (s != SFSEG_OK) return s;
  const size_t thr_ws = sfseg_threshold_ws_bytes(sh);
  if ((s = check_ws(ws, ws_bytes, P.ws_fwd + thr_ws)) != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nvox = (size_t)(sh.B * sh.T * sh.H * sh.W);
  SF_CUDA(cudaMemcpyAsync(d_ch, ch_host, sizeof(float) * nvox * C, cudaMemcpyHostToDevice, st));
  s = sfseg_power_iterate(d_ch, C, w_host, b, act, sh, gauss, K, nullptr, d_x, nullptr, nullptr, 0, nullptr, ws,
                          P.ws_fwd, nullptr, stream);
  if (s != SFSEG_OK) return s;
  s = sfseg_threshold(d_x, sh, tau, thr_mode, d_mask, static_cast<char*>(ws) + P.ws_fwd, thr_ws, stream);
  if (s != SFSEG_OK) return s;
  if (x_out_host) SF_CUDA(cudaMemcpyAsync(x_out_host, d_x, sizeof(float) * nvox, cudaMemcpyDeviceToHost, st));
  if (mask_out_host) SF_CUDA(cudaMemcpyAsync(mask_out_host, d_mask, nvox, cudaMemcpyDeviceToHost, st));
  return sfseg_sync_status(ws, stream);
}

sfseg_status sfseg_solve_host_batch(const float* const* ch_host, int32_t n, int32_t C, const float* w_host, float b,
                                    int32_t act, sfseg_shape sh, sfseg_gauss gauss, int32_t K, float tau,
                                    int32_t thr_mode, float* d_ch, float* d_x, uint8_t* d_mask,
                                    float* const* x_out_host, uint8_t* const* mask_out_host, void* ws,
                                    size_t ws_bytes, void* stream, void* stream_h2d, void* stream_d2h) {
  if (!ch_host || n < 1 || !d_ch || !d_x || !d_mask || !w_host || !stream_h2d || !stream_d2h ||
      !validate_act(act) || !std::isfinite(tau) || thr_mode < 0 || thr_mode > 2)
    return SFSEG_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; ++i)
    if (!ch_host[i]) return SFSEG_ERR_INVALID_ARGUMENT;
  Plan P;
  sfseg_status s = make_plan(sh, C, gauss, K, &P);
  if (s != SFSEG_OK) return s;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  const size_t thr_ws = sfseg_threshold_ws_bytes(sh);
  if ((s = check_ws(ws, ws_bytes, P.ws_fwd + thr_ws)) != SFSEG_OK) return s;
  cudaStream_t sc = static_cast<cudaStream_t>(stream), si = static_cast<cudaStream_t>(stream_h2d),
               so = static_cast<cudaStream_t>(stream_d2h);
  const size_t nvox = (size_t)(sh.B * sh.T * sh.H * sh.W);
  cudaEvent_t ev[3][2] = {};
  for (auto& row : ev)
    for (auto& e : row) SF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto destroy = [&]() {
    for (auto& row : ev)
      for (auto& e : row)
        if (e) cudaEventDestroy(e);
  };
  cudaError_t ce = cudaSuccess;
  for (int i = 0; i < n && s == SFSEG_OK && ce == cudaSuccess; ++i) {
    const int sl = i & 1;
    float* dch = d_ch + (size_t)sl * nvox * C;
    float* dx = d_x + (size_t)sl * nvox;
    uint8_t* dm = d_mask + (size_t)sl * nvox;
    // H2D of volume i while volume i-1 solves: its slot's previous solve must be done reading
    if (i >= 2 && (ce = cudaStreamWaitEvent(si, ev[1][sl], 0)) != cudaSuccess) break;
    if ((ce = cudaMemcpyAsync(dch, ch_host[i], sizeof(float) * nvox * C, cudaMemcpyHostToDevice, si)) != cudaSuccess) break;
    if ((ce = cudaEventRecord(ev[0][sl], si)) != cudaSuccess) break;
    if ((ce = cudaStreamWaitEvent(sc, ev[0][sl], 0)) != cudaSuccess) break;
    // the slot's x / mask of volume i-2 must be copied out before they are overwritten
    if (i >= 2 && (ce = cudaStreamWaitEvent(sc, ev[2][sl], 0)) != cudaSuccess) break;
    s = sfseg_power_iterate(dch, C, w_host, b, act, sh, gauss, K, nullptr, dx, nullptr, nullptr, 0, nullptr, ws,
                            P.ws_fwd, nullptr, stream);
    if (s != SFSEG_OK) break;
    s = sfseg_threshold(dx, sh, tau, thr_mode, dm, static_cast<char*>(ws) + P.ws_fwd, thr_ws, stream);
    if (s != SFSEG_OK) break;
    if ((ce = cudaEventRecord(ev[1][sl], sc)) != cudaSuccess) break;
    // D2H of volume i while volume i+1 solves
    if ((ce = cudaStreamWaitEvent(so, ev[1][sl], 0)) != cudaSuccess) break;
    if (x_out_host && x_out_host[i] &&
        (ce = cudaMemcpyAsync(x_out_host[i], dx, sizeof(float) * nvox, cudaMemcpyDeviceToHost, so)) != cudaSuccess)
      break;
    if (mask_out_host && mask_out_host[i] &&
        (ce = cudaMemcpyAsync(mask_out_host[i], dm, nvox, cudaMemcpyDeviceToHost, so)) != cudaSuccess)
      break;
    if ((ce = cudaEventRecord(ev[2][sl], so)) != cudaSuccess) break;
  }
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(so);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(si);
  destroy();
  if (ce != cudaSuccess) return map_cuda(ce);
  if (s != SFSEG_OK) return s;
  return sfseg_sync_status(ws, stream);   // first device error of any volume (sticky)
}

sfseg_status sfseg_get_unique_id(uint8_t id_host[128]) {
  if (!id_host) return SFSEG_ERR_INVALID_ARGUMENT;
  NcclApi& api = nccl();
  if (!api.ok) return SFSEG_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return SFSEG_ERR_NCCL;
  static_assert(sizeof(id.internal) == 128, "NCCL unique id size");
  std::memcpy(id_host, id.internal, 128);
  return SFSEG_OK;
}

sfseg_status sfseg_comm_create(const uint8_t id_host[128], int32_t nranks, int32_t rank, int32_t device,
                               sfseg_comm** out) {
  if (!id_host || !out || nranks < 1 || rank < 0 || rank >= nranks || device < 0) return SFSEG_ERR_INVALID_ARGUMENT;
  NcclApi& api = nccl();
  if (!api.ok) return SFSEG_ERR_UNSUPPORTED;
  SF_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(id.internal, id_host, 128);
  sfseg_comm* c = new (std::nothrow) sfseg_comm;
  if (!c) return SFSEG_ERR_CUDA;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (cudaMalloc(&c->flag, sizeof(int32_t)) != cudaSuccess) {  // agreement word (setup call, not a solve)
    delete c;
    return SFSEG_ERR_CUDA;
  }
  // the overlapped time-slab schedule's comm stream and hand-off events (setup call, not a solve)
  bool ok = create_comm_stream(&c->cs) == cudaSuccess;
  for (int i = 0; i < 4 && ok; ++i) ok = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok || api.CommInitRank(&c->comm, nranks, id, rank) != ncclSuccess) {
    cudaFree(c->flag);
    for (cudaEvent_t e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
    return ok ? SFSEG_ERR_NCCL : SFSEG_ERR_CUDA;
  }
  *out = c;
  return SFSEG_OK;
}

sfseg_status sfseg_slab_launch_ranges(int32_t T, int32_t radius_t, int32_t has_lo, int32_t has_hi,
                                      int32_t* ranges_host, int32_t* n_ranges_host, int32_t* n_boundary_host) {
  if (!ranges_host || !n_ranges_host || !n_boundary_host || T < 1 || radius_t < 0) return SFSEG_ERR_INVALID_ARGUMENT;
  *n_ranges_host = slab_ranges(T, radius_t, has_lo != 0, has_hi != 0, ranges_host, n_boundary_host);
  return SFSEG_OK;
}

sfseg_status sfseg_comm_destroy(sfseg_comm* c) {
  if (!c) return SFSEG_ERR_INVALID_ARGUMENT;
  NcclApi& api = nccl();
  sfseg_status s = SFSEG_OK;
  if (c->comm && api.ok && api.CommDestroy(c->comm) != ncclSuccess) s = SFSEG_ERR_NCCL;
  if (c->flag) cudaFree(c->flag);
  for (cudaEvent_t e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->cs) cudaStreamDestroy(c->cs);
  delete c;
  return s;
}

sfseg_status sfseg_profiler_create(sfseg_profiler** out) {
  if (!out) return SFSEG_ERR_INVALID_ARGUMENT;
  *out = new (std::nothrow) sfseg_profiler;
  return *out ? SFSEG_OK : SFSEG_ERR_CUDA;
}

sfseg_status sfseg_profiler_destroy(sfseg_profiler* p) {
  if (!p) return SFSEG_ERR_INVALID_ARGUMENT;
  for (ProfRec& r : p->recs) {
    cudaEventSynchronize(r.b);
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : p->pool) cudaEventDestroy(e);
  delete p;
  return SFSEG_OK;
}

sfseg_status sfseg_profiler_read(sfseg_profiler* pp, double* ms_host, int64_t* count_host) {
  if (!pp || !ms_host || !count_host) return SFSEG_ERR_INVALID_ARGUMENT;
  Profiler& p = *pp;
  std::lock_guard<std::mutex> g(p.mu);
  for (int i = 0; i < PC_N; ++i) {
    ms_host[i] = 0.0;
    count_host[i] = 0;
  }
  sfseg_status s = SFSEG_OK;
  for (ProfRec& r : p.recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess)
      s = SFSEG_ERR_CUDA;
    ms_host[r.cat] += ms;
    count_host[r.cat] += 1;
    p.pool.push_back(r.a);
    p.pool.push_back(r.b);
  }
  p.recs.clear();
  return s;
}

// n emulated ranks on one GPU (single stream): the time-slab decomposition with
// in-process halo copies and a rank-ordered reduction (test / validation path).
sfseg_status sfseg_slabs_workspace_bytes(sfseg_shape sh, int32_t C, sfseg_gauss gauss, int32_t K, int32_t nslabs,
                                         size_t* ws_bytes_host) {
  if (!ws_bytes_host || nslabs < 1 || nslabs > kMaxLocalRanks) return SFSEG_ERR_INVALID_ARGUMENT;
  size_t tot = 0;
  for (int i = 0; i < nslabs; ++i) {
    sfseg_shape ls = sh;
    ls.T = slab_start(sh.T, nslabs, i + 1) - slab_start(sh.T, nslabs, i);
    Plan P;
    sfseg_status s = make_plan(ls, C, gauss, K, &P);
    if (s != SFSEG_OK) return s;
    tot += align_up(slab_offsets(P).total);
  }
  *ws_bytes_host = tot;
  return SFSEG_OK;
}

sfseg_status sfseg_slabs_tape_bytes(sfseg_shape sh, int32_t C, sfseg_gauss gauss, int32_t K, int32_t nslabs,
                                     size_t* tape_bytes_host) {
  if (!tape_bytes_host || nslabs < 1 || nslabs > kMaxLocalRanks) return SFSEG_ERR_INVALID_ARGUMENT;
  size_t tot = 0;
  for (int i = 0; i < nslabs; ++i) {
    sfseg_shape ls = sh;
    ls.T = slab_start(sh.T, nslabs, i + 1) - slab_start(sh.T, nslabs, i);
    Plan P;
    sfseg_status s = make_plan(ls, C, gauss, K, &P);
    if (s != SFSEG_OK) return s;
    tot += align_up(P.tape_bytes);
  }
  *tape_bytes_host = tot;
  return SFSEG_OK;
}

sfseg_status sfseg_power_iterate_slabs(const float* ch, int32_t C, const float* w_host, float b, int32_t act,
                                       sfseg_shape sh, sfseg_gauss gauss, int32_t K, int32_t nslabs,
                                       const float* x0, float* x_out, double* stats, int32_t want_rayleigh,
                                       void* tape, void* ws, size_t ws_bytes, const sfseg_options* opt,
                                       void* stream) {
  if (!ch || !w_host || !x_out || !validate_act(act) || nslabs < 1 || nslabs > kMaxLocalRanks)
    return SFSEG_ERR_INVALID_ARGUMENT;
  if (opt && opt->binarize) return SFSEG_ERR_UNSUPPORTED;
  if (tape && (reinterpret_cast<uintptr_t>(tape) % kAlign) != 0) return SFSEG_ERR_WORKSPACE;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  size_t need = 0;
  sfseg_status s = sfseg_slabs_workspace_bytes(sh, C, gauss, K, nslabs, &need);
  if (s != SFSEG_OK) return s;
  if ((s = check_ws(ws, ws_bytes, need)) != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<Rank> R(nslabs);
  size_t off = 0, toff = 0;
  for (int i = 0; i < nslabs; ++i) {
    const int64_t t0 = slab_start(sh.T, nslabs, i), t1 = slab_start(sh.T, nslabs, i + 1);
    sfseg_shape ls = sh;
    ls.T = t1 - t0;
    if ((s = make_plan(ls, C, gauss, K, &R[i].P, opt)) != SFSEG_OK) return s;
    if (tape) {
      R[i].tape = static_cast<char*>(tape) + toff;
      toff += align_up(R[i].P.tape_bytes);
    }
    if (nslabs > 1 && R[i].P.T < R[i].P.RT) return SFSEG_ERR_SHAPE;
    R[i].ch = ch;
    R[i].x0 = x0;
    R[i].in_T = (int)sh.T;
    R[i].in_t0 = (int)t0;
    R[i].x_out = x_out;
    R[i].out_T = (int)sh.T;
    R[i].out_t0 = (int)t0;
    R[i].stats = stats;
    R[i].rayleigh = want_rayleigh;
    R[i].ws = static_cast<char*>(ws) + off;
    R[i].has_lo = i > 0;
    R[i].has_hi = i < nslabs - 1;
    off += align_up(slab_offsets(R[i].P).total);
  }
  for (auto& r : R)
    if ((s = rank_setup(r, st)) != SFSEG_OK) return s;
  for (auto& r : R)
    if ((s = ph_combine(r, w_host, b, act, st)) != SFSEG_OK) return s;
  if ((s = local_allreduce(R, st)) != SFSEG_OK) return s;
  for (auto& r : R)
    if ((s = ph_finalize(r, 0, st)) != SFSEG_OK) return s;
  if ((s = local_exchange(R, st)) != SFSEG_OK) return s;
  SlabSched S;
  SF_CUDA(S.init_own(st, nslabs > 1 && !(opt && opt->slab_schedule == SFSEG_SLAB_SERIAL)));
  std::vector<Rank*> RP;
  for (auto& r : R) RP.push_back(&r);
  if ((s = slab_iterations(
           RP, S, [&](cudaStream_t q) { return local_exchange(R, q); },
           [&](cudaStream_t q) { return local_allreduce(R, q); })) != SFSEG_OK)
    return s;
  for (auto& r : R)
    if ((s = ph_final(r, st)) != SFSEG_OK) return s;
  return SFSEG_OK;
}

// The time-slab backward emulated on one GPU (the per-rank phases of the NCCL path with
// in-process halo copies and rank-ordered reductions), on the tape of sfseg_power_iterate_slabs.
sfseg_status sfseg_power_iterate_slabs_backward(const float* ch, int32_t C, const float* w_host, float b,
                                                int32_t act, sfseg_shape sh, sfseg_gauss gauss, int32_t K,
                                                int32_t nslabs, const void* tape, const float* dL_dx,
                                                double* dL_dw_host, double* dL_db_host, void* ws, size_t ws_bytes,
                                                const sfseg_options* opt, void* stream) {
  if (!ch || !w_host || !tape || !dL_dx || !dL_dw_host || !validate_act(act) || nslabs < 1 ||
      nslabs > kMaxLocalRanks)
    return SFSEG_ERR_INVALID_ARGUMENT;
  if (opt && opt->binarize) return SFSEG_ERR_UNSUPPORTED;
  if (!finite_weights(w_host, C, b)) return SFSEG_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(tape) % kAlign) != 0) return SFSEG_ERR_WORKSPACE;
  size_t need = 0;
  sfseg_status s = sfseg_slabs_workspace_bytes(sh, C, gauss, K, nslabs, &need);
  if (s != SFSEG_OK) return s;
  if ((s = check_ws(ws, ws_bytes, need)) != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<Rank> R(nslabs);
  std::vector<BwdRank> Q(nslabs);
  size_t off = 0, toff = 0;
  for (int i = 0; i < nslabs; ++i) {
    const int64_t t0 = slab_start(sh.T, nslabs, i), t1 = slab_start(sh.T, nslabs, i + 1);
    sfseg_shape ls = sh;
    ls.T = t1 - t0;
    if ((s = make_plan(ls, C, gauss, K, &R[i].P, opt)) != SFSEG_OK) return s;
    if (nslabs > 1 && R[i].P.T < R[i].P.RT) return SFSEG_ERR_SHAPE;
    R[i].ch = ch;
    R[i].in_T = (int)sh.T;
    R[i].in_t0 = (int)t0;
    R[i].ws = static_cast<char*>(ws) + off;
    R[i].tape = const_cast<char*>(static_cast<const char*>(tape)) + toff;
    R[i].has_lo = i > 0;
    R[i].has_hi = i < nslabs - 1;
    off += align_up(slab_offsets(R[i].P).total);
    toff += align_up(R[i].P.tape_bytes);
    Q[i].r = &R[i];
    Q[i].g = dL_dx;
    Q[i].g_T = (int)sh.T;
    Q[i].g_t0 = (int)t0;
  }
  for (int i = 0; i < nslabs; ++i) {
    if ((s = rank_setup(R[i], st)) != SFSEG_OK) return s;
    if ((s = bw_setup(Q[i], st)) != SFSEG_OK) return s;
  }
  for (auto& r : R)
    if ((s = ph_combine(r, w_host, b, act, st)) != SFSEG_OK) return s;
  for (auto& q : Q)
    if ((s = bw_init(q, st)) != SFSEG_OK) return s;
  if ((s = local_allreduce(R, st)) != SFSEG_OK) return s;
  for (auto& q : Q)
    if ((s = bw_init_fin(q, st)) != SFSEG_OK) return s;
  for (int k = K; k >= 1; --k) {
    for (auto& q : Q)
      if ((s = bw_halo(q, k, st)) != SFSEG_OK) return s;
    if ((s = local_bwd_exchange(R, Q, st)) != SFSEG_OK) return s;
    for (auto& q : Q)
      if ((s = bw_step(q, k, st)) != SFSEG_OK) return s;
    if ((s = local_allreduce(R, st)) != SFSEG_OK) return s;
    for (auto& q : Q)
      if ((s = bw_step_fin(q, k, st)) != SFSEG_OK) return s;
  }
  for (auto& q : Q)
    if ((s = bw_contract(q, w_host, b, act, st)) != SFSEG_OK) return s;
  if ((s = local_allreduce(R, st, C + 1)) != SFSEG_OK) return s;
  std::vector<double> out(C + 1);
  SF_CUDA(cudaMemcpyAsync(out.data(), R[0].glob, sizeof(double) * (C + 1), cudaMemcpyDeviceToHost, st));
  s = sfseg_slabs_sync_status(sh, C, gauss, K, nslabs, ws, stream);
  for (int i = 0; i < C; ++i) dL_dw_host[i] = out[i];
  if (dL_db_host) *dL_db_host = out[C];
  return s;
}

// Device error word of slab i inside a sfseg_power_iterate_slabs workspace.
sfseg_status sfseg_slabs_sync_status(sfseg_shape sh, int32_t C, sfseg_gauss gauss, int32_t K, int32_t nslabs,
                                     void* ws, void* stream) {
  if (!ws || nslabs < 1 || nslabs > kMaxLocalRanks) return SFSEG_ERR_INVALID_ARGUMENT;
  size_t off = 0;
  sfseg_status worst = SFSEG_OK;
  for (int i = 0; i < nslabs; ++i) {
    sfseg_shape ls = sh;
    ls.T = slab_start(sh.T, nslabs, i + 1) - slab_start(sh.T, nslabs, i);
    Plan P;
    sfseg_status s = make_plan(ls, C, gauss, K, &P);
    if (s != SFSEG_OK) return s;
    s = sfseg_sync_status(static_cast<char*>(ws) + off, stream);
    if (s != SFSEG_OK && worst == SFSEG_OK) worst = s;
    off += align_up(slab_offsets(P).total);
  }
  return worst;
}

// ====================================================================== learning loop (§8(f) f4)
sfseg_status sfseg_adamw_step(double* w, const double* grad, double* state, int32_t n, int64_t t,
                              const sfseg_adamw* hp, void* stream) {
  if (!w || !grad || !state || !hp || n < 1 || t < 1) return SFSEG_ERR_INVALID_ARGUMENT;
  if (!(hp->lr >= 0.0) || !(hp->beta1 >= 0.0 && hp->beta1 < 1.0) || !(hp->beta2 >= 0.0 && hp->beta2 < 1.0) ||
      !(hp->eps > 0.0) || !(hp->weight_decay >= 0.0) || !std::isfinite(hp->lr) || !std::isfinite(hp->weight_decay))
    return SFSEG_ERR_INVALID_ARGUMENT;
  AdamwParams P;
  P.w = w;
  P.grad = grad;
  P.state = state;
  P.n = n;
  P.lr = hp->lr;
  P.beta1 = hp->beta1;
  P.beta2 = hp->beta2;
  P.eps = hp->eps;
  P.weight_decay = hp->weight_decay;
  P.c1 = 1.0 - std::pow(hp->beta1, (double)t);
  P.c2 = 1.0 - std::pow(hp->beta2, (double)t);
  P.amsgrad = hp->amsgrad ? 1 : 0;
  adamw_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(P);
  return map_cuda(cudaGetLastError());
}

size_t sfseg_focal_dice_ws_bytes(sfseg_shape sh) {
  if (sh.B < 1 || sh.T < 1) return 0;
  const size_t BT = (size_t)(sh.B * sh.T);
  return align_up(sizeof(WsHeader)) + align_up(sizeof(double) * 3 * BT * kFdGx) + align_up(sizeof(double) * BT);
}

sfseg_status sfseg_focal_dice(const float* x, const uint8_t* mask, sfseg_shape sh, double gamma, double* loss,
                              float* dL_dx, void* ws, size_t ws_bytes, void* stream) {
  if (!x || !mask || !loss || !dL_dx || !(gamma > 0.0) || !std::isfinite(gamma)) return SFSEG_ERR_INVALID_ARGUMENT;
  if (sh.B < 1 || sh.T < 1 || sh.H < 1 || sh.W < 1) return SFSEG_ERR_SHAPE;
  sfseg_status s = check_ws(ws, ws_bytes, sfseg_focal_dice_ws_bytes(sh));
  if (s != SFSEG_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FocalDiceParams P;
  P.x = x;
  P.t = mask;
  P.grad = dL_dx;
  P.counter = &at<WsHeader>(ws, 0)->counter[0];
  P.part = at<double>(ws, align_up(sizeof(WsHeader)));
  P.frame_loss = at<double>(ws, align_up(sizeof(WsHeader)) + align_up(sizeof(double) * 3 * (size_t)(sh.B * sh.T) * kFdGx));
  P.loss = loss;
  P.HW = (long)(sh.H * sh.W);
  P.BT = (int)(sh.B * sh.T);
  P.gamma = gamma;
  SF_CUDA(cudaMemsetAsync(ws, 0, align_up(sizeof(WsHeader)), st));
  const dim3 grid(kFdGx, (unsigned)(sh.B * sh.T));
  focal_dice_sums_kernel<<<grid, kEwThreads, 0, st>>>(P);
  SF_CUDA(after_launch("focal_dice_sums", st));
  focal_dice_grad_kernel<<<grid, kEwThreads, 0, st>>>(P);
  SF_CUDA(after_launch("focal_dice_grad", st));
  return SFSEG_OK;
}

}  // extern "C"
