// fv2d_api.cu -- host side of libfv2d: the C ABI of include/fv2d.h.
//
// Owns the device state (two ping-pong SoA buffers per slab, packed ghost
// rows, device scalars), launches the sm_100a kernels of fv2d_kernels.cuh on
// the caller's stream, and drives the NCCL halo exchange / max-all-reduce for
// nranks > 1 (libnccl.so.2 is loaded at run time with dlopen, so a process
// that already holds torch's NCCL shares that one copy).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <vector>
#include <vector>

#include <nccl.h>

#include "fv2d.h"
#include "fv2d_kernels.cuh"

using namespace fv2d;

namespace {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.loaded) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define SYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name))
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(AllReduce, "ncclAllReduce");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  g_nccl.loaded = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.GroupStart &&
                  g_nccl.GroupEnd && g_nccl.Send && g_nccl.Recv && g_nccl.AllReduce;
  return g_nccl.loaded;
}

// ------------------------------------------------------------------ GL-24 table
// Gauss-Legendre nodes/weights on [0,1] by Newton's method on P_24 in long
// double; uploaded once to constant memory as 2 w_q t_q^k (the
// factor 2 of the moments folded into the weights: scaling by 2 is exact, so
// every partial sum is exactly twice the unscaled one).
void gl24_table(double t[24], double wt[24][kGLW]) {
  const int n = 24;
  for (int k = 0; k < n; ++k) {
    long double x = cosl(3.14159265358979323846264338327950288L * (k + 0.75L) / (n + 0.5L));
    long double dp = 0;
    for (int it = 0; it < 200; ++it) {
      long double p0 = 1, p1 = x;
      for (int l = 2; l <= n; ++l) {
        long double p2 = ((2 * l - 1) * x * p1 - (l - 1) * p0) / l;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1);
      long double d = p1 / dp;
      x -= d;
      if (fabsl(d) < 1e-21L) break;
    }
    long double p0 = 1, p1 = x;
    for (int l = 2; l <= n; ++l) {
      long double p2 = ((2 * l - 1) * x * p1 - (l - 1) * p0) / l;
      p0 = p1;
      p1 = p2;
    }
    dp = n * (x * p1 - p0) / (x * x - 1);
    const long double w = 2 / ((1 - x * x) * dp * dp);
    const int q = n - 1 - k;  // ascending t
    t[q] = (double)((x + 1) / 2);
    const double wq = (double)(w / 2);
    double tp = 1.0;
    for (int m = 0; m < kGLW; ++m) {
      wt[q][m] = 2.0 * (wq * tp);  // the moments' factor 2, folded in (exact: a power of two)
      tp = tp * t[q];
    }
  }
}

int nvar_of(int system) {
  switch (system) {
    case FV2D_ADVECTION: return 1;
    case FV2D_EULER: return 4;
    case FV2D_SPRAY: return 6;
    default: return -1;
  }
}

#ifndef FV2D_WARPS
#define FV2D_WARPS 4  // warps per CTA of the marching kernels (tuning knob)
#endif
constexpr int kWarps = FV2D_WARPS;

}  // namespace

// ------------------------------------------------------------------ context
struct fv2d_ctx {
  fv2d_config cfg{};
  cudaStream_t stream = nullptr;
  int nv = 0, nx = 0, H = 0, pitch = 0, nslabs = 1, G = 1, rps = 64;
  // rank grid: px x py blocks, rank = ry * px + rx (px = 1: y-slabs).  nx is the
  // local block width; gnx the global one; col0 the block's first global column;
  // xoff the row-base offset that makes room for the ghost columns (px > 1).
  int px = 1, py = 1, rx = 0, ry = 0, gnx = 0, col0 = 0, xoff = 0;
  bool xg = false;  // stored ghost columns: px > 1 or FV2D_FLAG_GHOST_COLUMNS
  int ring_depth = 4;  // rows in the pair kernel's per-warp prefetch ring
  int tiles_x = 1, tiles_y = 1;  // launch decomposition of a step (granularity study)
  cudaStream_t launch_stream = nullptr;  // stream kernels are launched on (capture stream while capturing)
  // CUDA graph of one step per parity (FV2D_FLAG_GRAPH)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  bool graph_ready = false;
  int graph_adaptive = -1;
  double graph_dt = 0.0, graph_cfl = 0.0;
  int graph_lam_hist = 0;
  const double* graph_dt_log = nullptr;
  // asynchronous output (fv2d_snapshot)
  cudaStream_t out_stream = nullptr;
  cudaEvent_t ev_snap_start = nullptr, ev_snap_conv = nullptr;
  double* snap_buf = nullptr;
  int snap_parity = -1;  // buffer being converted; the step that overwrites it must wait
  long long rs = 0;  // row stride (nv * pitch); a buffer holds rows -1..H
  double dx = 0, dy = 0, hmin = 0;
  // per local slab: two ping-pong buffers of (H+2) rows (ghost rows -1 and H inside)
  double* buf[kMaxSlabs][2] = {};
  double* send_s = nullptr;  // nranks > 1: boundary rows to send
  double* send_n = nullptr;
  double* send_w = nullptr;  // px > 1 (NCCL): packed boundary columns [H][nv] to send
  double* send_e = nullptr;
  double* recv_w = nullptr;  // ... and received, unpacked into the ghost columns
  double* recv_e = nullptr;
  double* staging = nullptr;
  size_t staging_bytes = 0;
  // fv2d_step_host pipeline: output staging, copy streams, per-band events
  double* staging_out = nullptr;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::vector<cudaEvent_t> ev_band;
  // device scalars
  unsigned long long* dscal = nullptr;  // [0]=smax [1]=pending [2]=status [3]=bad_cell [4..5]=reduced
  unsigned int* done = nullptr;
  double* dt_dev = nullptr;
  double* dt_log = nullptr;
  long long dt_log_cap = 0;
  unsigned long long* newton = nullptr;
  double* trig = nullptr;  // sx[nx] cx[nx] sy[ny] cy[ny]
  // spray: Newton warm start, two caches of nslabs x H x 4 x pitch: the pass
  // the multipliers after step n are in lam_buf[n % 3]; the kernels select the
  // levels from the device step counter (StepArgs::lam3), so a CUDA graph
  // captured per parity stays valid (it is recaptured when lam_hist changes)
  double* lam_buf[3] = {nullptr, nullptr, nullptr};
  int lam_hist = 0;  // valid levels: 0 (cold start), 1 (lambda_n), 2 (+lambda_{n-1}), 3 (+lambda_{n-2})
  ncclComm_t comm = nullptr;
  bool use_nccl = false;  // nranks > 1, or FV2D_FLAG_NCCL_LOOPBACK (self exchange on 1 rank)
  // FV2D_FLAG_PEER_HALO: halo rows and the CFL max-all-reduce through peer memory
  bool peer = false, peer_connected = false;
  PeerSync* sync = nullptr;               // own sync block
  PeerArgs pa{};                          // every rank's sync block
  double* peer_buf_s[2] = {nullptr, nullptr};  // south neighbour's buffers (parity 0/1)
  double* peer_buf_n[2] = {nullptr, nullptr};  // north neighbour's buffers
  double* peer_buf_w[2] = {nullptr, nullptr};  // west / east neighbours' buffers (px > 1)
  double* peer_buf_e[2] = {nullptr, nullptr};
  std::vector<void*> ipc_opened;          // IPC mappings to close
  unsigned long long epoch = 0;           // collective points issued so far
  cudaStream_t comm_stream = nullptr;  // NCCL halo exchange overlapped with the interior pass
  cudaEvent_t ev_bnd = nullptr, ev_int = nullptr, ev_fin = nullptr;
  // host state
  bool has_state = false;
  bool dt_valid = false;
  double dt_cfl = 0.0;       // the C that dt_dev was computed with (adaptive mode)
  // pinned scratch for the small host<->device scalars (status, smax, dt): a
  // copy to/from pageable memory is staged by the driver and can wait behind
  // another rank's spinning collective in the same process (peer path, ranks
  // as threads), which then never sees this rank arrive
  unsigned long long* hpin = nullptr;
  int sms = 0;               // multiprocessors of cfg.device
  int slots = 0;             // resident CTAs of the marching step kernel (sms x occupancy)
  int src_slots = 0;         // resident CTAs of the spray source pass (its persistent grid)
  bool guard_done = false;   // S:440 guard passed since the last set_state
  long long steps = 0;
  long long launches = 0;
  // Branch-free division / square root in the Euler pair kernel (FAST, adaptive
  // dt only): used by single-rank contexts (no NCCL or peer path) at the default ring depth, with
  // an in-range Dirichlet state and no snapshot taken.  Steps are journaled
  // until a status read finds nothing latched; a latched E_NONFINITE at a FAST
  // step k (possibly an operand outside the fast range) is answered by
  // recover_fast: the device state of "step k not taken" is restored (W^k is
  // intact in its ping-pong buffer, later steps were no-ops) and steps k.. are
  // re-run with the exact kernels, so results and errors are the exact ones.
  bool fast_ok = false;
  bool force_exact = false;  // fv2d_step_host: exact kernels
  bool snap_used = false;
  struct StepRec {
    int adaptive;
    double dt, cfl;
    bool fast;
  };
  std::vector<StepRec> journal;  // journal[i] = step steps - journal.size() + i
  int graph_fast = -1;
  long long recoveries = 0;  // recover_fast re-runs (stats)
  // profiling: event pairs around step-kernel launches
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  double prof_ms = 0.0;
  long long prof_n = 0;
  std::vector<char> ev_tag;     // per event pair: 0 = step kernel, 1 = spray source kernel
  double prof_src_ms = 0.0;
  long long prof_src_n = 0;
  std::string err;
  long long err_step = -1, err_cell = -1;
  double err_value = NAN;
};

extern "C" {
static fv2d_status recover_fast(fv2d_ctx* ctx, unsigned long long st, bool* redone);
}

namespace {

fv2d_status set_err(fv2d_ctx* c, fv2d_status st, const char* fmt, ...) {
  if (c) {
    char b[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(b, sizeof b, fmt, ap);
    va_end(ap);
    c->err = b;
  }
  return st;
}

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return set_err(ctx, FV2D_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));            \
  } while (0)

#define CKN(call)                                                                                  \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess)                                                                         \
      return set_err(ctx, FV2D_E_NCCL, "%s failed: %s", #call,                                     \
                     g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "?");                     \
  } while (0)

#define CKL()                                                                                      \
  do {                                                                                             \
    ++ctx->launches;                                                                               \
    cudaError_t e_ = cudaGetLastError();                                                           \
    if (e_ != cudaSuccess) return set_err(ctx, FV2D_E_CUDA, "launch failed: %s", cudaGetErrorString(e_)); \
  } while (0)

double* row_ptr(const fv2d_ctx* ctx, int s, int p, int j) {
  return ctx->buf[s][p] + (long long)(j + 1) * ctx->rs + ctx->xoff;
}
// Rank of the block at grid position (x, y), with wrap.
int rank_at(const fv2d_ctx* ctx, int x, int y) {
  return ((y + ctx->py) % ctx->py) * ctx->px + (x + ctx->px) % ctx->px;
}
double* ghost_s(const fv2d_ctx* ctx, int s, int p) { return row_ptr(ctx, s, p, -1); }
double* ghost_n(const fv2d_ctx* ctx, int s, int p) { return row_ptr(ctx, s, p, ctx->H); }

// Ghost targets of local slab s for writes landing in ghost rows of parity q.
void ghost_targets(const fv2d_ctx* ctx, int s, int q, SlabDesc& d) {
  const int g = ctx->ry * ctx->nslabs + s;
  const int G = ctx->G;
  const bool per = ctx->cfg.bc_y == FV2D_BC_PERIODIC;
  const int my_y = nvar_of(ctx->cfg.system) == 4 ? 2 : (nvar_of(ctx->cfg.system) == 6 ? 5 : -1);
  d.dst_s = nullptr;
  d.dst_n = nullptr;
  d.mirror_s = -1;
  d.mirror_n = -1;
  // south boundary row (row 0) -> south neighbour's north ghost row (row H)
  if (g > 0 || per) {
    const int gs_ = (g - 1 + G) % G;
    if (ctx->peer)
      d.dst_s = ctx->peer_buf_s[q] ? ctx->peer_buf_s[q] + (long long)(ctx->H + 1) * ctx->rs + ctx->xoff : nullptr;
    else if (!ctx->use_nccl && gs_ / ctx->nslabs == ctx->ry) d.dst_s = ghost_n(ctx, gs_ % ctx->nslabs, q);
    else d.dst_s = ctx->send_s + ctx->xoff;
  } else if (ctx->cfg.bc_y == FV2D_BC_WALL) {
    d.dst_s = ghost_s(ctx, s, q);
    d.mirror_s = my_y;
  }
  // north boundary row (row H-1) -> north neighbour's south ghost row (row -1)
  if (g < G - 1 || per) {
    const int gn_ = (g + 1) % G;
    if (ctx->peer) d.dst_n = ctx->peer_buf_n[q] ? ctx->peer_buf_n[q] + ctx->xoff : nullptr;  // its row -1
    else if (!ctx->use_nccl && gn_ / ctx->nslabs == ctx->ry) d.dst_n = ghost_s(ctx, gn_ % ctx->nslabs, q);
    else d.dst_n = ctx->send_n + ctx->xoff;
  } else if (ctx->cfg.bc_y == FV2D_BC_WALL) {
    d.dst_n = ghost_n(ctx, s, q);
    d.mirror_n = my_y;
  }
  // 2-D rank blocks: column 0 -> west neighbour's ghost column nx, column nx-1
  // -> east neighbour's ghost column -1 (same row layout on every rank); at a
  // global wall, this buffer's own ghost column, mirrored (R13)
  d.dst_w = d.dst_e = nullptr;
  d.mirror_w = d.mirror_e = -1;
  d.csr_w = d.csr_e = ctx->rs;
  d.csv_w = d.csv_e = ctx->pitch;
  if (ctx->xg) {
    const bool perx = ctx->cfg.bc_x == FV2D_BC_PERIODIC;
    const int my_x = nvar_of(ctx->cfg.system) == 4 ? 1 : (nvar_of(ctx->cfg.system) == 6 ? 4 : -1);
    double* own0 = row_ptr(ctx, s, q, 0);
    if (ctx->rx > 0 || perx) {
      if (ctx->peer) {
        d.dst_w = ctx->peer_buf_w[q] ? ctx->peer_buf_w[q] + ctx->rs + ctx->xoff + ctx->nx : nullptr;
      } else if (!ctx->use_nccl) {
        d.dst_w = own0 + ctx->nx;  // one block along x (px = 1): its own east ghost column
      } else {
        d.dst_w = ctx->send_w;
        d.csr_w = ctx->nv;
        d.csv_w = 1;
      }
    } else if (ctx->cfg.bc_x == FV2D_BC_WALL) {
      d.dst_w = own0 - 1;
      d.mirror_w = my_x;
    }
    if (ctx->rx < ctx->px - 1 || perx) {
      if (ctx->peer) {
        d.dst_e = ctx->peer_buf_e[q] ? ctx->peer_buf_e[q] + ctx->rs + ctx->xoff - 1 : nullptr;
      } else if (!ctx->use_nccl) {
        d.dst_e = own0 - 1;
      } else {
        d.dst_e = ctx->send_e;
        d.csr_e = ctx->nv;
        d.csv_e = 1;
      }
    } else if (ctx->cfg.bc_x == FV2D_BC_WALL) {
      d.dst_e = own0 + ctx->nx;
      d.mirror_e = my_x;
    }
  }
}

// Strip height of a marching-kernel launch over ncols x nrows cells.  A CTA
// marches one strip of rps rows (+2 halo rows) of kWarps x 62 columns; the
// launch has C x S CTAs (C column blocks, S = ceil(nrows/rps) strips) of which
// `slots` = SMs x resident CTAs per SM are resident at a time (queried at
// fv2d_create from the device and the occupancy API for the kernel the context
// launches: 148 x 3 = 444 for the B200 pair kernel).  The cost model ceil(C*S / slots) * (rps + 2)
// (waves x rows marched per CTA) is minimised over S with 4 <= rps <= 128: it
// avoids a nearly empty last wave and gives small domains one wave of short
// strips (latency-bound: 1024^2 -> rps 12).  The cap: in short bursts ~64-row
// strips are 3-8% faster at large sizes (tools/rps_sweep.py,
// profiles/r1_rps_sweep.jsonl: 16384^2 97.2 vs 92.8 G/s), but under sustained
// load the GPU runs at its power cap, and there the longer strips -- fewer
// re-read halo rows, less energy per step -- win by ~1% (200-300-step bench
// A/B, profiles/r1_rps_powercap_ab.txt); the bench measures sustained load.
int num_sms(const fv2d_ctx* ctx) { return ctx->sms > 0 ? ctx->sms : 148; }

int pick_rps(const fv2d_ctx* ctx, int ncols, int nrows) {
  static const int rps_max = getenv("FV2D_RPS_MAX") ? atoi(getenv("FV2D_RPS_MAX")) : 128;  // tuning knob
  static const int rps_force = getenv("FV2D_RPS") ? atoi(getenv("FV2D_RPS")) : 0;          // tuning knob
  if (rps_force > 0) return std::min(rps_force, std::max(1, nrows));
  const long long C = ((ncols + 62) / 62 + kWarps - 1) / kWarps;
  const long long slots = std::max(1, ctx->slots);
  const int s_min = std::max(1, (nrows + rps_max - 1) / rps_max);
  const int s_max = std::max(s_min, nrows / 4);
  long long best_cost = -1;
  int best_rps = std::min(nrows, rps_max);
  for (int S = s_min; S <= s_max; ++S) {
    const int rps = (nrows + S - 1) / S;
    if (rps < 4 && S > s_min) break;
    if ((nrows + rps - 1) / rps != S) continue;  // same rps as a smaller S
    const long long cost = ((C * S + slots - 1) / slots) * (rps + 2);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_rps = rps;
    }
  }
  return std::max(1, best_rps);
}

// Row ranges of a marching-kernel launch (see StepArgs).
void set_ranges(StepArgs& a, int lo0, int hi0, int rps0, int lo1, int hi1, int rps1) {
  a.row_lo[0] = lo0; a.row_hi[0] = hi0; a.rps[0] = rps0;
  a.row_lo[1] = lo1; a.row_hi[1] = hi1; a.rps[1] = rps1;
  a.nstrips0 = hi0 > lo0 ? (hi0 - lo0 + rps0 - 1) / rps0 : 0;
  a.nranges = hi1 > lo1 ? 2 : 1;
}
int total_strips(const StepArgs& a) {
  return a.nstrips0 + (a.row_hi[1] > a.row_lo[1] ? (a.row_hi[1] - a.row_lo[1] + a.rps[1] - 1) / a.rps[1] : 0);
}

// Arguments of a pass reading parity p (and writing parity 1-p).
StepArgs make_args(const fv2d_ctx* ctx, int p) {
  StepArgs a;
  memset(&a, 0, sizeof a);
  const int q = 1 - p;
  a.nslabs = ctx->nslabs;
  for (int s = 0; s < ctx->nslabs; ++s) {
    SlabDesc& d = a.slab[s];
    d.in = row_ptr(ctx, s, p, 0);
    d.out = row_ptr(ctx, s, q, 0);
    ghost_targets(ctx, s, q, d);
    d.row0 = (ctx->ry * ctx->nslabs + s) * ctx->H;
    d.H = ctx->H;
  }
  a.nx = ctx->nx;
  a.pitch = ctx->pitch;
  a.rs = ctx->rs;
  set_ranges(a, 0, ctx->H, ctx->rps, 0, 0, 1);
  a.bcx = ctx->cfg.bc_x;
  for (int v = 0; v < kMaxVar; ++v) a.dirx[v] = ctx->cfg.dirichlet[v];
  a.dx = ctx->dx;
  a.dy = ctx->dy;
  a.hmin = ctx->hmin;
  switch (ctx->cfg.system) {
    case FV2D_ADVECTION: a.sys[0] = ctx->cfg.param[0]; a.sys[1] = ctx->cfg.param[1]; break;
    case FV2D_EULER: a.sys[0] = ctx->cfg.param[0]; a.sys[1] = ctx->cfg.param[0] - 1.0; break;
    case FV2D_SPRAY: a.sys[0] = ctx->cfg.param[0]; a.sys[1] = ctx->cfg.param[1]; break;
  }
  a.dt_dev = ctx->dt_dev;
  a.dt_log = ctx->dt_log;
  a.smax_slot = ctx->dscal + 0;
  a.pending = ctx->dscal + 1;
  a.status = ctx->dscal + 2;
  a.bad_cell = ctx->dscal + 3;
  a.done = ctx->done;
  a.fused_finalize = ctx->use_nccl ? 0 : 1;
  if (ctx->trig) {  // tables over the global mesh; x tables offset to this block
    a.sx_tab = ctx->trig + ctx->col0;
    a.cx_tab = ctx->trig + ctx->gnx + ctx->col0;
    a.sy_tab = ctx->trig + 2 * ctx->gnx;
    a.cy_tab = ctx->trig + 2 * ctx->gnx + ctx->cfg.ny;
  }
  a.newton_iters = ctx->newton;
  a.step_dev = reinterpret_cast<long long*>(ctx->dscal + 6);
  a.col_lo = 0;
  a.col_hi = ctx->nx;
  for (int k = 0; k < 3; ++k) a.lam3[k] = ctx->lam_buf[k];
  a.lam_hist = ctx->lam_hist;
  a.peer_fence = ctx->peer ? 1 : 0;
  if (ctx->peer) a.fused_finalize = 0;
  a.xghost = ctx->xg ? 1 : 0;
  a.col0 = ctx->col0;
  a.gnx = ctx->gnx;
  return a;
}

// Kernel dispatch on the system.
template <template <class> class K, class... Args>
void dispatch(int system, Args&&... args) {
  switch (system) {
    case FV2D_ADVECTION: K<Advection>::run(args...); break;
    case FV2D_EULER: K<Euler>::run(args...); break;
    case FV2D_SPRAY: K<Spray>::run(args...); break;
  }
}

template <class Sys, int D, int XM, bool ADAPT, bool FAST = false>
void launch_pair_1(const fv2d_ctx* ctx, const StepArgs& a, dim3 grid) {
  // (the dynamic shared-memory opt-in was set once at fv2d_create: preload_kernels)
  const int smem = kWarps * D * Sys::NV * 64 * (int)sizeof(double);
  fv_step_pair_kernel<Sys, XM, ADAPT, kWarps, D, FAST><<<grid, kWarps * 32, smem, ctx->launch_stream>>>(a);
}

// The branch-free division / square root variant exists for Euler's adaptive
// instantiation at the default ring depth: there it removes the second
// derive's branches (0.87 -> 0.80 ms per 8192^2 step, adaptive within 0-5% of
// fixed dt; profiles/r2s3_fastdiv_*.jsonl); the fixed-dt kernel does not gain
// from it (it spills 8-16 B and ran 0.5% slower), so fixed dt stays exact.
template <class Sys, int D>
constexpr bool kHasFast = std::is_same<Sys, Euler>::value && D == 4;

template <class Sys, int D, int XM>
void launch_pair_x(const fv2d_ctx* ctx, const StepArgs& a, dim3 grid) {
  if constexpr (kHasFast<Sys, D>) {
    if (a.fast && a.adaptive) {
      launch_pair_1<Sys, D, XM, true, true>(ctx, a, grid);
      return;
    }
#if FV2D_FAST_FIXED
    if (a.fast) {
      launch_pair_1<Sys, D, XM, false, true>(ctx, a, grid);
      return;
    }
#endif
  }
  if (a.adaptive) launch_pair_1<Sys, D, XM, true>(ctx, a, grid);
  else launch_pair_1<Sys, D, XM, false>(ctx, a, grid);
}

template <class Sys, int D>
void launch_pair(const fv2d_ctx* ctx, const StepArgs& a, dim3 grid) {
  if (ctx->xg) launch_pair_x<Sys, D, XM_GHOST>(ctx, a, grid);
  else if (ctx->cfg.bc_x == FV2D_BC_PERIODIC) launch_pair_x<Sys, D, XM_PERIODIC>(ctx, a, grid);
  else launch_pair_x<Sys, D, XM_CLAMP>(ctx, a, grid);
}

template <class Sys>
struct LaunchStep {
  static void run(const fv2d_ctx* ctx, const StepArgs& a) {
    if (ctx->cfg.flags & FV2D_FLAG_NAIVE) {
      dim3 grid((ctx->nx + 31) / 32, (ctx->H + 7) / 8, ctx->nslabs);
      fv_step_naive_kernel<Sys><<<grid, 256, 0, ctx->launch_stream>>>(a);
    } else {
      constexpr int D = 4;
      const bool xper = ctx->cfg.bc_x == FV2D_BC_PERIODIC && !ctx->xg;
      // spray (nVar 6) uses the one-cell kernel: two cells of 6 variables per lane would spill
      if constexpr (Sys::NV == 6) {
        const int cols = 30 * kWarps;
        dim3 grid((a.col_hi - a.col_lo + cols - 1) / cols, total_strips(a), ctx->nslabs);
        cudaStream_t ls = ctx->launch_stream;
        if (xper && !a.adaptive) fv_step_kernel<Sys, true, false, kWarps, D><<<grid, kWarps * 32, 0, ls>>>(a);
        if (xper && a.adaptive) fv_step_kernel<Sys, true, true, kWarps, D><<<grid, kWarps * 32, 0, ls>>>(a);
        if (!xper && !a.adaptive) fv_step_kernel<Sys, false, false, kWarps, D><<<grid, kWarps * 32, 0, ls>>>(a);
        if (!xper && a.adaptive) fv_step_kernel<Sys, false, true, kWarps, D><<<grid, kWarps * 32, 0, ls>>>(a);
      } else if (ctx->cfg.flags & FV2D_FLAG_ONE_CELL) {
        const int cols = 30 * kWarps;
        dim3 grid((a.col_hi - a.col_lo + cols - 1) / cols, total_strips(a), ctx->nslabs);
        if (xper && !a.adaptive) fv_step_kernel<Sys, true, false, kWarps, D><<<grid, kWarps * 32, 0, ctx->launch_stream>>>(a);
        if (xper && a.adaptive) fv_step_kernel<Sys, true, true, kWarps, D><<<grid, kWarps * 32, 0, ctx->launch_stream>>>(a);
        if (!xper && !a.adaptive) fv_step_kernel<Sys, false, false, kWarps, D><<<grid, kWarps * 32, 0, ctx->launch_stream>>>(a);
        if (!xper && a.adaptive) fv_step_kernel<Sys, false, true, kWarps, D><<<grid, kWarps * 32, 0, ctx->launch_stream>>>(a);
      } else {
        const int warps = (a.col_hi - a.col_lo + 1 + 61) / 62;
        dim3 grid((warps + kWarps - 1) / kWarps, total_strips(a), ctx->nslabs);
        switch (ctx->ring_depth) {
          case 6: launch_pair<Sys, 6>(ctx, a, grid); break;
          case 8: launch_pair<Sys, 8>(ctx, a, grid); break;
          default: launch_pair<Sys, 4>(ctx, a, grid); break;
        }
      }
    }
  }
};

template <class Sys>
struct LaunchReduce {
  static void run(const fv2d_ctx* ctx, const StepArgs& a) {
    const long long n = (long long)ctx->nx * ctx->H;
    int blocks = (int)std::min<long long>((n + 255) / 256, num_sms(ctx) * 8);
    reduce_smax_kernel<Sys><<<dim3(blocks, 1, ctx->nslabs), 256, 0, ctx->stream>>>(a);
  }
};

template <class Sys>
struct LaunchArgmax {
  static void run(const fv2d_ctx* ctx, const StepArgs& a, double smax, unsigned long long* out) {
    const long long n = (long long)ctx->nx * ctx->H;
    int blocks = (int)std::min<long long>((n + 255) / 256, num_sms(ctx) * 8);
    argmax_kernel<Sys><<<dim3(blocks, 1, ctx->nslabs), 256, 0, ctx->stream>>>(a, smax, out);
  }
};

// Device geometry for the launch-shape cost models: SM count and the resident
// CTAs per SM of the marching kernel this context launches (fixed-dt
// instantiation), from the occupancy API -- so a register-budget change or
// another GPU re-tunes the strip height instead of silently mis-tuning it.
template <class Sys>
struct Occupancy {
  static cudaError_t run(const fv2d_ctx* ctx, int* per_sm) {
    constexpr int D = 4;
    const bool xper = ctx->cfg.bc_x == FV2D_BC_PERIODIC && !ctx->xg;
    if constexpr (Sys::NV == 6) {  // the one-cell kernel (LaunchStep)
      return xper ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fv_step_kernel<Sys, true, false, kWarps, D>, kWarps * 32, 0)
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fv_step_kernel<Sys, false, false, kWarps, D>, kWarps * 32, 0);
    } else {
    if (ctx->cfg.flags & FV2D_FLAG_ONE_CELL)
      return xper ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fv_step_kernel<Sys, true, false, kWarps, D>, kWarps * 32, 0)
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fv_step_kernel<Sys, false, false, kWarps, D>, kWarps * 32, 0);
    const int Dr = ctx->ring_depth == 6 || ctx->ring_depth == 8 ? ctx->ring_depth : 4;
    const size_t smem = (size_t)kWarps * Dr * Sys::NV * 64 * sizeof(double);
    auto occ = [&](auto kern) { return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, kWarps * 32, smem); };
    if (Dr == 4) {
      if (ctx->xg) return occ(fv_step_pair_kernel<Sys, XM_GHOST, false, kWarps, 4>);
      if (xper) return occ(fv_step_pair_kernel<Sys, XM_PERIODIC, false, kWarps, 4>);
      return occ(fv_step_pair_kernel<Sys, XM_CLAMP, false, kWarps, 4>);
    }
    if (Dr == 6) {
      if (ctx->xg) return occ(fv_step_pair_kernel<Sys, XM_GHOST, false, kWarps, 6>);
      if (xper) return occ(fv_step_pair_kernel<Sys, XM_PERIODIC, false, kWarps, 6>);
      return occ(fv_step_pair_kernel<Sys, XM_CLAMP, false, kWarps, 6>);
    }
    if (ctx->xg) return occ(fv_step_pair_kernel<Sys, XM_GHOST, false, kWarps, 8>);
    if (xper) return occ(fv_step_pair_kernel<Sys, XM_PERIODIC, false, kWarps, 8>);
    return occ(fv_step_pair_kernel<Sys, XM_CLAMP, false, kWarps, 8>);
    }
  }
};

cudaError_t query_geometry(fv2d_ctx* ctx) {
  cudaError_t e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  switch (ctx->cfg.system) {
    case FV2D_ADVECTION: e = Occupancy<Advection>::run(ctx, &per_sm); break;
    case FV2D_EULER: e = Occupancy<Euler>::run(ctx, &per_sm); break;
    default: e = Occupancy<Spray>::run(ctx, &per_sm); break;
  }
  if (e != cudaSuccess) return e;
  ctx->slots = ctx->sms * std::max(1, per_sm);
  if (ctx->cfg.system == FV2D_SPRAY) {
    int src = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&src, spray_source_step_kernel, kSrcThreads, 0);
    if (e != cudaSuccess) return e;
    ctx->src_slots = ctx->sms * std::max(1, src);
  }
  return cudaSuccess;
}

// Persistent grid of the spray source pass over `rows` rows of `nslabs` slabs.
dim3 src_grid(const fv2d_ctx* ctx, int rows, int nslabs) {
  const long long tiles = (long long)rows * ((ctx->nx + kSrcThreads - 1) / kSrcThreads) * nslabs;
  return dim3((unsigned)std::max<long long>(1, std::min<long long>(tiles, std::max(1, ctx->src_slots))));
}

// Load every kernel a context can launch, and set the pair kernels' dynamic
// shared-memory opt-in, once per process and system at fv2d_create -- never
// while stepping.  Both a lazy module load and cudaFuncSetAttribute can wait
// for kernels already running in the same CUDA context; when several ranks of
// the peer-memory path share one process, a rank's spinning collective kernel
// would then hold back another rank's first step (a deadlock until the
// collective's timeout).  cudaFuncGetAttributes forces the load.
template <class F>
cudaError_t touch(F* f) {
  cudaFuncAttributes at;
  return cudaFuncGetAttributes(&at, (const void*)f);
}
template <class Sys, int D, int XM>
cudaError_t pair_attrs_x() {
  const int smem = kWarps * D * Sys::NV * 64 * (int)sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(fv_step_pair_kernel<Sys, XM, false, kWarps, D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaError_t e2 = cudaFuncSetAttribute(fv_step_pair_kernel<Sys, XM, true, kWarps, D>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if constexpr (kHasFast<Sys, D>) {
    cudaError_t e3 = cudaFuncSetAttribute(fv_step_pair_kernel<Sys, XM, true, kWarps, D, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e2 == cudaSuccess) e2 = e3;
  }
  return e != cudaSuccess ? e : e2;
}
template <class Sys, int D>
cudaError_t pair_attrs() {
  cudaError_t e = pair_attrs_x<Sys, D, XM_CLAMP>();
  if (e == cudaSuccess) e = pair_attrs_x<Sys, D, XM_PERIODIC>();
  if (e == cudaSuccess) e = pair_attrs_x<Sys, D, XM_GHOST>();
  return e;
}
template <class Sys>
struct Preload {
  static cudaError_t run() {
    cudaError_t e = cudaSuccess;
    auto t = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
    if constexpr (Sys::NV != 6) {  // spray transport always uses the one-cell kernel
      t(pair_attrs<Sys, 4>());
      t(pair_attrs<Sys, 6>());
      t(pair_attrs<Sys, 8>());
    }
    t(touch(fv_step_naive_kernel<Sys>));
    t(touch(reduce_smax_kernel<Sys>));
    t(touch(argmax_kernel<Sys>));
    t(touch(fv_step_kernel<Sys, true, false, kWarps, 4>));
    t(touch(fv_step_kernel<Sys, true, true, kWarps, 4>));
    t(touch(fv_step_kernel<Sys, false, false, kWarps, 4>));
    t(touch(fv_step_kernel<Sys, false, true, kWarps, 4>));
    t(touch(finalize_kernel));
    t(touch(peer_collective_kernel));
    t(touch(promote_pending_kernel));
    t(touch(spray_source_kernel));
    t(touch(spray_source_step_kernel));
    t(touch(spray_guard_kernel));
    t(touch(fill_halo_kernel));
    t(touch(fill_halo_cols_kernel));
    t(touch(unpack_col_kernel));
    t(touch(aos_to_dev_kernel));
    t(touch(dev_to_aos_kernel));
    return e;
  }
};
cudaError_t preload_kernels(int system, int device) {  // (the current device)
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({device, system})) return cudaSuccess;
  cudaError_t e;
  switch (system) {
    case FV2D_ADVECTION: e = Preload<Advection>::run(); break;
    case FV2D_EULER: e = Preload<Euler>::run(); break;
    default: e = Preload<Spray>::run(); break;
  }
  if (e == cudaSuccess) done.insert({device, system});
  return e;
}

int cur_parity(const fv2d_ctx* ctx) { return (int)(ctx->steps & 1); }

// NCCL halo exchange into ghost buffers of parity q, from send_s/send_n.
fv2d_status exchange(fv2d_ctx* ctx, int q, cudaStream_t stream = nullptr) {
  if (!ctx->use_nccl) return FV2D_OK;
  if (!stream) stream = ctx->stream;
  const int x = ctx->rx, y = ctx->ry, PY = ctx->py, PX = ctx->px;
  const bool per = ctx->cfg.bc_y == FV2D_BC_PERIODIC;
  const bool has_s = y > 0 || per, has_n = y < PY - 1 || per;
  const int rs_ = rank_at(ctx, x, y - 1), rn_ = rank_at(ctx, x, y + 1);
  const size_t cnt = (size_t)ctx->rs;  // one whole cell row: nv variable rows (ghost columns included)
  // Per peer, NCCL matches sends and receives in posting order; posting
  // "send to the lower side, receive from the upper side, send to the upper
  // side, receive from the lower side" keeps that correct when both sides are
  // the same peer (2 blocks along an axis).
  CKN(g_nccl.GroupStart());
  if (has_s) CKN(g_nccl.Send(ctx->send_s, cnt, ncclFloat64, rs_, ctx->comm, stream));
  if (has_n) CKN(g_nccl.Recv(ghost_n(ctx, 0, q) - ctx->xoff, cnt, ncclFloat64, rn_, ctx->comm, stream));
  if (has_n) CKN(g_nccl.Send(ctx->send_n, cnt, ncclFloat64, rn_, ctx->comm, stream));
  if (has_s) CKN(g_nccl.Recv(ghost_s(ctx, 0, q) - ctx->xoff, cnt, ncclFloat64, rs_, ctx->comm, stream));
  const bool perx = ctx->cfg.bc_x == FV2D_BC_PERIODIC;
  const bool has_w = ctx->xg && (x > 0 || perx), has_e = ctx->xg && (x < PX - 1 || perx);
  const int rw_ = rank_at(ctx, x - 1, y), re_ = rank_at(ctx, x + 1, y);
  const size_t cc = (size_t)ctx->nv * ctx->H;  // one packed column
  if (has_w) CKN(g_nccl.Send(ctx->send_w, cc, ncclFloat64, rw_, ctx->comm, stream));
  if (has_e) CKN(g_nccl.Recv(ctx->recv_e, cc, ncclFloat64, re_, ctx->comm, stream));
  if (has_e) CKN(g_nccl.Send(ctx->send_e, cc, ncclFloat64, re_, ctx->comm, stream));
  if (has_w) CKN(g_nccl.Recv(ctx->recv_w, cc, ncclFloat64, rw_, ctx->comm, stream));
  CKN(g_nccl.GroupEnd());
  const int nb = (ctx->H + 127) / 128;
  if (has_w) {
    unpack_col_kernel<<<nb, 128, 0, stream>>>(ctx->recv_w, row_ptr(ctx, 0, q, 0) - 1, ctx->nv, ctx->H, ctx->pitch,
                                               ctx->rs);
    CKL();
  }
  if (has_e) {
    unpack_col_kernel<<<nb, 128, 0, stream>>>(ctx->recv_e, row_ptr(ctx, 0, q, 0) + ctx->nx, ctx->nv, ctx->H,
                                               ctx->pitch, ctx->rs);
    CKL();
  }
  return FV2D_OK;
}

// max-all-reduce of [smax bits, pending status] into dscal[4..5].
fv2d_status allreduce_scalars(fv2d_ctx* ctx, cudaStream_t stream = nullptr) {
  CKN(g_nccl.AllReduce(ctx->dscal + 0, ctx->dscal + 4, 2, ncclUint64, ncclMax, ctx->comm,
                       stream ? stream : ctx->stream));
  return FV2D_OK;
}

// One collective point of the peer path: max-all-reduce dscal[0..1] -> dscal[4..5].
fv2d_status peer_collective(fv2d_ctx* ctx, cudaStream_t stream) {
  static const bool dbg = getenv("FV2D_DEBUG_PEER") != nullptr;
  if (dbg) fprintf(stderr, "[fv2d] rank %d collective epoch %llu steps %lld\n", ctx->cfg.rank, ctx->epoch, ctx->steps);
  peer_collective_kernel<<<1, 32, 0, stream>>>(ctx->pa, ctx->dscal + 0, ctx->dscal + 4, ctx->epoch, ctx->dscal + 2);
  ++ctx->epoch;
  ++ctx->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ctx, FV2D_E_CUDA, "launch failed: %s", cudaGetErrorString(e));
  return FV2D_OK;
}

// Cross-rank reduction of [smax, pending] after a local pass: NCCL or peer memory.
fv2d_status reduce_ranks(fv2d_ctx* ctx, cudaStream_t stream) {
  if (ctx->peer) return peer_collective(ctx, stream);
  return allreduce_scalars(ctx, stream);
}

fv2d_status ensure_dt_log(fv2d_ctx* ctx, long long need) {
  if (need <= ctx->dt_log_cap) return FV2D_OK;
  long long cap = std::max<long long>(need, std::max<long long>(1024, 2 * ctx->dt_log_cap));
  double* nb = nullptr;
  // stream-ordered: no legacy-stream or device-wide synchronisation while
  // stepping (ranks of a peer group may be waiting on this one's progress)
  CK(cudaMallocAsync(&nb, cap * sizeof(double), ctx->stream));
  CK(cudaMemsetAsync(nb, 0, cap * sizeof(double), ctx->stream));
  if (ctx->dt_log) {
    CK(cudaMemcpyAsync(nb, ctx->dt_log, ctx->dt_log_cap * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaFreeAsync(ctx->dt_log, ctx->stream));
  }
  ctx->dt_log = nb;
  ctx->dt_log_cap = cap;
  return FV2D_OK;
}

// Device -> host copy of n (<= 8) words through the pinned scratch, synchronous.
fv2d_status d2h_words(fv2d_ctx* ctx, unsigned long long* dst, const unsigned long long* src, int n) {
  CK(cudaMemcpyAsync(ctx->hpin, src, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  memcpy(dst, ctx->hpin, n * sizeof(unsigned long long));
  return FV2D_OK;
}

fv2d_status read_status(fv2d_ctx* ctx, unsigned long long* st_out) {
  fv2d_status s0 = d2h_words(ctx, st_out, ctx->dscal + 2, 1);
  if (s0 || ctx->journal.empty()) return s0;
  if (*st_out == 0) {  // every journaled step completed without a latched error
    ctx->journal.clear();
    return FV2D_OK;
  }
  bool redone = false;
  s0 = recover_fast(ctx, *st_out, &redone);
  if (s0) return s0;
  return redone ? read_status(ctx, st_out) : FV2D_OK;
}

// Translate a latched status word into an error code + description.
fv2d_status report(fv2d_ctx* ctx, unsigned long long st);

// Smax of the current state over all slabs/ranks -> dscal[0] (or [4] after all-reduce).
fv2d_status reduce_current(fv2d_ctx* ctx, double* smax_out, unsigned long long* pending_out) {
  StepArgs a = make_args(ctx, cur_parity(ctx));
  CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
  dispatch<LaunchReduce>(ctx->cfg.system, ctx, a);
  CKL();
  unsigned long long h[2];
  if (ctx->use_nccl || ctx->peer) {
    fv2d_status s = reduce_ranks(ctx, ctx->stream);
    if (s) return s;
    CK(cudaMemcpyAsync(ctx->hpin, ctx->dscal + 4, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    CK(cudaMemcpyAsync(ctx->hpin, ctx->dscal + 0, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  memcpy(h, ctx->hpin, sizeof h);
  double s;
  memcpy(&s, &h[0], sizeof s);
  *smax_out = s;
  *pending_out = h[1];
  return FV2D_OK;
}

fv2d_status report(fv2d_ctx* ctx, unsigned long long st) {
  if (st == 0) return FV2D_OK;
  const int code = (int)(st >> 56);
  const long long step = (long long)(st & 0x00FFFFFFFFFFFFFFull);
  ctx->err_step = step;
  unsigned long long bc = ~0ull;
  if (d2h_words(ctx, &bc, ctx->dscal + 3, 1) != FV2D_OK) bc = ~0ull;
  ctx->err_cell = bc == ~0ull ? -1 : (long long)bc;
  switch (code) {
    case ST_CFL:
      return set_err(ctx, FV2D_E_CFL, "CFL violated at the start of step %lld: dt*smax > min(dx,dy) (cell %lld)",
                     step, ctx->err_cell);
    case ST_NONFINITE:
      return set_err(ctx, FV2D_E_NONFINITE, "non-admissible state W^%lld (cell %lld)", step, ctx->err_cell);
    case ST_COMM:
      return set_err(ctx, FV2D_E_NCCL, "peer-memory collective timed out at epoch %lld (a rank did not arrive)", step);
    case ST_RECON:
      return set_err(ctx, FV2D_E_RECON, "NDF reconstruction failed in step %lld (cell %lld)", step, ctx->err_cell);
    default:
      return set_err(ctx, FV2D_E_STATE, "unknown latched status %llx", st);
  }
}

// Locate the diagnostic cell of a latched error on the state W^k.
fv2d_status diagnose(fv2d_ctx* ctx, unsigned long long st) {
  const int code = (int)(st >> 56);
  const long long step = (long long)(st & 0x00FFFFFFFFFFFFFFull);
  const int p = (int)(step & 1);
  StepArgs a = make_args(ctx, p);
  if (code == ST_CFL || code == ST_NONFINITE) {
    CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
    CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
    dispatch<LaunchReduce>(ctx->cfg.system, ctx, a);
    CKL();
    unsigned long long h[2];
    fv2d_status s2 = d2h_words(ctx, h, ctx->dscal, 2);
    if (s2) return s2;
    double smax;
    memcpy(&smax, &h[0], sizeof smax);
    if (code == ST_CFL) {
      ctx->err_value = smax;
      CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
      dispatch<LaunchArgmax>(ctx->cfg.system, ctx, a, smax, ctx->dscal + 3);
      CKL();
    }
    CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return FV2D_OK;
}

}  // namespace

// ============================================================== C ABI
extern "C" {

fv2d_status fv2d_version(int32_t* major, int32_t* minor) {
  if (major) *major = FV2D_VERSION_MAJOR;
  if (minor) *minor = FV2D_VERSION_MINOR;
  return FV2D_OK;
}

fv2d_status fv2d_config_default(fv2d_config* cfg, int32_t nx, int32_t ny, int32_t system) {
  if (!cfg) return FV2D_E_ARG;
  memset(cfg, 0, sizeof *cfg);
  cfg->nx = nx;
  cfg->ny = ny;
  cfg->system = system;
  cfg->nvar = nvar_of(system);
  cfg->x0 = 0.0; cfg->x1 = 1.0; cfg->y0 = 0.0; cfg->y1 = 1.0;
  if (system == FV2D_EULER) cfg->param[0] = 1.4;
  if (system == FV2D_ADVECTION) { cfg->param[0] = 1.0; cfg->param[1] = 0.5; }
  if (system == FV2D_SPRAY) { cfg->param[0] = 1.0; cfg->param[1] = 1.0; }
  cfg->rank = 0;
  cfg->nranks = 1;
  cfg->nslabs = 1;
  return cfg->nvar > 0 ? FV2D_OK : FV2D_E_ARG;
}

fv2d_status fv2d_nccl_unique_id(uint8_t id[128]) {
  if (!id) return FV2D_E_ARG;
  if (!load_nccl()) return FV2D_E_NCCL;
  ncclUniqueId u;
  if (g_nccl.GetUniqueId(&u) != ncclSuccess) return FV2D_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return FV2D_OK;
}

fv2d_status fv2d_destroy(fv2d_ctx* ctx) {
  if (!ctx) return FV2D_OK;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (int s = 0; s < kMaxSlabs; ++s)
    for (int p = 0; p < 2; ++p)
      if (ctx->buf[s][p]) cudaFree(ctx->buf[s][p]);
  if (ctx->send_s) cudaFree(ctx->send_s);
  if (ctx->send_n) cudaFree(ctx->send_n);
  for (double* b : {ctx->send_w, ctx->send_e, ctx->recv_w, ctx->recv_e})
    if (b) cudaFree(b);
  if (ctx->staging) cudaFree(ctx->staging);
  if (ctx->staging_out) cudaFree(ctx->staging_out);
  for (cudaEvent_t e : ctx->ev_band) cudaEventDestroy(e);
  if (ctx->h2d_stream) cudaStreamDestroy(ctx->h2d_stream);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  if (ctx->dscal) cudaFree(ctx->dscal);
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  if (ctx->done) cudaFree(ctx->done);
  if (ctx->dt_dev) cudaFree(ctx->dt_dev);
  if (ctx->dt_log) cudaFree(ctx->dt_log);
  if (ctx->newton) cudaFree(ctx->newton);
  if (ctx->trig) cudaFree(ctx->trig);
  for (double* b : ctx->lam_buf)
    if (b) cudaFree(b);
  if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  if (ctx->sync) cudaFree(ctx->sync);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->ev_bnd) cudaEventDestroy(ctx->ev_bnd);
  if (ctx->ev_int) cudaEventDestroy(ctx->ev_int);
  if (ctx->ev_fin) cudaEventDestroy(ctx->ev_fin);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  for (int p = 0; p < 2; ++p)
    if (ctx->graph[p]) cudaGraphExecDestroy(ctx->graph[p]);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->out_stream) {
    cudaStreamSynchronize(ctx->out_stream);
    cudaStreamDestroy(ctx->out_stream);
  }
  if (ctx->ev_snap_start) cudaEventDestroy(ctx->ev_snap_start);
  if (ctx->ev_snap_conv) cudaEventDestroy(ctx->ev_snap_conv);
  if (ctx->snap_buf) cudaFree(ctx->snap_buf);
  delete ctx;
  return FV2D_OK;
}

fv2d_status fv2d_create(const fv2d_config* cfg_in, const uint8_t* nccl_id, void* cuda_stream, fv2d_ctx** out) {
  if (!cfg_in || !out) return FV2D_E_ARG;
  *out = nullptr;
  const fv2d_config& c = *cfg_in;
  const int nv = nvar_of(c.system);
  if (nv < 0 || c.nvar != nv || c.nx < 1 || c.ny < 1 || c.nranks < 1 || c.rank < 0 || c.rank >= c.nranks ||
      c.nslabs < 1 || c.nslabs > kMaxSlabs || ((c.nranks > 1 || (c.flags & FV2D_FLAG_NCCL_LOOPBACK)) && c.nslabs != 1) ||
      !(c.x1 > c.x0) || !(c.y1 > c.y0) || c.bc_x < 0 || c.bc_x > 2 || c.bc_y < 0 || c.bc_y > 2)
    return FV2D_E_ARG;
  // the rank grid before any division by it: 0 <= nranks_x <= nranks, nranks % nranks_x == 0
  if (c.nranks_x < 0 || c.nranks_x > c.nranks || (c.nranks_x > 1 && c.nranks % c.nranks_x != 0)) return FV2D_E_ARG;
  if (c.ny % ((c.nranks_x > 1 ? c.nranks / c.nranks_x : c.nranks) * c.nslabs) != 0) return FV2D_E_ARG;
  if (c.system == FV2D_ADVECTION && (c.bc_x == FV2D_BC_WALL || c.bc_y == FV2D_BC_WALL)) return FV2D_E_ARG;
  if (c.system == FV2D_EULER && !(c.param[0] > 1.0)) return FV2D_E_ARG;
  if (c.system == FV2D_SPRAY && !(c.param[1] > 0.0)) return FV2D_E_ARG;
  // FV2D_FLAG_FUSE_SOURCE (a one-pass spray step) was measured slower than the
  // split source pass on B200 and removed; the bit stays reserved
  if (c.flags & FV2D_FLAG_FUSE_SOURCE) return FV2D_E_ARG;
  for (int k = 0; k < 4; ++k)
    if (c.reserved[k] != 0) return FV2D_E_ARG;
  // 2-D rank blocks (nranks_x > 1): nranks_x x (nranks/nranks_x) blocks
  const int px = c.nranks_x <= 1 ? 1 : c.nranks_x;
  // stored ghost columns: 2-D blocks, the test flag, and every non-periodic x
  // boundary (wall/Dirichlet ghosts then live in the buffer instead of being
  // built in registers: the pair kernel's XM_GHOST mode carries no per-cell
  // boundary code; 2.92 vs 3.42 ms at 16384²)
  const bool xg = px > 1 || (c.flags & FV2D_FLAG_GHOST_COLUMNS) || c.bc_x != FV2D_BC_PERIODIC;
  if (c.nranks_x < 0 || c.nranks % px != 0 || c.nx % px != 0 || c.nx / px < 2 || (px > 1 && c.nslabs != 1))
    return FV2D_E_ARG;
  const int py = c.nranks / px;
  const int nxl = c.nx / px;
  if (c.tiles_x < 0 || c.tiles_y < 0 || c.tiles_x > 256 || c.tiles_y > 256) return FV2D_E_ARG;
  const long long H = c.ny / (py * c.nslabs);
  if (H < 1) return FV2D_E_ARG;
  if (std::max(1, c.tiles_y) > H || 2 * std::max(1, c.tiles_x) > nxl) return FV2D_E_ARG;
  const bool peer = (c.flags & FV2D_FLAG_PEER_HALO) != 0;
  if (peer && (c.nranks < 2 || c.nranks > kMaxRanks || c.nslabs != 1 || (c.flags & FV2D_FLAG_NCCL_LOOPBACK)))
    return FV2D_E_ARG;
  const bool use_nccl = !peer && (c.nranks > 1 || (c.flags & FV2D_FLAG_NCCL_LOOPBACK));
  if (use_nccl && (!nccl_id || !load_nccl())) return FV2D_E_NCCL;

  fv2d_ctx* ctx = new fv2d_ctx();
  ctx->cfg = c;
  ctx->use_nccl = use_nccl;
  ctx->peer = peer;
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->launch_stream = ctx->stream;
  ctx->tiles_x = std::max(1, c.tiles_x);
  ctx->tiles_y = std::max(1, c.tiles_y);
  ctx->nv = nv;
  ctx->px = px;
  ctx->py = py;
  ctx->rx = c.rank % px;
  ctx->ry = c.rank / px;
  ctx->gnx = c.nx;
  ctx->nx = nxl;
  ctx->col0 = ctx->rx * nxl;
  ctx->xg = xg;
  ctx->xoff = xg ? 2 : 0;  // row: [pad, ghost -1 | 0 .. nx-1 | ghost nx, ...]
  ctx->H = (int)H;
  ctx->pitch = (nxl + ctx->xoff + (xg ? 1 : 0) + 31) / 32 * 32;
  if (const char* e = getenv("FV2D_RING_DEPTH")) ctx->ring_depth = atoi(e);  // tuning knob
  {
    // FAST pair kernel (see fv2d_ctx::fast_ok): single rank, default kernel and
    // ring, and a Dirichlet state (never an output cell, so never checked by the
    // kernel) whose derive stays inside the fast range: 1e-300 < rho < 1e300,
    // p > 0 and 1e-300 < gamma p / rho < 1e300
    bool dir_ok = true;
    if (c.system == FV2D_EULER && (c.bc_x == FV2D_BC_DIRICHLET || c.bc_y == FV2D_BC_DIRICHLET)) {
      const double rho = c.dirichlet[0], mx = c.dirichlet[1], my = c.dirichlet[2], E = c.dirichlet[3];
      const double g = c.param[0], inv = 1.0 / rho, p = (g - 1.0) * (E - 0.5 * (mx * mx + my * my) * inv),
                   X = g * p * inv;
      dir_ok = rho > 1e-300 && rho < 1e300 && p > 0.0 && X > 1e-300 && X < 1e300 && std::isfinite(E);
    }
    const char* ex = getenv("FV2D_EXACT_DIV");  // 1: never the FAST kernel (A/B knob)
    ctx->fast_ok = c.system == FV2D_EULER && !use_nccl && !peer && c.nranks <= 1 && ctx->ring_depth == 4 &&
                   !(c.flags & (FV2D_FLAG_NAIVE | FV2D_FLAG_ONE_CELL)) && dir_ok && !(ex && atoi(ex) == 1);
  }
  ctx->rs = (long long)ctx->pitch * nv;
  ctx->nslabs = c.nslabs;
  ctx->G = py * c.nslabs;
  ctx->dx = (c.x1 - c.x0) / c.nx;
  ctx->dy = (c.y1 - c.y0) / c.ny;
  ctx->hmin = ctx->dx < ctx->dy ? ctx->dx : ctx->dy;

  auto fail = [&](fv2d_status s) {
    std::string m = ctx->err;
    fv2d_destroy(ctx);
    (void)m;
    return s;
  };
#define CKC(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      fprintf(stderr, "fv2d_create: %s failed: %s\n", #call, cudaGetErrorString(e_));              \
      return fail(FV2D_E_CUDA);                                                                    \
    }                                                                                              \
  } while (0)
  CKC(cudaSetDevice(c.device));
  const size_t state_bytes = ((size_t)(H + 2) * ctx->rs + 64) * sizeof(double);
  const size_t row_bytes = (size_t)ctx->rs * sizeof(double);
  for (int s = 0; s < ctx->nslabs; ++s)
    for (int p = 0; p < 2; ++p) {
      CKC(cudaMalloc(&ctx->buf[s][p], state_bytes));
      CKC(cudaMemset(ctx->buf[s][p], 0, state_bytes));
    }
  if (use_nccl) {
    CKC(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    CKC(cudaEventCreateWithFlags(&ctx->ev_bnd, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_int, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_fin, cudaEventDisableTiming));
    CKC(cudaMalloc(&ctx->send_s, row_bytes));
    CKC(cudaMalloc(&ctx->send_n, row_bytes));
    CKC(cudaMemset(ctx->send_s, 0, row_bytes));
    CKC(cudaMemset(ctx->send_n, 0, row_bytes));
    if (xg) {
      const size_t col_bytes = (size_t)nv * H * sizeof(double);
      for (double** b : {&ctx->send_w, &ctx->send_e, &ctx->recv_w, &ctx->recv_e}) {
        CKC(cudaMalloc(b, col_bytes));
        CKC(cudaMemset(*b, 0, col_bytes));
      }
    }
  }
  CKC(preload_kernels(c.system, c.device));
  CKC(query_geometry(ctx));
  ctx->rps = pick_rps(ctx, nxl, (int)H);
  if (peer) {
    CKC(cudaMalloc(&ctx->sync, sizeof(PeerSync)));
    CKC(cudaMemset(ctx->sync, 0, sizeof(PeerSync)));
  }
  CKC(cudaMalloc(&ctx->dscal, 8 * sizeof(unsigned long long)));
  CKC(cudaHostAlloc(&ctx->hpin, 16 * sizeof(unsigned long long), cudaHostAllocPortable));
  CKC(cudaMemset(ctx->dscal, 0, 8 * sizeof(unsigned long long)));
  CKC(cudaMemset(ctx->dscal + 3, 0xff, sizeof(unsigned long long)));
  CKC(cudaMalloc(&ctx->done, sizeof(unsigned int)));
  CKC(cudaMemset(ctx->done, 0, sizeof(unsigned int)));
  CKC(cudaMalloc(&ctx->dt_dev, sizeof(double)));
  CKC(cudaMemset(ctx->dt_dev, 0, sizeof(double)));
  ctx->dt_log_cap = 1 << 16;  // grown stream-ordered by ensure_dt_log if a run is longer
  CKC(cudaMalloc(&ctx->dt_log, ctx->dt_log_cap * sizeof(double)));
  CKC(cudaMemset(ctx->dt_log, 0, ctx->dt_log_cap * sizeof(double)));
  CKC(cudaMalloc(&ctx->newton, sizeof(unsigned long long)));
  CKC(cudaMemset(ctx->newton, 0, sizeof(unsigned long long)));
  if (c.system == FV2D_SPRAY) {
    CKC(cudaMalloc(&ctx->trig, (size_t)(2 * c.nx + 2 * c.ny) * sizeof(double)));
    for (double*& b : ctx->lam_buf) CKC(cudaMalloc(&b, (size_t)ctx->nslabs * H * 4 * ctx->pitch * sizeof(double)));
    trig_table_kernel<<<(c.nx + 255) / 256, 256>>>(ctx->trig, ctx->trig + c.nx, c.nx, c.x0, ctx->dx);
    trig_table_kernel<<<(c.ny + 255) / 256, 256>>>(ctx->trig + 2 * c.nx, ctx->trig + 2 * c.nx + c.ny, c.ny, c.y0,
                                                    ctx->dy);
    CKC(cudaGetLastError());
    // __constant__ symbols exist once per device: upload the table to every
    // device a spray context is created on (under the preload mutex: contexts
    // may be created from several threads)
    {
      static std::mutex gl_mu;
      static std::set<int> gl_devices;
      std::lock_guard<std::mutex> lk(gl_mu);
      if (!gl_devices.count(c.device)) {
        double t[24], wt[24][kGLW];
        gl24_table(t, wt);
        CKC(cudaMemcpyToSymbol(c_gl_t, t, sizeof t));
        CKC(cudaMemcpyToSymbol(c_gl_wt, wt, sizeof wt));
        double e2[64];  // 2^(j/64), correctly rounded from long double (exp_tab)
        for (int jj = 0; jj < 64; ++jj) e2[jj] = (double)exp2l((long double)jj / 64.0L);
        CKC(cudaMemcpyToSymbol(c_exp2_64, e2, sizeof e2));
        gl_devices.insert(c.device);
      }
    }
  }
  // Dirichlet ghost rows are constant for the whole run.
  if (c.bc_y == FV2D_BC_DIRICHLET) {
    for (int s = 0; s < ctx->nslabs; ++s) {
      const int g = ctx->ry * c.nslabs + s;
      for (int p = 0; p < 2; ++p) {
        if (g == 0)
          fill_const_row_kernel<<<(nxl + 255) / 256, 256>>>(ghost_s(ctx, s, p), nv, nxl, ctx->pitch, c.dirichlet[0],
                                                            c.dirichlet[1], c.dirichlet[2], c.dirichlet[3],
                                                            c.dirichlet[4], c.dirichlet[5]);
        if (g == ctx->G - 1)
          fill_const_row_kernel<<<(nxl + 255) / 256, 256>>>(ghost_n(ctx, s, p), nv, nxl, ctx->pitch, c.dirichlet[0],
                                                            c.dirichlet[1], c.dirichlet[2], c.dirichlet[3],
                                                            c.dirichlet[4], c.dirichlet[5]);
      }
    }
    CKC(cudaGetLastError());
  }
  // ... and so are Dirichlet ghost columns of blocks on the global x boundary
  if (xg && c.bc_x == FV2D_BC_DIRICHLET) {
    for (int s = 0; s < ctx->nslabs; ++s)
    for (int p = 0; p < 2; ++p) {
      double* cols[2] = {ctx->rx == 0 ? ghost_s(ctx, s, p) - 1 : nullptr,
                         ctx->rx == px - 1 ? ghost_s(ctx, s, p) + nxl : nullptr};
      for (double* col : cols)
        if (col)
          fill_const_col_kernel<<<(int)((H + 2 + 127) / 128), 128>>>(col, nv, (int)H + 2, ctx->pitch, ctx->rs,
                                                                     c.dirichlet[0], c.dirichlet[1], c.dirichlet[2],
                                                                     c.dirichlet[3], c.dirichlet[4], c.dirichlet[5]);
    }
    CKC(cudaGetLastError());
  }
  CKC(cudaDeviceSynchronize());
  if (use_nccl) {
    ncclUniqueId u;
    memcpy(&u, nccl_id, sizeof u);
    if (g_nccl.CommInitRank(&ctx->comm, c.nranks, u, c.rank) != ncclSuccess) return fail(FV2D_E_NCCL);
  }
#undef CKC
  *out = ctx;
  return FV2D_OK;
}

static fv2d_status after_set_state(fv2d_ctx* ctx) {
  // ghost rows of parity 0 from the new W^0, then reset the counters
  ctx->steps = 0;
  StepArgs a = make_args(ctx, 1);  // "reading" parity 1 means ghost targets of parity 0
  for (int s = 0; s < ctx->nslabs; ++s) a.slab[s].in = row_ptr(ctx, s, 0, 0);
  fill_halo_kernel<<<dim3((ctx->nx + 127) / 128, 1, ctx->nslabs), 128, 0, ctx->stream>>>(a, ctx->nv);
  CKL();
  if (ctx->xg) {
    fill_halo_cols_kernel<<<dim3((ctx->H + 127) / 128, 1, ctx->nslabs), 128, 0, ctx->stream>>>(a, ctx->nv);
    CKL();
  }
  fv2d_status st = exchange(ctx, 0);
  if (st) return st;
  if (ctx->peer) {
    // barrier: every rank has written its halo rows into its neighbours' ghost rows
    CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
    st = peer_collective(ctx, ctx->stream);
    if (st) return st;
  }
  // dscal = {0, 0, 0, ~0, 0, 0, 0, 0} (no pageable host source, see hpin)
  CK(cudaMemsetAsync(ctx->dscal, 0, 8 * sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->done, 0, sizeof(unsigned int), ctx->stream));
  CK(cudaMemsetAsync(ctx->dt_dev, 0, sizeof(double), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->has_state = true;
  ctx->dt_valid = false;
  ctx->guard_done = false;
  ctx->lam_hist = 0;
  ctx->journal.clear();
  ctx->err.clear();
  ctx->err_step = ctx->err_cell = -1;
  return FV2D_OK;
}

static fv2d_status ensure_staging(fv2d_ctx* ctx) {
  const size_t need = (size_t)ctx->nv * ctx->nx * ctx->H * ctx->nslabs * sizeof(double);
  if (ctx->staging_bytes >= need) return FV2D_OK;
  if (ctx->staging) CK(cudaFreeAsync(ctx->staging, ctx->stream));
  ctx->staging = nullptr;
  CK(cudaMallocAsync(&ctx->staging, need, ctx->stream));
  ctx->staging_bytes = need;
  return FV2D_OK;
}

static fv2d_status upload(fv2d_ctx* ctx, const double* src, fv2d_layout layout, cudaMemcpyKind kind) {
  CK(cudaSetDevice(ctx->cfg.device));
  if (ctx->snap_parity >= 0) {
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_snap_conv, 0));
    ctx->snap_parity = -1;
  }
  const int nv = ctx->nv, nx = ctx->nx, H = ctx->H;
  if (layout == FV2D_SOA) {
    // SoA [nv][ny_local][nx]: per variable, slab rows are contiguous in the source
    const long long nyl = (long long)H * ctx->nslabs;
    for (int s = 0; s < ctx->nslabs; ++s)
      for (int v = 0; v < nv; ++v)
        CK(cudaMemcpy2DAsync(row_ptr(ctx, s, 0, 0) + v * ctx->pitch, ctx->rs * sizeof(double),
                             src + (size_t)v * nyl * nx + (size_t)s * H * nx, nx * sizeof(double),
                             nx * sizeof(double), H, kind, ctx->stream));
  } else {
    fv2d_status st = ensure_staging(ctx);
    if (st) return st;
    const size_t bytes = (size_t)nv * nx * H * ctx->nslabs * sizeof(double);
    CK(cudaMemcpyAsync(ctx->staging, src, bytes, kind, ctx->stream));
    for (int s = 0; s < ctx->nslabs; ++s) {
      aos_to_dev_kernel<<<num_sms(ctx) * 8, 256, 0, ctx->stream>>>(ctx->staging + (size_t)s * H * nx * nv,
                                                          row_ptr(ctx, s, 0, 0), nv, nx, H, ctx->pitch, ctx->rs);
      CKL();
    }
  }
  return after_set_state(ctx);
}

fv2d_status fv2d_set_state(fv2d_ctx* ctx, const double* host, fv2d_layout layout) {
  if (!ctx || !host || (layout != FV2D_AOS && layout != FV2D_SOA)) return FV2D_E_ARG;
  if (ctx->peer && !ctx->peer_connected) return set_err(ctx, FV2D_E_STATE, "peer halo: call fv2d_peer_connect first");
  return upload(ctx, host, layout, cudaMemcpyHostToDevice);
}

fv2d_status fv2d_set_state_device(fv2d_ctx* ctx, const double* dev, fv2d_layout layout) {
  if (!ctx || !dev || (layout != FV2D_AOS && layout != FV2D_SOA)) return FV2D_E_ARG;
  if (ctx->peer && !ctx->peer_connected) return set_err(ctx, FV2D_E_STATE, "peer halo: call fv2d_peer_connect first");
  return upload(ctx, dev, layout, cudaMemcpyDeviceToDevice);
}

fv2d_status fv2d_get_state(fv2d_ctx* ctx, double* host, fv2d_layout layout) {
  if (!ctx || !host || (layout != FV2D_AOS && layout != FV2D_SOA)) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  CK(cudaSetDevice(ctx->cfg.device));
  unsigned long long st;
  fv2d_status s0 = read_status(ctx, &st);
  if (s0) return s0;
  const int p = st ? (int)((st & 0x00FFFFFFFFFFFFFFull) & 1) : cur_parity(ctx);
  const int nv = ctx->nv, nx = ctx->nx, H = ctx->H;
  if (layout == FV2D_SOA) {
    const long long nyl = (long long)H * ctx->nslabs;
    for (int s = 0; s < ctx->nslabs; ++s)
      for (int v = 0; v < nv; ++v)
        CK(cudaMemcpy2DAsync(host + (size_t)v * nyl * nx + (size_t)s * H * nx, nx * sizeof(double),
                             row_ptr(ctx, s, p, 0) + v * ctx->pitch, ctx->rs * sizeof(double), nx * sizeof(double),
                             H, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    fv2d_status s1 = ensure_staging(ctx);
    if (s1) return s1;
    for (int s = 0; s < ctx->nslabs; ++s) {
      dev_to_aos_kernel<<<num_sms(ctx) * 8, 256, 0, ctx->stream>>>(row_ptr(ctx, s, p, 0),
                                                          ctx->staging + (size_t)s * H * nx * nv, nv, nx, H,
                                                          ctx->pitch, ctx->rs);
      CKL();
    }
    CK(cudaMemcpyAsync(host, ctx->staging, (size_t)nv * nx * H * ctx->nslabs * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return report(ctx, st);
}

fv2d_status fv2d_compute_dt(fv2d_ctx* ctx, double cfl, double* dt, double* smax) {
  if (!ctx || !(cfl > 0.0) || !(cfl <= 1.0)) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  CK(cudaSetDevice(ctx->cfg.device));
  unsigned long long st;
  fv2d_status s0 = read_status(ctx, &st);
  if (s0) return s0;
  if (st) return report(ctx, st);
  double s;
  unsigned long long pend;
  s0 = reduce_current(ctx, &s, &pend);
  if (s0) return s0;
  if (smax) *smax = s;
  if (pend) {
    const unsigned long long w = ((unsigned long long)ST_NONFINITE << 56) | (unsigned long long)ctx->steps;
    return report(ctx, w);
  }
  const double d = (cfl * ctx->hmin) / s;
  if (dt) *dt = d;
  memcpy(ctx->hpin + 8, &d, sizeof d);
  CK(cudaMemcpyAsync(ctx->dt_dev, ctx->hpin + 8, sizeof d, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->dt_valid = true;
  ctx->dt_cfl = cfl;
  return FV2D_OK;
}

fv2d_status fv2d_check_dt(fv2d_ctx* ctx, double dt, double* smax) {
  if (!ctx || !(dt > 0.0)) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  CK(cudaSetDevice(ctx->cfg.device));
  if (!ctx->journal.empty()) {
    unsigned long long st0;
    fv2d_status s0 = read_status(ctx, &st0);
    if (s0) return s0;
  }
  double s;
  unsigned long long pend;
  fv2d_status s0 = reduce_current(ctx, &s, &pend);
  if (s0) return s0;
  if (smax) *smax = s;
  if (pend) return set_err(ctx, FV2D_E_NONFINITE, "non-admissible state");
  if (dt * s > ctx->hmin) {
    ctx->err_value = s;
    return set_err(ctx, FV2D_E_CFL, "dt*smax = %.17g > min(dx,dy) = %.17g", dt * s, ctx->hmin);
  }
  return FV2D_OK;
}

static fv2d_status prof_flush(fv2d_ctx* ctx) {
  if (ctx->ev_used == 0) return FV2D_OK;
  CK(cudaEventSynchronize(ctx->ev_pool[ctx->ev_used - 1]));
  for (size_t k = 0; k + 1 < ctx->ev_used; k += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev_pool[k], ctx->ev_pool[k + 1]));
    if (ctx->ev_tag[k / 2]) {
      ctx->prof_src_ms += ms;
      ctx->prof_src_n += 1;
    } else {
      ctx->prof_ms += ms;
      ctx->prof_n += 1;
    }
  }
  ctx->ev_used = 0;
  return FV2D_OK;
}

static fv2d_status prof_events(fv2d_ctx* ctx, cudaEvent_t* e0, cudaEvent_t* e1, char tag = 0) {
  // flush only at a step's first pair (tag 0), keeping room for its source pair,
  // so no pair is ever read before both of its events are recorded
  if (tag == 0 && ctx->ev_used + 4 > 4096) {
    fv2d_status st = prof_flush(ctx);
    if (st) return st;
  }
  while (ctx->ev_pool.size() < ctx->ev_used + 2) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->ev_pool.push_back(e);
  }
  *e0 = ctx->ev_pool[ctx->ev_used];
  *e1 = ctx->ev_pool[ctx->ev_used + 1];
  if (ctx->ev_tag.size() < ctx->ev_used / 2 + 1) ctx->ev_tag.resize(ctx->ev_used / 2 + 1);
  ctx->ev_tag[ctx->ev_used / 2] = tag;
  ctx->ev_used += 2;
  return FV2D_OK;
}

// The split source pass of a step: dt is the fixed dt or, in adaptive mode,
// the device scalar (read inside the kernel so the launch stays asynchronous).
static void spray_source_dt_kernel_launch(fv2d_ctx* ctx, const StepArgs& a, dim3 grid, int p) {
  StepArgs b = a;
  for (int s = 0; s < ctx->nslabs; ++s) b.slab[s].out = row_ptr(ctx, s, 1 - p, 0);
  spray_source_step_kernel<<<grid, kSrcThreads, 0, ctx->launch_stream>>>(b);
}

// The launches of one time step reading parity p, on ctx->launch_stream (the
// caller's stream, or the capture stream while recording a CUDA graph).
static fv2d_status issue_step(fv2d_ctx* ctx, int p, int adaptive, double dt, double cfl, cudaEvent_t e1,
                              bool fast) {
  fv2d_status st = FV2D_OK;
  const bool split = ctx->cfg.system == FV2D_SPRAY;
  const bool tiled = ctx->tiles_x * ctx->tiles_y > 1 && !(ctx->cfg.flags & FV2D_FLAG_NAIVE);
  StepArgs a = make_args(ctx, p);
  a.adaptive = adaptive;
  a.fast = fast ? 1 : 0;
  a.dt = dt;
  a.cfl = cfl;
  a.step = ctx->steps;
  if (ctx->use_nccl || tiled) a.fused_finalize = 0;
  // peer-memory path, one launch per pass: the pass's last CTA does the
  // max-all-reduce over the ranks and the finalize (StepArgs::peer_fused)
  const bool peer_fused = ctx->peer && !tiled && !(ctx->cfg.flags & FV2D_FLAG_PEER_SPLIT);
  if (peer_fused) {
    a.fused_finalize = 1;
    a.peer_fused = 1;
    a.peer = ctx->pa;
    static const bool dbg = getenv("FV2D_DEBUG_PEER") != nullptr;
    if (dbg) fprintf(stderr, "[fv2d] rank %d step collective epoch %llu steps %lld\n", ctx->cfg.rank, ctx->epoch, ctx->steps);
    a.peer_epoch = ctx->epoch++;
  }
  StepArgs at = a;  // transport pass
  if (split) {
    at.fused_finalize = 0;  // the source pass ends the step
    at.no_smax = 1;         // adaptive: smax of the post-source state comes from the source pass
  }
  cudaStream_t ls = ctx->launch_stream;
  // NCCL path for transport-only systems: boundary strips first (rows, and
  // with ghost columns the west/east column strips too), halo exchange on the
  // comm stream overlapped with the interior.
  const int hb = 8, cb = 64;  // boundary rows / columns (even: column cuts are on even columns)
  const bool overlap = ctx->use_nccl && !split && !tiled && !(ctx->cfg.flags & FV2D_FLAG_NAIVE) &&
                       ctx->H > 4 * hb && (!ctx->xg || ctx->nx >= 4 * cb);
  if (overlap) {
    StepArgs ab = at, ai = at;
    set_ranges(ab, 0, hb, hb, ctx->H - hb, ctx->H, hb);
    set_ranges(ai, hb, ctx->H - hb, ctx->rps, 0, 0, 1);
    dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, ab);
    CKL();
    if (ctx->xg) {  // column strips [0, cb) and [ce, nx) of the interior rows
      const int ce = (ctx->nx - cb) & ~1;
      StepArgs bw = at, be = at;
      set_ranges(bw, hb, ctx->H - hb, pick_rps(ctx, cb, ctx->H - 2 * hb), 0, 0, 1);
      set_ranges(be, hb, ctx->H - hb, pick_rps(ctx, ctx->nx - ce, ctx->H - 2 * hb), 0, 0, 1);
      bw.col_lo = 0;
      bw.col_hi = cb;
      be.col_lo = ce;
      be.col_hi = ctx->nx;
      ai.col_lo = cb;
      ai.col_hi = ce;
      dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, bw);
      CKL();
      dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, be);
      CKL();
    }
    CK(cudaEventRecord(ctx->ev_bnd, ls));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_bnd, 0));
    st = exchange(ctx, 1 - p, ctx->comm_stream);
    if (st) return st;
    dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, ai);
    CKL();
    if (e1) CK(cudaEventRecord(e1, ls));
    CK(cudaEventRecord(ctx->ev_int, ls));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_int, 0));
    st = allreduce_scalars(ctx, ctx->comm_stream);
    if (st) return st;
    finalize_kernel<<<1, 32, 0, ctx->comm_stream>>>(a, ctx->dscal + 4);
    CKL();
    CK(cudaEventRecord(ctx->ev_fin, ctx->comm_stream));
    CK(cudaStreamWaitEvent(ls, ctx->ev_fin, 0));
    return FV2D_OK;
  }
  if (tiled) {
    // the domain as tiles_x x tiles_y separate launches (the paper's NPartX x
    // NPartY tasks, P:215-220 / P:741-754); column cuts on even columns
    for (int ty = 0; ty < ctx->tiles_y; ++ty)
      for (int tx = 0; tx < ctx->tiles_x; ++tx) {
        StepArgs t = at;
        const int r_lo = (int)((long long)ty * ctx->H / ctx->tiles_y);
        const int r_hi = (int)((long long)(ty + 1) * ctx->H / ctx->tiles_y);
        t.col_lo = (int)((long long)tx * ctx->nx / ctx->tiles_x) & ~1;
        t.col_hi = tx + 1 == ctx->tiles_x ? ctx->nx : (int)((long long)(tx + 1) * ctx->nx / ctx->tiles_x) & ~1;
        set_ranges(t, r_lo, r_hi, pick_rps(ctx, t.col_hi - t.col_lo, r_hi - r_lo), 0, 0, 1);
        dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, t);
        CKL();
      }
  } else {
    dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, at);
    CKL();
  }
  if (e1) CK(cudaEventRecord(e1, ls));
  if (split) {
    // in place on the transport output; dt: the fixed dt, or read from the
    // device in adaptive mode (the finalize writes dt_{n+1} only after this pass)
    const dim3 grid = src_grid(ctx, ctx->H, ctx->nslabs);
    StepArgs b = a;
    if (tiled) b.fused_finalize = 0;
    cudaEvent_t s0 = nullptr, s1 = nullptr;
    if (e1) {  // profiling, not capturing: time the source kernel on its own
      st = prof_events(ctx, &s0, &s1, 1);
      if (st) return st;
      CK(cudaEventRecord(s0, ls));
    }
    spray_source_dt_kernel_launch(ctx, b, grid, p);
    CKL();
    if (s1) CK(cudaEventRecord(s1, ls));
  }
  if (peer_fused) {
    // nothing left: halo rows/columns were stored into the neighbours' ghost
    // cells and [smax, status] all-reduced by the pass itself
  } else if (ctx->peer) {
    // the halo rows are already in the neighbours' ghost rows (peer stores of
    // the step kernel); reduce [smax, status] over the ranks through peer memory
    st = peer_collective(ctx, ls);
    if (st) return st;
    finalize_kernel<<<1, 32, 0, ls>>>(a, ctx->dscal + 4);
    CKL();
  } else if (ctx->use_nccl) {
    st = exchange(ctx, 1 - p, ls);
    if (st) return st;
    st = allreduce_scalars(ctx, ls);
    if (st) return st;
    finalize_kernel<<<1, 32, 0, ls>>>(a, ctx->dscal + 4);
    CKL();
  } else if (!a.fused_finalize) {
    finalize_kernel<<<1, 32, 0, ls>>>(a, nullptr);
    CKL();
  }
  return FV2D_OK;
}

// Record one step per parity into CUDA graphs (FV2D_FLAG_GRAPH).
static fv2d_status capture_graphs(fv2d_ctx* ctx, int adaptive, double dt, double cfl, bool fast) {
  if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  for (int p = 0; p < 2; ++p) {
    if (ctx->graph[p]) {
      CK(cudaGraphExecDestroy(ctx->graph[p]));
      ctx->graph[p] = nullptr;
    }
    cudaGraph_t g;
    ctx->launch_stream = ctx->cap_stream;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    fv2d_status st = issue_step(ctx, p, adaptive, dt, cfl, nullptr, fast);
    cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &g);
    ctx->launch_stream = ctx->stream;
    if (st) return st;
    if (ce != cudaSuccess) return set_err(ctx, FV2D_E_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
    CK(cudaGraphInstantiate(&ctx->graph[p], g, 0));
    CK(cudaGraphDestroy(g));
  }
  ctx->graph_ready = true;
  ctx->graph_fast = fast ? 1 : 0;
  ctx->graph_adaptive = adaptive;
  ctx->graph_dt = dt;
  ctx->graph_cfl = cfl;
  ctx->graph_lam_hist = ctx->lam_hist;
  ctx->graph_dt_log = ctx->dt_log;
  return FV2D_OK;
}

static fv2d_status launch_steps(fv2d_ctx* ctx, int adaptive, double dt, double cfl, int32_t nsteps,
                                bool exact = false) {
  fv2d_status st = ensure_dt_log(ctx, ctx->steps + nsteps);
  if (st) return st;
  // dt_dev holds dt_{n} = (C*hmin)/smax(W^n) only after adaptive steps with
  // this C: the fixed-dt finalize does not refresh it
  if (nsteps > 0) {
    ctx->dt_valid = adaptive != 0;
    ctx->dt_cfl = cfl;
  }
  const bool split = ctx->cfg.system == FV2D_SPRAY;
  const bool use_graph = (ctx->cfg.flags & FV2D_FLAG_GRAPH) && !ctx->use_nccl && !ctx->peer;
  const bool fast = ctx->fast_ok && (adaptive || FV2D_FAST_FIXED) && !exact && !ctx->force_exact && !ctx->snap_used;
  for (int32_t k = 0; k < nsteps; ++k) {
    const int p = cur_parity(ctx);
    if (ctx->snap_parity == 1 - p) {  // this step writes the buffer a snapshot is reading
      CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_snap_conv, 0));
      ctx->snap_parity = -1;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->profiling) {
      st = prof_events(ctx, &e0, &e1);
      if (st) return st;
      CK(cudaEventRecord(e0, ctx->stream));
    }
    if (use_graph) {
      if (!ctx->graph_ready || ctx->graph_adaptive != adaptive || ctx->graph_dt != dt || ctx->graph_cfl != cfl ||
          ctx->graph_lam_hist != ctx->lam_hist || ctx->graph_dt_log != ctx->dt_log ||
          ctx->graph_fast != (fast ? 1 : 0)) {
        st = capture_graphs(ctx, adaptive, dt, cfl, fast);
        if (st) return st;
      }
      CK(cudaGraphLaunch(ctx->graph[p], ctx->stream));
      ctx->launches += 1;
      if (e1) CK(cudaEventRecord(e1, ctx->stream));
    } else {
      st = issue_step(ctx, p, adaptive, dt, cfl, e1, fast);
      if (st) return st;
    }
    if (ctx->fast_ok) {
      ctx->journal.push_back({adaptive, dt, cfl, fast});
      if (ctx->journal.size() >= (1u << 16)) {  // bound the journal: settle it (one sync per 65536 steps)
        unsigned long long s1;
        st = read_status(ctx, &s1);
        if (st) return st;
      }
    }
    if (split) ctx->lam_hist = std::min(3, ctx->lam_hist + 1);  // the source pass wrote lambda_{n+1}
    ctx->steps += 1;
  }
  return FV2D_OK;
}

// A latched E_NONFINITE at step k that ran the FAST pair kernel: restore the
// device state of "step k not taken" (no latched status, accumulators clear,
// step counter k, dt_dev = dt_k for an adaptive step -- the failing finalize
// logged it before overwriting dt_dev) and re-run steps k .. steps-1 from the
// journal with the exact kernels.  W^k is intact: step k wrote the other
// ping-pong buffer and every later step returned at its status check.
static fv2d_status recover_fast(fv2d_ctx* ctx, unsigned long long st, bool* redone) {
  *redone = false;
  const int code = (int)(st >> 56);
  const long long k = (long long)(st & 0x00FFFFFFFFFFFFFFull);
  const long long base = ctx->steps - (long long)ctx->journal.size();
  if (code != ST_NONFINITE || k < base || k >= ctx->steps || !ctx->journal[k - base].fast) return FV2D_OK;
  const std::vector<fv2d_ctx::StepRec> redo(ctx->journal.begin() + (k - base), ctx->journal.end());
  ctx->journal.clear();
  CK(cudaMemsetAsync(ctx->dscal, 0, 3 * sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
  ctx->hpin[0] = (unsigned long long)k;
  CK(cudaMemcpyAsync(ctx->dscal + 6, ctx->hpin, sizeof(unsigned long long), cudaMemcpyHostToDevice, ctx->stream));
  if (redo[0].adaptive)
    CK(cudaMemcpyAsync(ctx->dt_dev, ctx->dt_log + k, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->steps = k;
  ctx->recoveries += 1;
  static const bool dbg = getenv("FV2D_DEBUG_FAST") != nullptr;
  if (dbg)
    fprintf(stderr, "[fv2d] fast-path recovery: steps %lld..%lld re-run with the exact kernels\n", k,
            k + (long long)redo.size() - 1);
  for (size_t i = 0; i < redo.size();) {
    size_t j = i + 1;
    while (j < redo.size() && redo[j].adaptive == redo[i].adaptive && redo[j].dt == redo[i].dt &&
           redo[j].cfl == redo[i].cfl)
      ++j;
    fv2d_status s1 = launch_steps(ctx, redo[i].adaptive, redo[i].dt, redo[i].cfl, (int32_t)(j - i), true);
    if (s1) return s1;
    i = j;
  }
  *redone = true;
  return FV2D_OK;
}

// S:440 startup guard of the spray (SPEC "Design decisions"), before the first
// step after set_state, in the oracle's order (or_run): a
// non-admissible W^0 and (fixed dt) a CFL violation take precedence -- the
// step itself then latches them -- else reject dt*K > 0.1*min(m3/m1) with
// FV2D_E_ARG and launch nothing.  Collective over the ranks (every rank calls
// the first step after set_state); synchronous, once per set_state.
static fv2d_status spray_guard(fv2d_ctx* ctx, double dt, bool fixed) {
  if (ctx->cfg.system != FV2D_SPRAY || ctx->guard_done || ctx->steps != 0) return FV2D_OK;
  unsigned long long st;
  fv2d_status s0 = read_status(ctx, &st);
  if (s0) return s0;
  if (st) return FV2D_OK;  // latched error: the steps are no-ops and report it
  if (fixed) {
    double smax;
    unsigned long long pend;
    s0 = reduce_current(ctx, &smax, &pend);
    if (s0) return s0;
    if (pend || dt * smax > ctx->hmin) return FV2D_OK;  // the step latches E_NONFINITE / E_CFL
  }
  const StepArgs a = make_args(ctx, cur_parity(ctx));
  const dim3 grid(num_sms(ctx) * 4, 1, ctx->nslabs);
  CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
  spray_guard_kernel<<<grid, 256, 0, ctx->stream>>>(a, ctx->dscal + 0, 0.0, nullptr);
  CKL();
  unsigned long long h = 0;
  if (ctx->use_nccl || ctx->peer) {
    s0 = reduce_ranks(ctx, ctx->stream);
    if (s0) return s0;
    CK(cudaMemcpyAsync(ctx->hpin, ctx->dscal + 4, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    CK(cudaMemcpyAsync(ctx->hpin, ctx->dscal + 0, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaMemsetAsync(ctx->dscal, 0, 2 * sizeof(unsigned long long), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  h = ctx->hpin[0];
  const double rmin = h ? min_key_decode(h) : INFINITY;
  const double K = ctx->cfg.param[0];
  if ((dt * K) > (0.1 * rmin)) {
    CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
    spray_guard_kernel<<<grid, 256, 0, ctx->stream>>>(a, nullptr, rmin, ctx->dscal + 3);
    CKL();
    unsigned long long cell = ~0ull;
    s0 = d2h_words(ctx, &cell, ctx->dscal + 3, 1);
    if (s0) return s0;
    CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->err_step = 0;
    ctx->err_cell = cell == ~0ull ? -1 : (long long)cell;
    ctx->err_value = rmin;
    return set_err(ctx, FV2D_E_ARG,
                   "S:440 guard: dt*K = %.17g > 0.1*min(m3/m1) = %.17g (cell %lld); no step taken", dt * K,
                   0.1 * rmin, ctx->err_cell);
  }
  ctx->guard_done = true;
  return FV2D_OK;
}

fv2d_status fv2d_step(fv2d_ctx* ctx, double dt, int32_t nsteps) {
  if (!ctx || !(dt > 0.0) || nsteps < 0 || !std::isfinite(dt)) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  CK(cudaSetDevice(ctx->cfg.device));
  if (nsteps > 0) {
    fv2d_status st = spray_guard(ctx, dt, true);
    if (st) return st;
  }
  return launch_steps(ctx, 0, dt, 0.0, nsteps);
}

fv2d_status fv2d_step_adaptive(fv2d_ctx* ctx, double cfl, int32_t nsteps, double* dt_log) {
  if (!ctx || !(cfl > 0.0) || !(cfl <= 1.0) || nsteps < 0) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  CK(cudaSetDevice(ctx->cfg.device));
  const bool guard = ctx->cfg.system == FV2D_SPRAY && !ctx->guard_done && ctx->steps == 0 && nsteps > 0;
  if (!ctx->dt_valid || ctx->dt_cfl != cfl || guard) {
    double d, s;
    fv2d_status st = fv2d_compute_dt(ctx, cfl, &d, &s);
    if (st) return st;
    if (guard) {
      st = spray_guard(ctx, d, false);
      if (st) return st;
    }
  }
  const long long first = ctx->steps;
  fv2d_status st = launch_steps(ctx, 1, 0.0, cfl, nsteps);
  if (st) return st;
  if (dt_log && nsteps > 0) {
    unsigned long long s;
    st = read_status(ctx, &s);  // (settles FAST steps first: recover_fast rewrites the log)
    if (st) return st;
    CK(cudaMemcpyAsync(dt_log, ctx->dt_log + first, nsteps * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (s) return report(ctx, s);
  }
  return FV2D_OK;
}

// Pipelined first step of fv2d_step_host (see fv2d.h).  Bands of R rows; band
// b's AoS rows are contiguous in host memory and in the staging buffers.
static fv2d_status step_host_pipelined(fv2d_ctx* ctx, const double* host_in, double* host_out, double dt) {
  const int nv = ctx->nv, nx = ctx->nx, H = ctx->H;
  static const int nb = getenv("FV2D_HOST_BANDS") ? atoi(getenv("FV2D_HOST_BANDS")) : 64;  // tuning knob
  const int R = std::max(64, (H + nb - 1) / std::max(1, nb));
  const int B = (H + R - 1) / R;
  const size_t row_doubles = (size_t)nx * nv;
  const size_t bytes = row_doubles * H * sizeof(double);
  if (ctx->snap_parity >= 0) {
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_snap_conv, 0));
    ctx->snap_parity = -1;
  }
  fv2d_status st = ensure_staging(ctx);
  if (st) return st;
  if (!ctx->staging_out) CK(cudaMalloc(&ctx->staging_out, bytes));
  if (!ctx->h2d_stream) CK(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
  if (!ctx->d2h_stream) CK(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
  while ((int)ctx->ev_band.size() < 3 * B + 1) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ev_band.push_back(e);
  }
  cudaEvent_t* ev_in = ctx->ev_band.data();          // band b uploaded
  cudaEvent_t* ev_conv = ev_in + B;                  // band b converted into the state buffer
  cudaEvent_t* ev_out = ev_in + 2 * B;               // band b's W^{n+1} converted to AoS
  cudaEvent_t ev_start = ctx->ev_band[3 * B];
  auto lo = [&](int b) { return b * R; };
  auto hi = [&](int b) { return std::min(H, (b + 1) * R); };
  // W^0 -> parity 0, uploads in band order on the H2D stream (after prior work)
  ctx->steps = 0;
  ctx->journal.clear();
  CK(cudaEventRecord(ev_start, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->h2d_stream, ev_start, 0));
  for (int b = 0; b < B; ++b) {
    CK(cudaMemcpyAsync(ctx->staging + row_doubles * lo(b), host_in + row_doubles * lo(b),
                       row_doubles * (hi(b) - lo(b)) * sizeof(double), cudaMemcpyHostToDevice, ctx->h2d_stream));
    CK(cudaEventRecord(ev_in[b], ctx->h2d_stream));
  }
  // reset the step's device scalars as after_set_state does
  CK(cudaMemsetAsync(ctx->dscal, 0, 8 * sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->dscal + 3, 0xff, sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->done, 0, sizeof(unsigned int), ctx->stream));
  CK(cudaMemsetAsync(ctx->dt_dev, 0, sizeof(double), ctx->stream));
  ctx->lam_hist = 0;  // a new W^0: the spray source starts Newton cold (R19)
  StepArgs a = make_args(ctx, 0);
  a.adaptive = 0;
  a.dt = dt;
  a.step = 0;
  a.fused_finalize = 0;
  const bool spray = ctx->cfg.system == FV2D_SPRAY;  // split source pass per band after its transport
  StepArgs at = a;
  at.no_smax = 1;
  StepArgs hf = make_args(ctx, 1);  // halo targets of parity 0 (as after_set_state)
  hf.slab[0].in = row_ptr(ctx, 0, 0, 0);
  auto convert_in = [&](int b) -> fv2d_status {
    CK(cudaStreamWaitEvent(ctx->stream, ev_in[b], 0));
    aos_to_dev_kernel<<<num_sms(ctx) * 2, 256, 0, ctx->stream>>>(ctx->staging + row_doubles * lo(b), row_ptr(ctx, 0, 0, lo(b)),
                                                        nv, nx, hi(b) - lo(b), ctx->pitch, ctx->rs);
    CKL();
    if (ctx->xg) {  // this band's ghost columns (wall mirror / periodic own columns)
      StepArgs hc = hf;
      hc.src_row_lo = lo(b);
      hc.src_row_hi = hi(b);
      fill_halo_cols_kernel<<<(hi(b) - lo(b) + 127) / 128, 128, 0, ctx->stream>>>(hc, nv);
      CKL();
    }
    CK(cudaEventRecord(ev_conv[b], ctx->stream));
    return FV2D_OK;
  };
  auto step_band = [&](int b) -> fv2d_status {
    StepArgs t = at;
    set_ranges(t, lo(b), hi(b), pick_rps(ctx, nx, hi(b) - lo(b)), 0, 0, 1);
    dispatch<LaunchStep>(ctx->cfg.system, (const fv2d_ctx*)ctx, t);
    CKL();
    if (spray) {
      StepArgs sb = a;
      sb.src_row_lo = lo(b);
      sb.src_row_hi = hi(b);
      spray_source_dt_kernel_launch(ctx, sb, src_grid(ctx, hi(b) - lo(b), 1), 0);
      CKL();
    }
    dev_to_aos_kernel<<<num_sms(ctx) * 2, 256, 0, ctx->stream>>>(row_ptr(ctx, 0, 1, lo(b)), ctx->staging_out + row_doubles * lo(b),
                                                        nv, nx, hi(b) - lo(b), ctx->pitch, ctx->rs);
    CKL();
    CK(cudaEventRecord(ev_out[b], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->d2h_stream, ev_out[b], 0));
    CK(cudaMemcpyAsync(host_out + row_doubles * lo(b), ctx->staging_out + row_doubles * lo(b),
                       row_doubles * (hi(b) - lo(b)) * sizeof(double), cudaMemcpyDeviceToHost, ctx->d2h_stream));
    return FV2D_OK;
  };
  // interior bands as soon as their neighbours are resident; the boundary
  // bands (0 and B-1, which read the ghost rows) after the halo fill
  for (int b = 0; b < B; ++b) {
    st = convert_in(b);
    if (st) return st;
    if (b >= 2 && b - 1 < B - 1) {
      st = step_band(b - 1);
      if (st) return st;
    }
  }
  fill_halo_kernel<<<dim3((nx + 127) / 128, 1, 1), 128, 0, ctx->stream>>>(hf, nv);
  CKL();
  if (B > 1) {
    st = step_band(B - 1);
    if (st) return st;
  }
  st = step_band(0);
  if (st) return st;
  finalize_kernel<<<1, 32, 0, ctx->stream>>>(a, nullptr);
  CKL();
  CK(cudaEventRecord(ev_start, ctx->d2h_stream));
  CK(cudaStreamWaitEvent(ctx->stream, ev_start, 0));
  ctx->has_state = true;
  ctx->dt_valid = false;
  ctx->lam_hist = spray ? 1 : 0;  // lambda_1 of every cell is in lam_buf[1 % 3]
  ctx->err.clear();
  ctx->err_step = ctx->err_cell = -1;
  ctx->steps = 1;
  return FV2D_OK;
}

fv2d_status fv2d_step_host(fv2d_ctx* ctx, const double* host_in, double* host_out, fv2d_layout layout, double dt,
                           int32_t nsteps) {
  if (!ctx || !host_in || !host_out || (layout != FV2D_AOS && layout != FV2D_SOA) || !(dt > 0.0) || nsteps < 0 ||
      !std::isfinite(dt))
    return FV2D_E_ARG;
  if (ctx->peer && !ctx->peer_connected) return set_err(ctx, FV2D_E_STATE, "peer halo: call fv2d_peer_connect first");
  CK(cudaSetDevice(ctx->cfg.device));
  // exact kernels throughout: the output is written as the steps complete, so
  // there is no later point at which recover_fast could re-run one
  struct ExactGuard {
    fv2d_ctx* c;
    ~ExactGuard() { c->force_exact = false; }
  } exact_guard{ctx};
  ctx->force_exact = true;
  // the spray's first step needs all of W^0 on the device before it starts
  // (the S:440 guard), so only transport systems pipeline the upload
  const bool pipelined = layout == FV2D_AOS && nsteps >= 1 && ctx->cfg.nranks == 1 && ctx->nslabs == 1 &&
                         ctx->cfg.system != FV2D_SPRAY &&
                         !ctx->use_nccl && !ctx->peer &&
                         !(ctx->cfg.flags & FV2D_FLAG_NAIVE) && ctx->H >= 128;
  fv2d_status st;
  if (pipelined) {
    st = ensure_dt_log(ctx, nsteps);
    if (st) return st;
    st = step_host_pipelined(ctx, host_in, host_out, dt);
    if (st) return st;
    if (nsteps > 1) {
      st = launch_steps(ctx, 0, dt, 0.0, nsteps - 1);
      if (st) return st;
    } else {
      unsigned long long s0;
      st = read_status(ctx, &s0);  // also waits for the last D2H band
      if (st) return st;
      if (s0 == 0) return FV2D_OK;
      // the step failed: host_out must hold W^0 (the already copied bands hold W^1)
    }
  } else {
    st = fv2d_set_state(ctx, host_in, layout);
    if (st) return st;
    st = fv2d_step(ctx, dt, nsteps);
    if (st == FV2D_E_ARG) {  // the S:440 guard: no step taken, host_out receives W^0
      const std::string msg = ctx->err;
      const long long cell = ctx->err_cell;
      const double val = ctx->err_value;
      fv2d_status g = fv2d_get_state(ctx, host_out, layout);
      if (g) return g;
      ctx->err = msg;
      ctx->err_step = 0;
      ctx->err_cell = cell;
      ctx->err_value = val;
      return FV2D_E_ARG;
    }
    if (st) return st;
  }
  return fv2d_get_state(ctx, host_out, layout);
}

fv2d_status fv2d_apply_source(fv2d_ctx* ctx, double dt) {
  if (!ctx || !(dt > 0.0)) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  if (ctx->cfg.system != FV2D_SPRAY) return FV2D_OK;  // S = 0
  CK(cudaSetDevice(ctx->cfg.device));
  if (ctx->snap_parity >= 0) {  // in place: a snapshot may still be converting this buffer
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_snap_conv, 0));
    ctx->snap_parity = -1;
  }
  const int p = cur_parity(ctx);
  // in place on parity p: halo targets are the ghost buffers of parity p
  StepArgs b = make_args(ctx, 1 - p);
  for (int s = 0; s < ctx->nslabs; ++s) b.slab[s].out = row_ptr(ctx, s, p, 0);
  b.step = ctx->steps;
  // the multipliers of the current state W^n are in lam_buf[n % 3]: warm start
  // from them, no extrapolation, write back in place (history broken)
  b.lam_inplace = 1;
  spray_source_kernel<<<src_grid(ctx, ctx->H, ctx->nslabs), kSrcThreads, 0, ctx->stream>>>(b, dt, 0);
  CKL();
  ctx->lam_hist = 1;
  fv2d_status st = exchange(ctx, p);
  if (st) return st;
  if (ctx->peer) {
    st = peer_collective(ctx, ctx->stream);  // halo rows of all ranks in place + global status
    if (st) return st;
    CK(cudaMemsetAsync(ctx->dscal + 1, 0, sizeof(unsigned long long), ctx->stream));
    promote_pending_kernel<<<1, 32, 0, ctx->stream>>>(ctx->dscal + 5, ctx->dscal + 2);
  } else {
    promote_pending_kernel<<<1, 32, 0, ctx->stream>>>(ctx->dscal + 1, ctx->dscal + 2);
  }
  CKL();
  ctx->dt_valid = false;
  return FV2D_OK;
}

fv2d_status fv2d_synchronize(fv2d_ctx* ctx) {
  if (!ctx) return FV2D_E_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  unsigned long long st;
  fv2d_status s0 = read_status(ctx, &st);
  if (s0) return s0;
  return report(ctx, st);
}

fv2d_status fv2d_device_state(fv2d_ctx* ctx, int32_t slab, double** d_ptr, int64_t* pitch, int64_t* row_stride,
                              int32_t* ny_slab) {
  if (!ctx || slab < 0 || slab >= ctx->nslabs) return FV2D_E_ARG;
  if (!ctx->journal.empty()) {  // settle the FAST steps first (recover_fast may re-run some)
    CK(cudaSetDevice(ctx->cfg.device));
    unsigned long long st;
    fv2d_status s0 = read_status(ctx, &st);
    if (s0) return s0;
  }
  if (d_ptr) *d_ptr = row_ptr(ctx, slab, cur_parity(ctx), 0);
  if (pitch) *pitch = ctx->pitch;
  if (row_stride) *row_stride = ctx->rs;
  if (ny_slab) *ny_slab = ctx->H;
  return FV2D_OK;
}

fv2d_status fv2d_last_error(fv2d_ctx* ctx, char* buf, size_t n, int64_t* step, int64_t* cell, double* value) {
  if (!ctx) return FV2D_E_ARG;
  unsigned long long st = 0;
  if (ctx->has_state && read_status(ctx, &st) == FV2D_OK && st) {
    report(ctx, st);
    diagnose(ctx, st);
    unsigned long long bc = ~0ull;
    if (d2h_words(ctx, &bc, ctx->dscal + 3, 1) != FV2D_OK) bc = ~0ull;
    ctx->err_cell = bc == ~0ull ? -1 : (long long)bc;
  }
  if (buf && n) {
    snprintf(buf, n, "%s", ctx->err.c_str());
  }
  if (step) *step = ctx->err_step;
  if (cell) *cell = ctx->err_cell;
  if (value) *value = ctx->err_value;
  return FV2D_OK;
}

fv2d_status fv2d_set_profiling(fv2d_ctx* ctx, int32_t enable) {
  if (!ctx) return FV2D_E_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  fv2d_status st = prof_flush(ctx);
  if (st) return st;
  ctx->profiling = enable != 0;
  ctx->prof_ms = 0.0;
  ctx->prof_n = 0;
  ctx->prof_src_ms = 0.0;
  ctx->prof_src_n = 0;
  return FV2D_OK;
}

fv2d_status fv2d_snapshot(fv2d_ctx* ctx, double* host, fv2d_layout layout) {
  if (!ctx || !host || (layout != FV2D_AOS && layout != FV2D_SOA)) return FV2D_E_ARG;
  if (!ctx->has_state) return set_err(ctx, FV2D_E_STATE, "no state set");
  CK(cudaSetDevice(ctx->cfg.device));
  if (!ctx->journal.empty()) {  // settle the FAST steps; snapshots then run with exact kernels only
    unsigned long long st;
    fv2d_status s0 = read_status(ctx, &st);
    if (s0) return s0;
  }
  ctx->snap_used = true;
  const int nv = ctx->nv, nx = ctx->nx, H = ctx->H;
  const size_t bytes = (size_t)nv * nx * H * ctx->nslabs * sizeof(double);
  if (!ctx->out_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->out_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_snap_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_snap_conv, cudaEventDisableTiming));
    CK(cudaMallocAsync(&ctx->snap_buf, bytes, ctx->stream));
  }
  if (ctx->snap_parity >= 0) {  // one conversion in flight at a time
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_snap_conv, 0));
    ctx->snap_parity = -1;
  }
  const int p = cur_parity(ctx);
  // "gather": convert W^k into the staging buffer on the side stream, after the
  // work already queued on the main stream
  CK(cudaEventRecord(ctx->ev_snap_start, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->out_stream, ctx->ev_snap_start, 0));
  for (int s = 0; s < ctx->nslabs; ++s) {
    if (layout == FV2D_AOS) {
      dev_to_aos_kernel<<<num_sms(ctx) * 4, 256, 0, ctx->out_stream>>>(row_ptr(ctx, s, p, 0),
                                                              ctx->snap_buf + (size_t)s * H * nx * nv, nv, nx, H,
                                                              ctx->pitch, ctx->rs);
      CKL();
    } else {
      const long long nyl = (long long)H * ctx->nslabs;
      for (int v = 0; v < nv; ++v)
        CK(cudaMemcpy2DAsync(ctx->snap_buf + (size_t)v * nyl * nx + (size_t)s * H * nx, nx * sizeof(double),
                             row_ptr(ctx, s, p, 0) + v * ctx->pitch, ctx->rs * sizeof(double), nx * sizeof(double),
                             H, cudaMemcpyDeviceToDevice, ctx->out_stream));
    }
  }
  CK(cudaEventRecord(ctx->ev_snap_conv, ctx->out_stream));
  ctx->snap_parity = p;
  // "outputToDisk" leg: device staging -> host, overlapped with later steps
  CK(cudaMemcpyAsync(host, ctx->snap_buf, bytes, cudaMemcpyDeviceToHost, ctx->out_stream));
  return FV2D_OK;
}

fv2d_status fv2d_snapshot_wait(fv2d_ctx* ctx) {
  if (!ctx) return FV2D_E_ARG;
  if (ctx->out_stream) CK(cudaStreamSynchronize(ctx->out_stream));
  return FV2D_OK;
}

fv2d_status fv2d_host_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return FV2D_E_ARG;
  return cudaHostAlloc(ptr, bytes, cudaHostAllocDefault) == cudaSuccess ? FV2D_OK : FV2D_E_CUDA;
}

fv2d_status fv2d_host_free(void* ptr) {
  if (!ptr) return FV2D_OK;
  return cudaFreeHost(ptr) == cudaSuccess ? FV2D_OK : FV2D_E_CUDA;
}

// Ranks of the south, north, west, east neighbour blocks (-1: none, i.e. a
// non-periodic global boundary; W/E only for 2-D rank blocks).
static void peer_neighbours(const fv2d_ctx* ctx, int nb[4]) {
  const bool pery = ctx->cfg.bc_y == FV2D_BC_PERIODIC, perx = ctx->cfg.bc_x == FV2D_BC_PERIODIC;
  const int x = ctx->rx, y = ctx->ry;
  nb[0] = (y > 0 || pery) ? rank_at(ctx, x, y - 1) : -1;
  nb[1] = (y < ctx->py - 1 || pery) ? rank_at(ctx, x, y + 1) : -1;
  nb[2] = ctx->xg && (x > 0 || perx) ? rank_at(ctx, x - 1, y) : -1;
  nb[3] = ctx->xg && (x < ctx->px - 1 || perx) ? rank_at(ctx, x + 1, y) : -1;
}

static fv2d_status peer_finish(fv2d_ctx* ctx) {
  ctx->pa.nranks = ctx->cfg.nranks;
  ctx->pa.me = ctx->cfg.rank;
  ctx->pa.sync[ctx->cfg.rank] = ctx->sync;
  ctx->peer_connected = true;
  return FV2D_OK;
}

fv2d_status fv2d_peer_export(fv2d_ctx* ctx, uint8_t* out) {
  if (!ctx || !out || !ctx->peer) return FV2D_E_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  cudaIpcMemHandle_t h[3];
  CK(cudaIpcGetMemHandle(&h[0], ctx->buf[0][0]));
  CK(cudaIpcGetMemHandle(&h[1], ctx->buf[0][1]));
  CK(cudaIpcGetMemHandle(&h[2], ctx->sync));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  memcpy(out, h, sizeof h);
  return FV2D_OK;
}

fv2d_status fv2d_peer_connect(fv2d_ctx* ctx, const uint8_t* all) {
  if (!ctx || !all || !ctx->peer) return FV2D_E_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  const int P = ctx->cfg.nranks, r = ctx->cfg.rank;
  // every handle opened at most once (a rank can be several neighbours);
  // this rank's own buffers are used directly
  std::vector<void*> opened((size_t)P * 3, nullptr);
  auto get = [&](int rank, int k, void** ptr) -> fv2d_status {
    if (rank == r) {
      *ptr = k == 2 ? (void*)ctx->sync : (void*)ctx->buf[0][k];
      return FV2D_OK;
    }
    void*& slot = opened[(size_t)rank * 3 + k];
    if (!slot) {
      cudaIpcMemHandle_t h;
      memcpy(&h, all + (size_t)rank * FV2D_PEER_HANDLE_BYTES + (size_t)k * 64, 64);
      CK(cudaIpcOpenMemHandle(&slot, h, cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_opened.push_back(slot);
    }
    *ptr = slot;
    return FV2D_OK;
  };
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    void* p = nullptr;
    fv2d_status st = get(q, 2, &p);
    if (st) return st;
    ctx->pa.sync[q] = (PeerSync*)p;
  }
  int nb[4];
  peer_neighbours(ctx, nb);
  double** tgt[4] = {ctx->peer_buf_s, ctx->peer_buf_n, ctx->peer_buf_w, ctx->peer_buf_e};
  for (int d = 0; d < 4; ++d)
    for (int k = 0; k < 2; ++k) {
      void* p = nullptr;
      if (nb[d] >= 0) {
        fv2d_status st = get(nb[d], k, &p);
        if (st) return st;
      }
      tgt[d][k] = (double*)p;
    }
  return peer_finish(ctx);
}

fv2d_status fv2d_peer_connect_local(fv2d_ctx* ctx, fv2d_ctx* const* group) {
  if (!ctx || !group || !ctx->peer) return FV2D_E_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  const int P = ctx->cfg.nranks;
  for (int q = 0; q < P; ++q) {
    if (!group[q] || group[q]->cfg.rank != q || group[q]->cfg.nranks != P || !group[q]->peer ||
        group[q]->px != ctx->px || group[q]->xg != ctx->xg)
      return FV2D_E_ARG;
    if (group[q]->cfg.device != ctx->cfg.device) {
      cudaError_t e = cudaDeviceEnablePeerAccess(group[q]->cfg.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return set_err(ctx, FV2D_E_CUDA, "peer access %d->%d: %s", ctx->cfg.device, group[q]->cfg.device,
                       cudaGetErrorString(e));
      cudaGetLastError();
    }
    ctx->pa.sync[q] = group[q]->sync;
  }
  int nb[4];
  peer_neighbours(ctx, nb);
  double** tgt[4] = {ctx->peer_buf_s, ctx->peer_buf_n, ctx->peer_buf_w, ctx->peer_buf_e};
  for (int d = 0; d < 4; ++d)
    for (int k = 0; k < 2; ++k) tgt[d][k] = nb[d] >= 0 ? group[nb[d]]->buf[0][k] : nullptr;
  return peer_finish(ctx);
}

fv2d_status fv2d_get_stats(fv2d_ctx* ctx, fv2d_stats* out) {
  if (!ctx || !out) return FV2D_E_ARG;
  fv2d_status st = prof_flush(ctx);
  if (st) return st;
  out->step_kernel_ms = ctx->prof_ms;
  out->step_kernels_timed = ctx->prof_n;
  out->source_kernel_ms = ctx->prof_src_ms;
  out->source_kernels_timed = ctx->prof_src_n;
  out->steps = ctx->steps;
  out->kernel_launches = ctx->launches;
  out->sms = ctx->sms;
  out->resident_ctas = ctx->slots;
  out->strip_rows = ctx->rps;
  out->reserved0 = 0;
  unsigned long long ni = 0, dbits = 0;
  if (ctx->newton) d2h_words(ctx, &ni, ctx->newton, 1);
  out->newton_iters = (int64_t)ni;
  if (ctx->dt_dev) d2h_words(ctx, &dbits, reinterpret_cast<const unsigned long long*>(ctx->dt_dev), 1);
  double d;
  memcpy(&d, &dbits, sizeof d);
  out->dt = d;
  return FV2D_OK;
}

}  // extern "C"
