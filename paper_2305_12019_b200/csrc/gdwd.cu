// gdwd_b200: context, one-time setup, the device-resident sGS-ADMM loop
// and the C ABI (include/gdwd_b200.h).
//
// The loop is the reference's sgs_admm_solve (solver.py:392-602) with every
// vector resident in HBM; the host only launches work and, every
// `poll_every` iterations, reads the device stop flag.  DIRECT and SMW2
// iteration bodies are captured once into a CUDA graph and replayed; the
// ITERATIVE body is host-driven because PSQMR's step count is data
// dependent (one 4-byte flag read per PSQMR step).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing unless a tool is attached
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <memory>
#include <cstdlib>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/gdwd_b200.h"
#include "common.cuh"
#include "gram.cuh"
#include "solver_ops.cuh"
#include "spops.cuh"
#include "select.cuh"
#include "persist.cuh"
#include "persist3.cuh"
#include "synth.cuh"
#include "zft.cuh"
#include "zops.cuh"

using namespace gdwd;

// ---------------------------------------------------------------------------
// NCCL, bound at run time (dlopen) so the library has no link-time NCCL
// dependency; the same libnccl.so.2 torch.distributed loads.
// ---------------------------------------------------------------------------
namespace nccl {
typedef struct { char internal[128]; } UniqueId;
typedef void* Comm;
typedef int Result;
enum { Float64 = 8, Sum = 0 };
struct Api {
  bool ok = false;
  Result (*GetUniqueId)(UniqueId*) = nullptr;
  Result (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  Result (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*CommDestroy)(Comm) = nullptr;
  const char* (*GetErrorString)(Result) = nullptr;
};
static Api& api() {
  static Api a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  const char* env = getenv("GDWD_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names)
    if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;  // local: a later `import torch` must bind its own NCCL
  if (!h) return a;
  a.GetUniqueId = (Result(*)(UniqueId*))dlsym(h, "ncclGetUniqueId");
  a.CommInitRank = (Result(*)(Comm*, int, UniqueId, int))dlsym(h, "ncclCommInitRank");
  a.AllReduce = (Result(*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))dlsym(h, "ncclAllReduce");
  a.CommDestroy = (Result(*)(Comm))dlsym(h, "ncclCommDestroy");
  a.GetErrorString = (const char* (*)(Result))dlsym(h, "ncclGetErrorString");
  a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy;
  return a;
}
}  // namespace nccl

namespace {

constexpr int NUM_SMS = 148;
// feature-blocked sliced ELL (sp_ztmv_fb_kernel): block width, parts (CTAs)
// and slice rows per lane in flight
#ifndef FB_COLS_V
#define FB_COLS_V 8192
#endif
#ifndef FB_PARTS_PER_SM
#define FB_PARTS_PER_SM 2
#endif
constexpr int FB_COLS = FB_COLS_V;
constexpr int FB_PARTS = FB_PARTS_PER_SM * NUM_SMS;
constexpr size_t FB_SMEM_MAX = 100 * 1024;
#ifndef FB_H
#define FB_H 1
#endif
#ifndef FB_U
#define FB_U 4
#endif

// Device memory comes from the device's default stream-ordered pool, whose
// release threshold is raised at context creation: freed blocks stay
// reserved, so repeated solves and fresh contexts (e2e: a new problem each
// call) reuse memory without driver mapping calls.  The allocation is
// complete when dmalloc returns (usable from any stream); frees are ordered
// on the context's stream after the work that uses the block.
static cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t st) {
  // + 512 B of slack: pool blocks are packed, and vector loads near the end
  // of a ragged row may be issued speculatively
  cudaError_t e = cudaMallocAsync(p, std::max<size_t>(bytes, 16) + 512, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}
static void dfree(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}
static void keep_pool_reserved(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;  // the owning context's stream
  cudaError_t ensure(size_t cnt) {
    if (cnt <= n && p) return cudaSuccess;
    dfree(p, st);
    p = nullptr;
    n = 0;
    cudaError_t e = dmalloc((void**)&p, std::max<size_t>(cnt, 1) * sizeof(double), st);
    if (e == cudaSuccess) n = cnt;
    return e;
  }
  void release() {
    dfree(p, st);
    p = nullptr;
    n = 0;
  }
};

// Grids are sized from the occupancy calculator: one full wave of resident
// CTAs (`slots` = blocks/SM x 148), work split evenly, so there is no tail
// wave and no per-launch CTA churn.
ZmvGeom zmv_geom(int64_t rows, int64_t cols, int slots) {
  ZmvGeom g;
  g.tiles = (int)((cols + ZMV_TILE - 1) / ZMV_TILE);
  int64_t segs = std::max<int64_t>(1, slots / g.tiles);
  // at least 32 rows per segment: short matrices (c1: 1000 samples) are
  // bound by the last CTA's in-order sum over segment partials, not by the
  // stream (measured: 125 -> 31 segments, c1 8.8k -> 10.5k it/s)
  segs = std::min<int64_t>(segs, std::max<int64_t>(1, rows / 32));
  g.seg_len = std::max<int64_t>(1, (rows + segs - 1) / segs);
  g.segs = (int)std::max<int64_t>(1, (rows + g.seg_len - 1) / g.seg_len);
  g.ldp = (cols + 1) / 2 * 2;
  return g;
}

ZtGeom zt_geom(int64_t rows, int64_t ld, int slots) {
  ZtGeom g;
  int64_t cw = std::min<int64_t>((ld + 63) / 64 * 64, ZT_CW);
  // short matrices: split rows into more chunks until the grid can fill the GPU
  while (cw > 512 && ((ld + cw - 1) / cw) * ((rows + 7) / 8) < NUM_SMS * 4) cw = (cw / 2 + 63) / 64 * 64;
  g.cw = (int)cw;
  g.chunks = (int)((ld + cw - 1) / cw);
  int64_t ranges = std::max<int64_t>(1, slots / g.chunks);
  ranges = std::min<int64_t>(ranges, std::max<int64_t>(1, (rows + 7) / 8));
  g.ranges = (int)ranges;
  return g;
}

template <class K>
int slots_for(K kernel, int threads, size_t smem) {
  static std::map<std::pair<const void*, size_t>, int> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair((const void*)kernel, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess || nb < 1) nb = 1;
  const int s = nb * NUM_SMS;
  cache[key] = s;
  return s;
}

int vm_grid(int64_t len) {
  int64_t b = (len + VM_THREADS - 1) / VM_THREADS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, NUM_SMS * 4));
}

}  // namespace

struct gdwd_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  // data
  int64_t n = 0, d = 0, ldz = 0;
  bool has_dense = false;
  double* Zs = nullptr;
  bool has_problem = false;
  double C = 0, q = 0, zscale = 0, yty = 0;
  double fro2 = -1.0;  // ||Z~||_F^2 (device reduction at upload)
  // overlapped dense upload (pinned source): row chunks on a copy stream,
  // the SMW Gram block-rows on a second stream as the chunks land
  static constexpr int UP_BLOCK = 128;  // samples per block (two Cholesky leaves)
  static constexpr int UP_MAXB = 24;    // n <= 2500 -> at most 20 blocks
  cudaStream_t cst = nullptr, gst = nullptr, fst = nullptr, sst = nullptr, ast = nullptr;
  cudaEvent_t up_ev[UP_MAXB] = {}, gr_ev[UP_MAXB] = {}, gram_ev = nullptr, st_ev = nullptr, pf_ev = nullptr;
  void* aux = nullptr;        // pooled stream / scalars / events (CtxAux)
  void* up_aux = nullptr;     // pooled streams / events (UploadAux)
  DevBuf pfw;                 // G | L^{-1} | scratch (n x ld each) of the bordered factorisation
  int64_t dg_gen = -1;        // zs_gen whose d x d Gram Z~ Z~^T (in fac, DIRECT layout) was summed during the upload
  int64_t pf_gen = -1;        // zs_gen whose G^{-1} (fac) was formed during the upload ...
  double pf_mu2 = 0.0;        // ... for this mu^2
  double hint_mu = 1.0;       // mu the next upload's speculative factor is built for
  int hint_backend = GDWD_BACKEND_AUTO;
  bool up_pending = false;    // copies of the current Zs may be in flight
  int64_t zs_gen = 0;         // bumped whenever the dense Z~ (Zs) changes
  int64_t k_gen = -1;         // zs_gen whose Gram K = Z~ Z~^T (kmat) was formed at upload
  bool fro2_pending = false;  // fro2_h holds the value once st is synchronized
  double* fro2_h = nullptr;   // pinned
  double* fro2_d = nullptr;
  DevBuf gram_ws;             // split-K workspace of the upload's chunked Gram
  double* pin[2] = {nullptr, nullptr};  // pinned staging for uploads
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  size_t pin_bytes = 0;
  // sparse Z~: CSC by sample (Z^T w) and CSR by feature (Z t), int32 indices
  bool has_sparse = false;
  int64_t nnz = 0;
  int64_t *csc_ptr = nullptr, *csr_ptr = nullptr;
  int *csc_idx = nullptr, *csr_idx = nullptr;
  double *csc_val = nullptr, *csr_val = nullptr;
  // feature-blocked CSC (spops.cuh FbView) for Z~^T w
  int* fb_ptr = nullptr;
  unsigned short *fb_perm = nullptr, *fb_cnt = nullptr, *fb_idx = nullptr;
  double* fb_val = nullptr;
  int fb_nb = 0, fb_parts = 0, fb_S = 0, fb_Q = 0;
  int64_t fb_entries = 0;  // padded entries
  bool sp_blocked = getenv("GDWD_SP_BLOCKED") ? atoi(getenv("GDWD_SP_BLOCKED")) != 0 : true;
  // sample-blocked sliced ELL for Z~ t (spops.cuh SbView)
  double* sb_val = nullptr;
  unsigned short* sb_idx = nullptr;
  int64_t* sb_base = nullptr;
  int *sb_h = nullptr, *sb_perm = nullptr, *sb_chunk = nullptr;
  int sb_nb = 0, sb_nslpb = 0;
  int64_t sb_entries = 0;
  DevBuf sb_part;  // [nb][d][R] partials
  bool sp_sb = getenv("GDWD_SP_SB") ? atoi(getenv("GDWD_SP_SB")) != 0 : true;
  DevBuf tbuf;  // materialised Z t inputs (2 x n)
  DevBuf y, e, wl;
  // scratch
  DevBuf part, npart, tpart;
  unsigned* tickets = nullptr;
  size_t ntickets = 0;
  Scratch scr{};
  // solver buffers
  DevBuf nvec, mvec, tabs, histb, fac, facw, colsq, kmat;
  int64_t ldm = 0, fac_rows = 0;
  int fac_kind = 0;
  double fac_mu2 = -1;
  uint64_t data_gen = 0, fac_gen = (uint64_t)-1;
  int* dinfo = nullptr;
  Scal* S = nullptr;
  Scal* Sh = nullptr;  // pinned mirror
  Dev D{};
  int64_t hist_rows = 0;
  std::vector<double> ps_per_iter;
  int last_kind = 0;
  // solve session (gdwd_solve_begin / _iterate / _end)
  bool in_solve = false;
  int kind = 0, poll = 16, max_iter = 0, max_steps = 50, k_host = 0, psqmr_total = 0;
  bool use_sgs = true, stopped = false, gram = false, persistent = false;
  bool iter_gram = false;  // ITERATIVE with the d x d Gram operator (gdmat)
  bool ft = false;         // X-space loop with the fused tail pass (zft.cuh)
  // persistent launch, configured once per solve (solve_begin); a launch made
  // by gdwd_time_iterations is settled (stop flag read back) after its end event
  const void* pk_kfn = nullptr;
  size_t pk_smem = 0;
  bool pk_pending = false, pk_defer = false;
  int pk_kend = 0;
  unsigned long long* pk_ts = nullptr;
  size_t pk_tsn = 0;
  unsigned long long* ft_ts = nullptr;  // GDWD_FT_TIMING stamps (diagnostics)
  bool ps_graph = false;   // ITERATIVE body captured with device-resident PSQMR (WHILE nodes)
  cudaStream_t cap_st = nullptr;  // capture-to-graph stream for conditional bodies
  int64_t ps_step_nodes = 0;      // kernels per device-resident PSQMR step (launch accounting)
  bool hist_ps_dev = false;       // the last solve's history holds device-recorded PSQMR steps
  DevBuf gdmat;
  int64_t ldg = 0;
  int fac_iter_gram = 0;
  DevBuf pk_part, gkmat;
  // proximal fallback (subsolvers.py:159-256)
  bool prox = false;
  int ell = 10;
  std::vector<double> lz_start;  // Lanczos start vector (numpy default_rng(seed))
  DevBuf pxbuf;                  // V [L][d] | coefs | sa, hp, tmp, zaz, wold
  // sample sharding: 0 none, 1 NCCL, 2 host all-reduce callback
  int comm_mode = 0, nranks = 1, rank = 0;
  int64_t n_global = 0;
  nccl::Comm comm = nullptr;
  gdwd_allreduce_cb host_ar = nullptr;
  void* host_ar_user = nullptr;
  DevBuf bundle;
  double* bundle_h = nullptr;  // pinned, host all-reduce mode
  size_t bundle_h_n = 0;
  int comm_err = 0;
  cudaGraphExec_t gexec = nullptr;
  int64_t body_nodes = 0;
  cudaEvent_t ev_begin = nullptr, ev_loop = nullptr, ev_end = nullptr;
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  int* poll_flag = nullptr;  // pinned [2]
  int poll_slot = 0, poll_pending = 0;
  double eps_c = 0, setup_ms = 0;
  // counters and per-kernel profile
  int64_t launches = 0;
  bool prof = false;
  struct ProfRec { const char* tag; cudaEvent_t a, b; };
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::map<std::string, std::pair<int64_t, double>> prof_acc;
  cudaEvent_t take_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
};

static void end_session(gdwd_ctx* ctx);

static int set_err(gdwd_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

static MatView zview(const gdwd_ctx* c) { return MatView{c->has_dense ? c->Zs : nullptr, c->n, c->d, c->ldz}; }

#define RC(call)                           \
  do {                                     \
    int rc_ = (call);                      \
    if (rc_ != GDWD_OK) return rc_;        \
  } while (0)

#define CK(call)                                                                 \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return set_err(ctx, GDWD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
struct Launch {  // counts launches; with profiling on, brackets the launch with events
  gdwd_ctx* c;
  const char* tag;
  cudaEvent_t a = nullptr;
  Launch(gdwd_ctx* c_, const char* t) : c(c_), tag(t) {
    nvtxRangePushA(t);  // host-side launch range, named like the profile tags
    c->launches++;
    if (c->prof) {
      a = c->take_event();
      cudaEventRecord(a, c->st);
    }
  }
  ~Launch() {
    static const bool dbg = getenv("GDWD_DEBUG_LAUNCH") != nullptr;
    if (dbg) {
      const cudaError_t e = cudaPeekAtLastError();
      if (e != cudaSuccess) fprintf(stderr, "gdwd launch %s: %s\n", tag, cudaGetErrorString(e));
    }
    if (c->prof) {
      cudaEvent_t b = c->take_event();
      cudaEventRecord(b, c->st);
      c->prof_pending.push_back({tag, a, b});
    }
    nvtxRangePop();
  }
};
// NVTX range over a host-side phase (upload, setup, iteration loop, download)
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

static int sp_grid(int64_t work_threads, int cap) {
  int64_t b = (work_threads + SP_THREADS - 1) / SP_THREADS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

// All-reduce (sum) of `count` doubles at dev across the sample shards.
static void allreduce(gdwd_ctx* ctx, double* dev, int64_t count) {
  if (ctx->comm_mode == 1) {
    Launch L(ctx, "nccl_allreduce");
    L.c->launches--;  // not one of our kernels
    const nccl::Result r = nccl::api().AllReduce(dev, dev, (size_t)count, nccl::Float64, nccl::Sum, ctx->comm, ctx->st);
    if (r != 0 && !ctx->comm_err) ctx->comm_err = r;
  } else if (ctx->comm_mode == 2) {
    if ((size_t)count > ctx->bundle_h_n) {
      if (ctx->bundle_h) cudaFreeHost(ctx->bundle_h);
      cudaMallocHost(&ctx->bundle_h, (size_t)count * sizeof(double));
      ctx->bundle_h_n = (size_t)count;
    }
    cudaMemcpyAsync(ctx->bundle_h, dev, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->st);
    cudaStreamSynchronize(ctx->st);
    if (ctx->host_ar(ctx->host_ar_user, ctx->bundle_h, count) != 0 && !ctx->comm_err) ctx->comm_err = -1;
    cudaMemcpyAsync(dev, ctx->bundle_h, count * sizeof(double), cudaMemcpyHostToDevice, ctx->st);
  }
}

static bool sharded(const gdwd_ctx* ctx) { return ctx->comm_mode != 0; }
static Scratch scr_bundle(const gdwd_ctx* ctx) {
  Scratch s = ctx->scr;
  s.bundle = ctx->bundle.p;
  return s;
}

// X.a == nullptr marks the context's sparse Z~ (CSR/CSC pair).  A product
// with Z~ over sharded samples runs as: local partial kernel -> all-reduce of
// [Z~_local t | n-sums] -> epilogue kernel on every rank.
template <class Op>
static void run_zmv(gdwd_ctx* ctx, const Op& op, MatView X, const char* tag = "zmv") {
  const bool sh = sharded(ctx);
  const Scratch sc = sh ? scr_bundle(ctx) : ctx->scr;
  if (!X.a) {
    const int g1 = sp_grid(ctx->n, NUM_SMS * 4);
    {
      Launch L(ctx, "sp_prep");
      sp_prep_kernel<Op><<<g1, SP_THREADS, 0, ctx->st>>>(op, ctx->n, ctx->tbuf.p, ctx->scr);
    }
    if (ctx->sb_nb && ctx->sp_sb) {
      SbView A{ctx->sb_val, ctx->sb_idx, ctx->sb_base, ctx->sb_h, ctx->sb_perm, ctx->sb_chunk, ctx->sb_nslpb,
               ctx->sb_nb, ctx->n, ctx->d};
      const size_t sm = (size_t)SB_S * Op::R * sizeof(double);
      static unsigned long long attr = 0;
      if (once_per_device(attr)) cudaFuncSetAttribute(sp_zmv_sb_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      {
        Launch L(ctx, tag);
        sp_zmv_sb_kernel<Op><<<SB_CHUNKS / (Op::R == 1 ? 1 : 2), sb_threads<Op::R>(), sm, ctx->st>>>(
            op, A, ctx->tbuf.p, ctx->sb_part.p);
      }
      Launch L(ctx, "sp_zmv_sb_reduce");
      sp_zmv_sb_reduce_kernel<Op><<<(unsigned)((ctx->d + 32 * SBR_F - 1) / (32 * SBR_F)), SP_THREADS, 0, ctx->st>>>(op, ctx->sb_part.p,
                                                                                          ctx->sb_nb, ctx->d, g1, sc);
    } else {
      Launch L(ctx, tag);
      SpView A{ctx->csr_ptr, ctx->csr_idx, ctx->csr_val, ctx->d, ctx->n};
      sp_zmv_kernel<Op><<<sp_grid(ctx->d * 32, NUM_SMS * 8), SP_THREADS, 0, ctx->st>>>(op, A, ctx->tbuf.p, g1, sc);
    }
  } else {
    Launch L(ctx, tag);
    ZmvGeom g = zmv_geom(X.rows, X.cols, slots_for(zmv_kernel<Op>, ZMV_THREADS, 0));
    zmv_kernel<Op><<<dim3(g.tiles, g.segs), ZMV_THREADS, 0, ctx->st>>>(op, X, g, sc);
  }
  if (sh) {
    allreduce(ctx, ctx->bundle.p, (int64_t)Op::R * ctx->d + Op::NN);
    Launch L(ctx, "zmv_epilogue");
    zmv_epi_kernel<Op><<<vm_grid(ctx->d), VM_THREADS, 0, ctx->st>>>(op, ctx->bundle.p, ctx->d, ctx->scr);
  }
}
template <class Op>
static void run_zt(gdwd_ctx* ctx, const Op& op, MatView X, const char* tag = "ztmv") {
  // sample-space reductions only for products with Z~ itself (not factors)
  const bool sh = sharded(ctx) && Op::HAS_FIN && (!X.a || X.a == ctx->Zs);
  const Scratch sc = sh ? scr_bundle(ctx) : ctx->scr;
  {
    Launch L(ctx, tag);
    if (!X.a && ctx->fb_parts && ctx->sp_blocked) {
      FbView A{ctx->fb_ptr, ctx->fb_perm, ctx->fb_cnt, ctx->fb_idx, ctx->fb_val, ctx->n, ctx->d,
               ctx->fb_nb, FB_COLS, ctx->fb_parts, ctx->fb_S, ctx->fb_Q};
      const size_t sm = (size_t)(FB_COLS + ctx->fb_S) * sizeof(double);
      static unsigned long long attr = 0;
      if (once_per_device(attr))
        cudaFuncSetAttribute(sp_ztmv_fb_kernel<Op, FB_H, FB_U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FB_SMEM_MAX);
      sp_ztmv_fb_kernel<Op, FB_H, FB_U><<<ctx->fb_parts, FB_THREADS, sm, ctx->st>>>(op, A, sc);
    } else if (!X.a) {
      SpView A{ctx->csc_ptr, ctx->csc_idx, ctx->csc_val, ctx->n, ctx->d};
      sp_ztmv_kernel<Op, 8><<<sp_grid(ctx->n, NUM_SMS * 8), SP_THREADS, 0, ctx->st>>>(op, A, sc);
    } else {
      const int cw = zt_geom(X.rows, X.ld, NUM_SMS).cw;
      const size_t sm = (size_t)(cw + ZT_BATCH) * sizeof(double);
      ZtGeom g = zt_geom(X.rows, X.ld, slots_for(ztmv_kernel<Op>, ZT_THREADS, sm));
      ztmv_kernel<Op><<<dim3(g.chunks, g.ranges), ZT_THREADS, sm, ctx->st>>>(op, X, g, sc);
    }
  }
  if (sh) {
    allreduce(ctx, ctx->bundle.p, Op::NN);
    fin_kernel<Op, Op::NN><<<1, 1, 0, ctx->st>>>(op, ctx->bundle.p);
  }
}
// `samples`: the range is this rank's samples, so the fused sums are
// all-reduced across shards before fin (d-space ranges are replicated).
template <class Op>
static void run_vm(gdwd_ctx* ctx, const Op& op, int64_t len, const char* tag = "vmap", bool samples = false) {
  const bool sh = samples && sharded(ctx) && Op::HAS_FIN;
  {
    Launch L(ctx, tag);
    vmap_kernel<Op><<<vm_grid(len), VM_THREADS, 0, ctx->st>>>(op, len, sh ? scr_bundle(ctx) : ctx->scr);
  }
  if (sh) {
    allreduce(ctx, ctx->bundle.p, Op::NR);
    fin_kernel<Op, Op::NR><<<1, 1, 0, ctx->st>>>(op, ctx->bundle.p);
  }
}

// Fused dot -> epilogue -> axpy pass (zft.cuh) geometry: the smallest
// cluster whose feature slices fit the axpy threads' registers (<= 8 column
// pairs per thread); stages of ~32 KB, as many as fit 192 KB with the slice
// of w.  cs = 0: not eligible (d > 8 x 5120).
struct FtPlan {
  int cs = 0, dw = 0, tr = 0, ns = 0, p2 = 0;
};
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static FtPlan ft_plan(int64_t d) {
  FtPlan p;
  // one CTA per feature range (cs = 1): the cluster variants (cs > 1, wide
  // d) were measured slower than the two unfused passes (zft.cuh header)
  const int cs = std::max(1, env_int("GDWD_FT_CS", 1));  // (env: tuning experiments)
  const int64_t dw = ((d + cs - 1) / cs + 1) / 2 * 2;
  const int need = ft_pairs((int)std::min<int64_t>(dw, 1 << 20));
  if (need > 8) return p;
  p.cs = cs;
  p.dw = (int)dw;
  p.p2 = need <= 1 ? 1 : (need <= 2 ? 2 : (need <= 4 ? 4 : 8));
  const int64_t rb = (int64_t)p.dw * 8;
  p.tr = (int)std::max<int64_t>(1, std::min<int64_t>(ft_tra(p.p2), 65536 / rb));
  if (env_int("GDWD_FT_TR", 0) > 0) p.tr = std::min(env_int("GDWD_FT_TR", 0), ft_tra(p.p2));
  p.ns = (int)std::min<int64_t>(FT_NSMAX, 196608 / (p.tr * rb));
  if (env_int("GDWD_FT_NS", 0) > 1) p.ns = std::min(env_int("GDWD_FT_NS", 0), FT_NSMAX);
  // each tile carries ~2 us of dot and hand-off latency: the pass pays off
  // only with >= 32 KB tiles and 3 stages in flight (measured, zft.cuh)
  const bool forced = env_int("GDWD_FT_FORCE", 0) != 0;
  if (!forced && (p.tr * rb < 32 * 1024 || p.ns < 3 || cs != 1)) p.cs = 0;
  if ((p.ns * p.tr + 1) * rb > 208 * 1024 || p.ns < 2) p.cs = 0;
  return p;
}
static bool ft_enabled() {
  const char* e = getenv("GDWD_FT");
  return !(e && atoi(e) == 0);
}

// (the occupancy query and attribute set run the first time a geometry is
// seen on a device; solve_begin calls run_ft with prepare_only before any
// graph capture, where they are not allowed)
template <class Op, int P2>
static void launch_ft(gdwd_ctx* ctx, const Op& op, MatView X, const FtPlan& p, FtGeom& g, const Scratch& sc,
                      bool prepare_only) {
  auto kfn = zft_kernel<Op, P2>;
  g = FtGeom{p.cs, 0, p.dw, p.tr, p.ns, (X.cols + 1) / 2 * 2};
  const size_t sm = ft_smem_bytes(g, Op::R);
  static std::map<std::pair<int, size_t>, int> cache;  // (device x cs, smem) -> co-resident clusters
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(FT_THREADS);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = ctx->st;
  cfg.attrs = at;
  cfg.numAttrs = p.cs > 1 ? 1 : 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    // the attribute is per function and device: only ever raise it (a smaller
    // geometry seen later must not shrink it under a cached larger one)
    static size_t attr_max[64] = {};
    if (prepare_only && sm > attr_max[dev & 63]) {
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr_max[dev & 63] = sm;
    }
    auto key = std::make_pair(dev * 16 + p.cs, sm);
    auto it = cache.find(key);
    if (it == cache.end()) {
      int nc = 0;
      if (p.cs > 1) {
        cfg.gridDim = dim3(p.cs * (NUM_SMS / p.cs));
        if (cudaOccupancyMaxActiveClusters(&nc, kfn, &cfg) != cudaSuccess) nc = 0;
      } else {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kfn, FT_THREADS, sm) != cudaSuccess) nb = 0;
        nc = nb * NUM_SMS;
      }
      cudaGetLastError();
      it = cache.emplace(key, std::max(nc, 1)).first;
    }
    g.clusters = it->second;
  }
  if (prepare_only) {
    if (getenv("GDWD_FT_TIMING")) {  // diagnostics: stamps of the last launch, ft_timing_report
      static unsigned long long* buf = nullptr;
      if (!buf) cudaMalloc(&buf, sizeof(unsigned long long) * FT_TS_TILES * FT_TS_PTS);
      cudaMemset(buf, 0, sizeof(unsigned long long) * FT_TS_TILES * FT_TS_PTS);
      cudaMemcpyToSymbol(g_ft_ts, &buf, sizeof(buf));
      ctx->ft_ts = buf;
    }
    return;
  }
  cfg.gridDim = dim3(g.clusters * p.cs);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, op, X, g, sc);
  if (e != cudaSuccess && getenv("GDWD_DEBUG_LAUNCH"))
    fprintf(stderr, "zft launch: %s (grid %d x %d, smem %zu)\n", cudaGetErrorString(e), g.clusters, p.cs, sm);
}

// One fused pass; the per-cluster partials are summed (cluster order) by the
// reduce kernel, which runs the per-feature epilogue and fin -- or, sharded,
// publishes the local products and n-sums for the all-reduce.
template <class Op>
static void run_ft(gdwd_ctx* ctx, const Op& op, MatView X, const char* tag = "zft", bool prepare_only = false) {
  const bool sh = sharded(ctx);
  const Scratch sc = sh ? scr_bundle(ctx) : ctx->scr;
  const FtPlan p = ft_plan(X.cols);
  FtGeom g{};
  if (prepare_only) {
    switch (p.p2) {
      case 1: launch_ft<Op, 1>(ctx, op, X, p, g, sc, true); break;
      case 2: launch_ft<Op, 2>(ctx, op, X, p, g, sc, true); break;
      case 4: launch_ft<Op, 4>(ctx, op, X, p, g, sc, true); break;
      default: launch_ft<Op, 8>(ctx, op, X, p, g, sc, true); break;
    }
    if (getenv("GDWD_FT_DEBUG"))
      fprintf(stderr, "zft plan: d=%lld cs=%d dw=%d p2=%d tr=%d ns=%d clusters=%d smem=%zu\n", (long long)X.cols,
              p.cs, p.dw, p.p2, p.tr, p.ns, g.clusters, ft_smem_bytes(g, Op::R));
    return;
  }
  {
    Launch L(ctx, tag);
    switch (p.p2) {
      case 1: launch_ft<Op, 1>(ctx, op, X, p, g, sc, false); break;
      case 2: launch_ft<Op, 2>(ctx, op, X, p, g, sc, false); break;
      case 4: launch_ft<Op, 4>(ctx, op, X, p, g, sc, false); break;
      default: launch_ft<Op, 8>(ctx, op, X, p, g, sc, false); break;
    }
  }
  {
    Launch L(ctx, "zft_reduce");
    zft_reduce_kernel<Op><<<(unsigned)((X.cols + 31) / 32), FTR_THREADS, 0, ctx->st>>>(op, X.cols, g.clusters, g.ldp, sc);
  }
  if (sh) {
    allreduce(ctx, ctx->bundle.p, (int64_t)Op::R * ctx->d + Op::NN);
    Launch L(ctx, "zmv_epilogue");
    zmv_epi_kernel<Op><<<vm_grid(ctx->d), VM_THREADS, 0, ctx->st>>>(op, ctx->bundle.p, ctx->d, ctx->scr);
  }
}

static void prof_flush(gdwd_ctx* ctx) {
  if (ctx->prof_pending.empty()) return;
  cudaStreamSynchronize(ctx->st);
  for (auto& r : ctx->prof_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& acc = ctx->prof_acc[r.tag];
    acc.first += 1;
    acc.second += ms;
  }
  ctx->prof_pending.clear();
  ctx->ev_used = 0;
}

// scratch sized for matrices with (rows, cols)
static int ensure_scratch(gdwd_ctx* ctx, int64_t rows, int64_t cols) {
  const int maxslots = NUM_SMS * 32;  // upper bound on resident CTAs
  ZmvGeom zg = zmv_geom(rows, cols, maxslots);
  ZtGeom tg = zt_geom(rows, (cols + 1) / 2 * 2, maxslots);
  size_t part = std::max<size_t>((size_t)zg.segs * 2 * zg.ldp, tg.chunks > 1 ? (size_t)tg.chunks * rows : 0);
  part = std::max<size_t>(part, (size_t)NUM_SMS * 2 * zg.ldp);  // fused tail: <= 148 clusters x 2 products
  size_t npart = (size_t)maxslots * 16;
  size_t tpart = (size_t)std::max<int64_t>(zg.tiles, NUM_SMS * 8) * 16 + 16;
  tpart = std::max<size_t>(tpart, (size_t)((cols + 31) / 32) * 4 + 16);  // per-32-feature reduce CTAs (ND <= 4)
  size_t nt = (size_t)std::max<int64_t>(zg.tiles, maxslots) + 4;
  CK(ctx->part.ensure(std::max(part, ctx->part.n)));
  CK(ctx->npart.ensure(std::max(npart, ctx->npart.n)));
  CK(ctx->tpart.ensure(std::max(tpart, ctx->tpart.n)));
  if (nt > ctx->ntickets) {
    dfree(ctx->tickets, ctx->st);
    CK(dmalloc((void**)&ctx->tickets, nt * sizeof(unsigned), ctx->st));
    // ordered on st (non-blocking: the legacy stream does not synchronise with it)
    CK(cudaMemsetAsync(ctx->tickets, 0, nt * sizeof(unsigned), ctx->st));
    ctx->ntickets = nt;
  }
  CK(ctx->bundle.ensure(std::max<size_t>((size_t)2 * cols + 32, ctx->bundle.n)));
  ctx->scr = Scratch{ctx->part.p, ctx->npart.p, ctx->tpart.p, ctx->tickets, nullptr};
  return GDWD_OK;
}

// column sums of squares (row_sq_sums, sparse.py:66-70): sequential per
// column (same order as np.bincount) for moderate n, segmented zmv beyond
struct OpColSq {
  static constexpr int R = 1, NN = 1, ND = 1;
  static constexpr bool SQ = true;
  double* out;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void input(int64_t, double (&t)[R], double (&)[NN]) const { t[0] = 1.0; }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const { out[j] = v[0]; }
  GDWD_DEV void fin(const double (&)[NN], const double (&)[ND]) const {}
};
// (sequential variant below)
struct OpColSqPrep {};
template <class Op>
__global__ void colsq_kernel(MatView X, double* out) {
  // one thread per column, fixed sample order (matches bincount's order)
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= X.cols) return;
  double s = 0.0;
  for (int64_t i = 0; i < X.rows; ++i) {
    const double v = X.a[i * X.ld + j];
    s += v * v;
  }
  out[j] = s;
}

__global__ void jacobi_kernel(const double* colsq, int64_t d, double mu2, double yty, double* jac) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < d) {
    const double v = colsq[j] + mu2;
    jac[j] = v > 1e-12 ? v : 1e-12;
  } else if (j == d) {
    const double v = yty > mu2 ? yty : mu2;
    jac[j] = v > 1e-12 ? v : 1e-12;
  }
}

__global__ void add_diag_kernel(double* A, int64_t ld, int64_t d, double v) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < d) A[j * ld + j] += v;
}

__global__ void assemble_direct_kernel(double* A, int64_t ld, int64_t d, const double* zy, double yty) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < d) {
    A[j * ld + d] = zy[j];
    A[d * ld + j] = zy[j];
  } else if (j == d) {
    A[d * ld + d] = yty;
  }
}

// sum of squares over rows x cols (row stride ld) into *out, deterministic
struct OpSumSq {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  const double* a;
  int64_t cols, ld;
  double* out;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void elem(int64_t idx, double (&acc)[NR]) const {
    const double v = a[(idx / cols) * ld + idx % cols];
    acc[0] += v * v;
  }
  GDWD_DEV void fin(const double (&sum)[NR]) const { *out = sum[0]; }
};

// G = K / mu^2 + I (subsolvers.py:109-110: gram / mu_sq, then += 1 on the diagonal)
__global__ void g_from_k_kernel(const double* K, double* G, int64_t n, int64_t ld, double mu2) {
  const int64_t tot = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx % n;
    double v = K[i * ld + j] / mu2;
    if (i == j) v += 1.0;
    G[i * ld + j] = v;
  }
}

// G^{-1} K = G^{-1} mu^2 (G - I) = mu^2 (I - G^{-1}) for G = K / mu^2 + I:
// the persistent loop's GK from the explicit inverse, elementwise.
__global__ void gk_from_ginv_kernel(const double* Gi, double* GK, int64_t n, int64_t ld, double mu2) {
  const int64_t tot = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx % n;
    const double v = (i == j ? 1.0 : 0.0) - Gi[i * ld + j];
    GK[i * ld + j] = mu2 == 1.0 ? v : mu2 * v;
  }
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

static void fill(gdwd_ctx* ctx, double* p, int64_t n, double v) {
  fill_kernel<<<vm_grid(n), 256, 0, ctx->st>>>(p, n, v);
}

// Host -> device copy of the [n][d] sample matrix into rows of stride ld.
// Default: one pageable 2-D copy (~10 GB/s measured on the B200 hosts).
// GDWD_UPLOAD=staged stages through two
// pinned 64 MB buffers (host threads copy chunk k+1 while the DMA engine
// drains chunk k); GDWD_UPLOAD=register page-locks the source in place.
// (Both measured slower per call: pinned allocation / registration cost.)
static int upload_rows(gdwd_ctx* ctx, const double* src, int64_t d, int64_t n, int64_t ld) {
  const char* mode = getenv("GDWD_UPLOAD");
  const size_t row_b = (size_t)d * sizeof(double);
  const size_t total = row_b * (size_t)n;
  if (!mode || !strcmp(mode, "pageable")) {
    CK(cudaMemcpy2DAsync(ctx->Zs, ld * sizeof(double), src, row_b, row_b, n, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return GDWD_OK;
  }
  if (mode && !strcmp(mode, "register")) {
    CK(cudaHostRegister((void*)src, total, cudaHostRegisterReadOnly));
    cudaError_t e = cudaMemcpy2DAsync(ctx->Zs, ld * sizeof(double), src, row_b, row_b, n, cudaMemcpyHostToDevice, ctx->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    cudaHostUnregister((void*)src);
    CK(e);
    return GDWD_OK;
  }
  const size_t chunk_rows = std::max<size_t>(1, ((size_t)64 << 20) / row_b);
  if (!ctx->pin[0]) {
    for (int b = 0; b < 2; ++b) {
      CK(cudaMallocHost(&ctx->pin[b], (size_t)64 << 20 < row_b ? row_b : (size_t)64 << 20));
      CK(cudaEventCreateWithFlags(&ctx->pin_ev[b], cudaEventDisableTiming));
    }
    ctx->pin_bytes = (size_t)64 << 20 < row_b ? row_b : (size_t)64 << 20;
  }
  if (chunk_rows * row_b > ctx->pin_bytes) return set_err(ctx, GDWD_ERR_CUDA, "staging buffer too small");
  const unsigned nthr = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  int b = 0;
  bool used[2] = {false, false};
  for (int64_t r0 = 0; r0 < n; r0 += (int64_t)chunk_rows, b ^= 1) {
    const int64_t rows = std::min<int64_t>((int64_t)chunk_rows, n - r0);
    if (used[b]) CK(cudaEventSynchronize(ctx->pin_ev[b]));
    const char* s0 = (const char*)(src + r0 * d);
    char* d0 = (char*)ctx->pin[b];
    const size_t bytes = (size_t)rows * row_b;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nthr; ++t) {
      const size_t lo = bytes * t / nthr, hi = bytes * (t + 1) / nthr;
      th.emplace_back([=] { memcpy(d0 + lo, s0 + lo, hi - lo); });
    }
    for (auto& x : th) x.join();
    CK(cudaMemcpy2DAsync(ctx->Zs + r0 * ld, ld * sizeof(double), ctx->pin[b], row_b, row_b, rows,
                         cudaMemcpyHostToDevice, ctx->st));
    CK(cudaEventRecord(ctx->pin_ev[b], ctx->st));
    used[b] = true;
  }
  CK(cudaStreamSynchronize(ctx->st));
  return GDWD_OK;
}

// one page-locked double per context from a process-wide block (contexts are
// created inside timed end-to-end calls; cudaMallocHost is milliseconds)
static double* pinned_slot() {
  static std::mutex mu;
  static double* block = nullptr;
  static int used = 0, cap = 0;
  std::lock_guard<std::mutex> g(mu);
  if (used == cap) {
    cap = 4096;
    used = 0;
    if (cudaMallocHost(&block, cap * sizeof(double)) != cudaSuccess) return nullptr;
  }
  return block + used++;
}

// ||Z~||_F^2 on the host, waiting for a deferred reduction if one is queued
static double get_fro2(gdwd_ctx* ctx) {
  if (ctx->fro2_pending) {
    cudaStreamSynchronize(ctx->st);
    ctx->fro2 = *ctx->fro2_h;
    ctx->fro2_pending = false;
  }
  return ctx->fro2;
}

// the host buffer of an overlapped upload is borrowed until its copies land
static void finish_upload(gdwd_ctx* ctx) {
  if (ctx->cst) cudaStreamSynchronize(ctx->cst);
  ctx->up_pending = false;
}

static int compute_fro2(gdwd_ctx* ctx, const double* a, int64_t rows, int64_t cols, int64_t ld) {
  ctx->fro2_pending = false;  // a deferred reduction of earlier data must not overwrite this value
  double* dv = nullptr;
  CK(cudaMalloc(&dv, sizeof(double)));
  run_vm(ctx, OpSumSq{a, cols, ld, dv}, rows * cols, "vmap_fro2", true);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&ctx->fro2, dv, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  cudaFree(dv);
  return GDWD_OK;
}

static void free_sparse(gdwd_ctx* ctx) {
  for (void* p : {(void*)ctx->csc_ptr, (void*)ctx->csr_ptr, (void*)ctx->csc_idx, (void*)ctx->csr_idx,
                  (void*)ctx->csc_val, (void*)ctx->csr_val, (void*)ctx->fb_ptr, (void*)ctx->fb_idx,
                  (void*)ctx->fb_val, (void*)ctx->fb_perm, (void*)ctx->fb_cnt, (void*)ctx->sb_val, (void*)ctx->sb_idx,
                  (void*)ctx->sb_base, (void*)ctx->sb_h, (void*)ctx->sb_perm, (void*)ctx->sb_chunk})
    dfree(p, ctx->st);
  ctx->sb_val = nullptr;
  ctx->sb_idx = nullptr;
  ctx->sb_base = nullptr;
  ctx->sb_h = ctx->sb_perm = ctx->sb_chunk = nullptr;
  ctx->sb_nb = ctx->sb_nslpb = 0;
  ctx->sb_entries = 0;
  ctx->csc_ptr = ctx->csr_ptr = nullptr;
  ctx->csc_idx = ctx->csr_idx = nullptr;
  ctx->csc_val = ctx->csr_val = nullptr;
  ctx->fb_ptr = nullptr;
  ctx->fb_idx = ctx->fb_perm = ctx->fb_cnt = nullptr;
  ctx->fb_val = nullptr;
  ctx->fb_nb = ctx->fb_parts = ctx->fb_S = ctx->fb_Q = 0;
  ctx->fb_entries = 0;
  ctx->has_sparse = false;
  ctx->nnz = 0;
}

// Diagnostics (GDWD_PK_TIMING): per-CTA %globaltimer stamps of the persistent
// kernel; for every phase point, the mean over iterations of the earliest,
// median and latest CTA relative to the iteration's first CTA start.
static void pk_timing_report(unsigned long long* ts, size_t tsn, int version) {
  std::vector<unsigned long long> h(tsn);
  if (cudaMemcpy(h.data(), ts, tsn * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) return;
  cudaFree(ts);
  const int NP = 32;
  if (version == 3) {  // launch prologue / epilogue: points 27 (entry), 28 (loop start), 29 (exit) in row 0
    std::vector<double> pro, epi;
    unsigned long long emin = ~0ull, emax = 0;
    for (int b = 0; b < NUM_SMS; ++b) {
      const unsigned long long* r = &h[(size_t)b * NP];
      if (r[27] && r[28]) pro.push_back((r[28] - r[27]) / 1965.0);
      if (r[27]) emin = std::min(emin, r[27]), emax = std::max(emax, r[27]);
    }
    if (!pro.empty()) {
      std::sort(pro.begin(), pro.end());
      fprintf(stderr, "[pk timing] launch prologue (entry -> loop) median %.2f us  slowest %.2f us\n",
              pro[pro.size() / 2], pro.back());
    }
  }
  const char* names[NP] = {"top", "A arrive", "A release", "C arrive", "C release", "D arrive", "D release",
                           "E arrive", "E release", "H arrive", "H release", "H staged", "H rows", "H step3",
                           "C staged", "C rows", "C scalars", "C writeback", "C waited", "C loop",
                           "D waited", "D staged", "", "", "A waited", "A loop", "A staged", "", "", "", "", ""};
  // per-CTA SM-clock intervals between consecutive points (1.965 GHz), the
  // median and the slowest CTA, averaged over iterations
  const int order2[] = {0, 24, 25, 26, 1, 2, 16, 17, 18, 19, 14, 15, 3, 4, 20, 21, 5, 6, 11, 12, 13, 9, 10};
  // persist3.cuh points, in time order (interval named by its start point)
  const char* names3[15] = {"A wait in", "A staging", "A sum+scal", "A rows", "A partials", "B1 barrier",
                            "B1 scalars", "D staging", "D rows", "D partials", "B2 barrier", "B2 scal+H rows",
                            "H partials", "B3 barrier", "B3 scalars"};
  const int order3[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14};
  const int* order = version == 3 ? order3 : order2;
  const int no = version == 3 ? 15 : (int)(sizeof(order2) / sizeof(order2[0]));
  std::vector<double> sum_med(no, 0.0), sum_max(no, 0.0);
  int cnt = 0;
  std::vector<double> v;
  for (int it = 1; it + 1 < PK_TS_ITERS; ++it) {
    const unsigned long long* r = &h[(size_t)it * NUM_SMS * NP];
    const unsigned long long* rn = &h[(size_t)(it + 1) * NUM_SMS * NP];
    bool ok = true;
    for (int b = 0; b < NUM_SMS && ok; ++b)
      for (int q = 0; q < no; ++q)
        if (!r[b * NP + order[q]] || !rn[b * NP]) ok = false;
    if (!ok) break;
    for (int q = 0; q < no; ++q) {
      v.clear();
      for (int b = 0; b < NUM_SMS; ++b) {
        const unsigned long long t0 = r[b * NP + order[q]];
        const unsigned long long t1 = q + 1 < no ? r[b * NP + order[q + 1]] : rn[b * NP];
        v.push_back((double)(long long)(t1 - t0) / 1965.0);
      }
      std::sort(v.begin(), v.end());
      sum_med[q] += v[v.size() / 2];
      sum_max[q] += v.back();
    }
    cnt++;
  }
  if (!cnt) return;
  double tot = 0.0;
  fprintf(stderr, "[pk timing] interval from point   median-CTA us   slowest-CTA us\n");
  for (int q = 0; q < no; ++q) {
    tot += sum_med[q] / cnt;
    fprintf(stderr, "[pk timing] %-14s %10.2f %10.2f\n", version == 3 ? names3[q] : names[order[q]], sum_med[q] / cnt,
            sum_max[q] / cnt);
  }
  fprintf(stderr, "[pk timing] sum of medians %.2f us over %d iterations\n", tot, cnt);
  if (version != 3) return;
  // arrival skew: per-CTA time from leaving one barrier's cross-sum to
  // arriving at the next barrier (median / slowest CTA), and the barrier
  // interval of the median CTA
  struct Seg { const char* name; int a, b; bool wrap; };
  const Seg segs[] = {{"B3 exit -> B1 arrive", 14, 5, true}, {"B1 exit -> B2 arrive", 6, 10, false},
                      {"B2 exit -> B3 arrive", 11, 13, false}};
  for (const Seg& g : segs) {
    double smed = 0.0, smax = 0.0;
    int c2 = 0;
    for (int it = 1; it + 1 < PK_TS_ITERS && c2 < cnt; ++it, ++c2) {
      const unsigned long long* r = &h[(size_t)it * NUM_SMS * NP];
      const unsigned long long* rn = &h[(size_t)(it + 1) * NUM_SMS * NP];
      v.clear();
      for (int b = 0; b < NUM_SMS; ++b) {
        const unsigned long long t0 = r[b * NP + g.a];
        const unsigned long long t1 = g.wrap ? rn[b * NP + g.b] : r[b * NP + g.b];
        v.push_back((double)(long long)(t1 - t0) / 1965.0);
      }
      std::sort(v.begin(), v.end());
      smed += v[v.size() / 2];
      smax += v.back();
    }
    if (c2) fprintf(stderr, "[pk timing] path %-22s median %6.2f slowest %6.2f us (skew %.2f)\n", g.name, smed / c2,
                    smax / c2, (smax - smed) / c2);
  }
}

// streams + events of the pipelined upload, pooled per device
struct UploadAux {
  int device = -1;
  cudaStream_t s[5] = {};
  cudaEvent_t e[2 * gdwd_ctx::UP_MAXB + 3] = {};
  double* pin = nullptr;  // page-locked staging ring for pageable sources (kept with the pooled object)
  size_t pin_bytes = 0;
};
constexpr int UP_NSLOT = 3;  // staging slots (blocks in flight between the host copy and the DMA)
constexpr int UP_NO_STAGING = -1;  // internal: the page-locked ring could not be allocated
static std::mutex g_aux_mu;
static std::vector<UploadAux*> g_aux_free;
static UploadAux* upload_aux_acquire(int device) {
  {
    std::lock_guard<std::mutex> g(g_aux_mu);
    for (size_t i = 0; i < g_aux_free.size(); ++i)
      if (g_aux_free[i]->device == device) {
        UploadAux* a = g_aux_free[i];
        g_aux_free.erase(g_aux_free.begin() + i);
        return a;
      }
  }
  UploadAux* a = new UploadAux;
  a->device = device;
  int lo = 0, hi = 0;
  bool ok = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&a->s[0], cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&a->s[1], cudaStreamNonBlocking) == cudaSuccess;
  // the dependent chain is latency-bound: its CTAs go ahead of the Gram's
  for (int i = 2; i < 5; ++i) ok = ok && cudaStreamCreateWithPriority(&a->s[i], cudaStreamNonBlocking, hi) == cudaSuccess;
  for (auto& e : a->e) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    delete a;
    return nullptr;
  }
  return a;
}
static void upload_aux_release(UploadAux* a) {
  if (!a) return;
  for (cudaStream_t x : a->s) cudaStreamSynchronize(x);
  std::lock_guard<std::mutex> g(g_aux_mu);
  g_aux_free.push_back(a);
}

// Host scratch array without the single-threaded zero fill of std::vector:
// the worker threads' first touch places (and faults in) the pages in
// parallel.  Every element is written before it is read.
template <class T>
struct RawBuf {
  std::unique_ptr<T[]> p;
  size_t n = 0;
  explicit RawBuf(size_t cnt) : p(new T[std::max<size_t>(cnt, 1)]), n(cnt) {}
  T* data() { return p.get(); }
  const T* data() const { return p.get(); }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
  size_t size() const { return n; }
};

// Per-context device/host scalars, streams and events, pooled per device:
// contexts are created inside timed end-to-end calls, and cudaMalloc /
// cudaMallocHost / stream and event creation cost ~0.4 ms per context.
struct CtxAux {
  int device = -1;
  cudaStream_t st = nullptr, cap_st = nullptr;
  Scal* S = nullptr;
  Scal* Sh = nullptr;
  int* dinfo = nullptr;
  int* poll_flag = nullptr;
  double* stage = nullptr;  // pinned, CTX_STAGE_DOUBLES: result download staging
  cudaEvent_t poll_ev[2] = {}, ev[3] = {};
};
constexpr size_t CTX_STAGE_DOUBLES = (size_t)1 << 17;  // 1 MB
static std::mutex g_ctxaux_mu;
static std::vector<CtxAux*> g_ctxaux_free;
static CtxAux* ctx_aux_acquire(int device) {
  {
    std::lock_guard<std::mutex> g(g_ctxaux_mu);
    for (size_t i = 0; i < g_ctxaux_free.size(); ++i)
      if (g_ctxaux_free[i]->device == device) {
        CtxAux* a = g_ctxaux_free[i];
        g_ctxaux_free.erase(g_ctxaux_free.begin() + i);
        return a;
      }
  }
  CtxAux* a = new CtxAux;
  a->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&a->st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a->cap_st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&a->S, sizeof(Scal));
  if (e == cudaSuccess) e = cudaMallocHost(&a->Sh, sizeof(Scal));
  if (e == cudaSuccess) e = cudaMalloc(&a->dinfo, sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&a->poll_flag, 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&a->stage, CTX_STAGE_DOUBLES * sizeof(double));
  for (auto& x : a->poll_ev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  for (auto& x : a->ev)
    if (e == cudaSuccess) e = cudaEventCreate(&x);
  if (e != cudaSuccess) {
    fprintf(stderr, "gdwd_ctx_create: %s\n", cudaGetErrorString(e));
    delete a;  // partial resources leak; the process is unusable anyway
    return nullptr;
  }
  return a;
}
static void ctx_aux_release(CtxAux* a) {
  if (!a) return;
  cudaStreamSynchronize(a->st);
  cudaStreamSynchronize(a->cap_st);
  std::lock_guard<std::mutex> g(g_ctxaux_mu);
  g_ctxaux_free.push_back(a);
}

extern "C" {

int gdwd_version(void) { return 1; }

void gdwd_abi_sizes(int64_t* config_bytes, int64_t* result_bytes) {
  if (config_bytes) *config_bytes = (int64_t)sizeof(gdwd_config);
  if (result_bytes) *result_bytes = (int64_t)sizeof(gdwd_result);
}

const char* gdwd_last_error(const gdwd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gdwd_ctx_create(int32_t device, gdwd_ctx** out) {
  if (!out) return GDWD_ERR_VALUE;
  *out = nullptr;
  gdwd_ctx* ctx = new gdwd_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  CtxAux* ax = e == cudaSuccess ? ctx_aux_acquire(device) : nullptr;
  if (!ax) {
    if (e != cudaSuccess) fprintf(stderr, "gdwd_ctx_create: %s\n", cudaGetErrorString(e));
    delete ctx;
    return GDWD_ERR_CUDA;
  }
  ctx->aux = ax;
  ctx->st = ax->st;
  ctx->cap_st = ax->cap_st;
  ctx->S = ax->S;
  ctx->Sh = ax->Sh;
  ctx->dinfo = ax->dinfo;
  ctx->poll_flag = ax->poll_flag;
  ctx->poll_ev[0] = ax->poll_ev[0];
  ctx->poll_ev[1] = ax->poll_ev[1];
  ctx->ev_begin = ax->ev[0];
  ctx->ev_loop = ax->ev[1];
  ctx->ev_end = ax->ev[2];
  if (e == cudaSuccess) {
    keep_pool_reserved(device);
    for (DevBuf* b : {&ctx->y, &ctx->e, &ctx->wl, &ctx->part, &ctx->npart, &ctx->tpart, &ctx->nvec, &ctx->mvec,
                    &ctx->tabs, &ctx->histb, &ctx->fac, &ctx->facw, &ctx->colsq, &ctx->tbuf, &ctx->kmat, &ctx->pk_part, &ctx->gkmat, &ctx->bundle, &ctx->pxbuf, &ctx->gdmat, &ctx->gram_ws, &ctx->sb_part, &ctx->pfw})
      b->st = ctx->st;
  }
  *out = ctx;
  return GDWD_OK;
}

void gdwd_ctx_destroy(gdwd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  if (ctx->cst) {
    cudaStreamSynchronize(ctx->cst);
    cudaStreamSynchronize(ctx->gst);
    upload_aux_release((UploadAux*)ctx->up_aux);  // synchronises its streams
    dfree(ctx->fro2_d, ctx->st);
  }
  dfree(ctx->Zs, ctx->st);
  free_sparse(ctx);
  for (DevBuf* b : {&ctx->y, &ctx->e, &ctx->wl, &ctx->part, &ctx->npart, &ctx->tpart, &ctx->nvec, &ctx->mvec,
                    &ctx->tabs, &ctx->histb, &ctx->fac, &ctx->facw, &ctx->colsq, &ctx->tbuf, &ctx->kmat, &ctx->pk_part, &ctx->gkmat, &ctx->bundle, &ctx->pxbuf, &ctx->gdmat, &ctx->gram_ws, &ctx->sb_part, &ctx->pfw})
    b->release();
  end_session(ctx);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->bundle_h) cudaFreeHost(ctx->bundle_h);
  if (ctx->comm && nccl::api().ok) nccl::api().CommDestroy(ctx->comm);
  for (int b = 0; b < 2; ++b) {
    if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
    if (ctx->pin_ev[b]) cudaEventDestroy(ctx->pin_ev[b]);
  }
  dfree(ctx->tickets, ctx->st);
  ctx_aux_release((CtxAux*)ctx->aux);  // synchronises st (the frees above are ordered on it)
  delete ctx;
}

static int select_kind(int64_t n, int64_t d);


// Page-locked dense upload in the sample-space regimes, pipelined with the
// one-time factorisation (subsolvers.py:109-113, cholesky.py:46,60-61): block
// b of samples is copied (contiguous rows) on cst; gst then forms its rows of
// K = Z~^T Z~ (DMMA, split-K partials summed in slice order) and of
// G = K/mu^2 + I; fst advances the bordered Cholesky factor -- the block's
// rows of L^{-1} from the rows before -- with the half that does not need the
// diagonal block on sst, and ast adds the block's term of
// G^{-1} = L^{-T} L^{-1}.  Only the last block's share runs after the last
// byte has landed.  mu comes from the upload hint (default 1); a solve with
// another mu, or outside the sample-space regimes, refactors from K.
static int upload_dense_pipelined(gdwd_ctx* ctx, const double* samples, int64_t d, int64_t n, int64_t ld,
                                  bool pinned) {
  Range nvtx_range("upload_dense_pipelined (copy + Gram + factor)");
  const auto t_pre0 = std::chrono::steady_clock::now();
  if (!ctx->cst) {
    // streams and events come from a process-wide pool (contexts are created
    // inside timed end-to-end calls; creating 5 streams + 51 events is ~0.25 ms)
    UploadAux* ax = upload_aux_acquire(ctx->device);
    if (!ax) return set_err(ctx, GDWD_ERR_CUDA, "upload streams");
    ctx->up_aux = ax;
    ctx->cst = ax->s[0]; ctx->gst = ax->s[1]; ctx->fst = ax->s[2]; ctx->sst = ax->s[3]; ctx->ast = ax->s[4];
    for (int i = 0; i < gdwd_ctx::UP_MAXB; ++i) {
      ctx->up_ev[i] = ax->e[i];
      ctx->gr_ev[i] = ax->e[gdwd_ctx::UP_MAXB + i];
    }
    ctx->gram_ev = ax->e[2 * gdwd_ctx::UP_MAXB];
    ctx->st_ev = ax->e[2 * gdwd_ctx::UP_MAXB + 1];
    ctx->pf_ev = ax->e[2 * gdwd_ctx::UP_MAXB + 2];
    ctx->fro2_h = pinned_slot();
    CK(dmalloc((void**)&ctx->fro2_d, sizeof(double), ctx->st));
  }
  // factor only where the solve will run in sample space (gdwd_solve_begin:
  // SMW2 with n <= d, DIRECT with 2n <= d)
  int hk = ctx->hint_backend == GDWD_BACKEND_AUTO ? select_kind(n, d) : ctx->hint_backend;
  const bool factor = (hk == GDWD_BACKEND_SMW2 || (hk == GDWD_BACKEND_DIRECT && 2 * n <= d)) &&
                      getenv("GDWD_UPLOAD_FACTOR") == nullptr;
  const double mu2 = ctx->hint_mu * ctx->hint_mu;
  const int64_t ldk = (n + 1) / 2 * 2;
  int64_t mb = gdwd_ctx::UP_BLOCK;
  if (const char* ev = getenv("GDWD_UP_BLOCK")) mb = std::max(16, atoi(ev));
  // GDWD_UP_FINE: the last `fine` rows in half-size blocks (measured: the
  // smaller launches lose more than the shorter last block gains; default 0)
  int64_t fine = 0;
  if (const char* ev = getenv("GDWD_UP_FINE")) fine = std::max(0, atoi(ev));
  while ((n + mb - 1) / mb + fine / mb > gdwd_ctx::UP_MAXB) mb += 64;
  int64_t rb[gdwd_ctx::UP_MAXB + 1];
  int nblk = 0;
  rb[0] = 0;
  while (rb[nblk] < n) {
    const int64_t left = n - rb[nblk];
    const int64_t step = (left <= fine && mb >= 32) ? mb / 2 : mb;
    rb[nblk + 1] = std::min<int64_t>(n, rb[nblk] + step);
    ++nblk;
  }
  const auto t_pre1 = std::chrono::steady_clock::now();
  CK(ctx->kmat.ensure((size_t)n * ldk));
  CK(ctx->fac.ensure((size_t)n * ldk));
  const int64_t bws = bordered_workspace(n, mb);
  CK(ctx->pfw.ensure((size_t)3 * n * ldk + (size_t)bws));
  CK(ctx->gram_ws.ensure((size_t)std::max(gram_rowblock_workspace(n, d, mb),
                                          gram_rowblock_workspace(n, d, std::max<int64_t>(mb / 2, 1)))));
  double* G = ctx->pfw.p;
  double* Wi = G + (size_t)n * ldk;
  double* T = Wi + (size_t)n * ldk;
  // zero: K's pad column (the persistent kernel's paired loads read it),
  // L^{-1}'s upper triangle, the accumulated G^{-1}
  CK(cudaMemsetAsync(ctx->kmat.p, 0, (size_t)n * ldk * sizeof(double), ctx->st));
  if (factor) {
    CK(cudaMemsetAsync(Wi, 0, (size_t)n * ldk * sizeof(double), ctx->st));
    CK(cudaMemsetAsync(ctx->fac.p, 0, (size_t)n * ldk * sizeof(double), ctx->st));
    CK(cudaMemsetAsync(ctx->dinfo, 0, sizeof(int), ctx->st));
  }
  CK(cudaEventRecord(ctx->st_ev, ctx->st));  // allocation / pad memsets first
  for (cudaStream_t x : {ctx->cst, ctx->gst, ctx->fst, ctx->ast}) CK(cudaStreamWaitEvent(x, ctx->st_ev, 0));
  const size_t row_b = (size_t)d * sizeof(double);
  const bool tmark = getenv("GDWD_SETUP_TIMING") != nullptr;
  // GDWD_SETUP_TIMING: device timeline (ms after the first copy starts) of
  // each block's copy / Gram rows / factor rows / G^{-1} term
  std::vector<cudaEvent_t> tl[4];
  cudaEvent_t tl0 = nullptr;
  auto tev = [&](int lane, int, cudaStream_t x) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, x);
    tl[lane].push_back(e);
  };
  if (tmark) {
    cudaEventCreate(&tl0);
    cudaEventRecord(tl0, ctx->cst);
  }
  const auto t_h0 = std::chrono::steady_clock::now();
  auto queue_copy = [&](int b, const double* src) -> int {
    const int64_t r0 = rb[b], r1 = rb[b + 1];
    if (ld == d)
      CK(cudaMemcpyAsync(ctx->Zs + r0 * ld, src, (size_t)(r1 - r0) * row_b, cudaMemcpyHostToDevice, ctx->cst));
    else
      CK(cudaMemcpy2DAsync(ctx->Zs + r0 * ld, ld * sizeof(double), src, row_b, row_b, r1 - r0,
                           cudaMemcpyHostToDevice, ctx->cst));
    CK(cudaEventRecord(ctx->up_ev[b], ctx->cst));
    if (tmark) tev(0, b, ctx->cst);
    return GDWD_OK;
  };
  // Pageable source: host threads copy block b into a page-locked ring
  // (UP_NSLOT slots) while the DMA engine drains the blocks before it; the
  // DMA of a block is queued as soon as every thread has delivered its share.
  UploadAux* ax = (UploadAux*)ctx->up_aux;
  const size_t slot_b = (size_t)mb * row_b;
  std::vector<std::thread> workers;
  std::atomic<int> allowed{UP_NSLOT};  // blocks [0, allowed) may be staged (their slot is free)
  std::unique_ptr<std::atomic<int>[]> staged(new std::atomic<int>[gdwd_ctx::UP_MAXB]);
  unsigned nthr = 1;
  struct Joiner {  // error returns must not leave running threads behind
    std::vector<std::thread>& w;
    std::atomic<int>& allowed;
    ~Joiner() {
      allowed.store(1 << 30, std::memory_order_release);
      for (auto& t : w)
        if (t.joinable()) t.join();
    }
  } joiner{workers, allowed};
  if (!pinned) {
    if (ax->pin_bytes < UP_NSLOT * slot_b) {
      if (ax->pin) cudaFreeHost(ax->pin);
      ax->pin = nullptr;
      ax->pin_bytes = 0;
      if (cudaMallocHost(&ax->pin, UP_NSLOT * slot_b) != cudaSuccess) {
        cudaGetLastError();
        ax->pin = nullptr;
        return UP_NO_STAGING;  // nothing queued yet: the caller takes the plain copy
      }
      ax->pin_bytes = UP_NSLOT * slot_b;
    }
    for (int b = 0; b < gdwd_ctx::UP_MAXB; ++b) staged[b].store(0, std::memory_order_relaxed);
    nthr = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const char* src0 = (const char*)samples;
    char* ring = (char*)ax->pin;
    const int64_t* rbp = rb;
    for (unsigned t = 0; t < nthr; ++t)
      workers.emplace_back([=, &allowed, &staged] {
        for (int b = 0; b < nblk; ++b) {
          while (allowed.load(std::memory_order_acquire) <= b) std::this_thread::yield();
          const size_t bytes = (size_t)(rbp[b + 1] - rbp[b]) * row_b;
          const size_t lo = bytes * t / nthr / 64 * 64, hi = t + 1 == nthr ? bytes : bytes * (t + 1) / nthr / 64 * 64;
          memcpy(ring + (size_t)(b % UP_NSLOT) * slot_b + lo, src0 + (size_t)rbp[b] * row_b + lo, hi - lo);
          staged[b].fetch_add(1, std::memory_order_release);
        }
      });
  } else {
    // page-locked source: every copy is queued before any compute launch, so
    // the copy engine never waits for the host
    for (int b = 0; b < nblk; ++b) RC(queue_copy(b, samples + rb[b] * d));
  }
  const auto t_h1 = std::chrono::steady_clock::now();
  for (int b = 0; b < nblk; ++b) {
    const int64_t r0 = rb[b], r1 = rb[b + 1];
    if (!pinned) {
      while (staged[b].load(std::memory_order_acquire) < (int)nthr) std::this_thread::yield();
      RC(queue_copy(b, ax->pin + (size_t)(b % UP_NSLOT) * (slot_b / sizeof(double))));
    }
    CK(cudaStreamWaitEvent(ctx->gst, ctx->up_ev[b], 0));
    CK(gram_rowblock(ctx->Zs, ld, d, r0, r1, ctx->kmat.p, ldk, G, ldk, mu2, ctx->gram_ws.p, ctx->gst));
    if (tmark) tev(1, b, ctx->gst);
    if (factor) {
      CK(cudaEventRecord(ctx->gr_ev[b], ctx->gst));
      CK(cudaStreamWaitEvent(ctx->fst, ctx->gr_ev[b], 0));
      CK(bordered_chol_step(G, Wi, T, ctx->fac.p, ldk, r0, r1, ctx->dinfo, ctx->fst, ctx->sst, ctx->ast,
                            T + (size_t)n * ldk, bws));
      if (tmark) tev(2, b, ctx->fst);
      if (tmark) tev(3, b, ctx->ast);
    }
    if (!pinned && b + 1 >= UP_NSLOT) {  // block b + 1 reuses the slot of block b + 1 - UP_NSLOT
      CK(cudaEventSynchronize(ctx->up_ev[b + 1 - UP_NSLOT]));
      allowed.store(b + 2, std::memory_order_release);
    }
  }
  const auto t_h2 = std::chrono::steady_clock::now();
  ctx->up_pending = true;
  ctx->n = n;
  ctx->d = d;
  ctx->ldz = ld;
  ctx->has_dense = true;
  ctx->has_problem = false;
  ctx->data_gen++;
  ctx->zs_gen++;
  ctx->k_gen = ctx->zs_gen;
  RC(ensure_scratch(ctx, n, d));  // may synchronise st: before st starts waiting for the copies
  CK(cudaStreamWaitEvent(ctx->st, ctx->up_ev[nblk - 1], 0));
  run_vm(ctx, OpSumSq{ctx->Zs, d, ld, ctx->fro2_d}, n * d, "vmap_fro2", false);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ctx->fro2_h, ctx->fro2_d, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  ctx->fro2_pending = true;
  // everything later on st sees the whole K (and G^{-1})
  CK(cudaEventRecord(ctx->gram_ev, ctx->gst));
  CK(cudaStreamWaitEvent(ctx->st, ctx->gram_ev, 0));
  if (factor) {
    CK(mirror_lower(ctx->fac.p, ldk, n, ctx->ast));
    CK(cudaEventRecord(ctx->pf_ev, ctx->ast));
    CK(cudaStreamWaitEvent(ctx->st, ctx->pf_ev, 0));
    ctx->pf_gen = ctx->zs_gen;
    ctx->pf_mu2 = mu2;
  }
  // the host buffer is only borrowed for the call: wait for the copies (the
  // Gram rows, the factor chain and the norm may still be running)
  const auto t_h3 = std::chrono::steady_clock::now();
  finish_upload(ctx);
  if (tmark) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t_h4 = std::chrono::steady_clock::now();
    for (cudaStream_t x : {ctx->gst, ctx->fst, ctx->ast}) cudaStreamSynchronize(x);
    const auto t_h5 = std::chrono::steady_clock::now();
    fprintf(stderr, "[upload timing] streams/events %.3f, buffers %.3f ms\n", ms(t_pre0, t_pre1), ms(t_pre1, t_h0));
    fprintf(stderr, "[upload timing] queue copies %.3f, queue compute %.3f, rest %.3f, wait copies %.3f, "
            "compute tail after the last byte %.3f ms (%d blocks of %lld)\n", ms(t_h0, t_h1), ms(t_h1, t_h2),
            ms(t_h2, t_h3), ms(t_h3, t_h4), ms(t_h4, t_h5), nblk, (long long)mb);
    const char* names[4] = {"copy", "gram", "chain", "ginv"};
    for (int l = 0; l < 4; ++l) {
      fprintf(stderr, "[upload timeline] %-5s", names[l]);
      for (cudaEvent_t e : tl[l]) {
        float t = 0.f;
        cudaEventElapsedTime(&t, tl0, e);
        fprintf(stderr, " %.2f", t);
        cudaEventDestroy(e);
      }
      fprintf(stderr, "\n");
    }
    cudaEventDestroy(tl0);
  }
  return GDWD_OK;
}

// Pageable [n][d] source outside the sample-space regimes: the same staging
// as upload_dense_pipelined without the factorisation -- host threads copy
// blocks of rows into the pooled page-locked ring while the DMA engine
// drains the blocks before them (a pageable cudaMemcpy2D runs at ~11 GB/s on
// these hosts, the staged copy at the host threads' ~35 GB/s).
// `pinned`: the source is page-locked (no staging, block-wise DMA).  `dgram`:
// the DIRECT regime's d x d Gram Z~ Z~^T (subsolvers.py:76) is summed block by
// block on a second stream as the rows land (into fac, the (d+1) x (d+1)
// layout build_factor completes), so only the last block's share is left
// after the copy.
static int upload_rows_staged(gdwd_ctx* ctx, const double* samples, int64_t d, int64_t n, int64_t ld, bool pinned,
                              bool dgram) {
  UploadAux* ax = upload_aux_acquire(ctx->device);
  if (!ax) return set_err(ctx, GDWD_ERR_CUDA, "upload streams");
  struct Release {
    UploadAux* a;
    ~Release() { upload_aux_release(a); }  // synchronises its streams
  } rel{ax};
  const size_t row_b = (size_t)d * sizeof(double);
  const int64_t mb = std::max<int64_t>(1, (int64_t)(((size_t)16 << 20) / row_b));
  const size_t slot_b = (size_t)mb * row_b;
  const int nblk = (int)((n + mb - 1) / mb);
  if (!pinned && ax->pin_bytes < UP_NSLOT * slot_b) {
    if (ax->pin) cudaFreeHost(ax->pin);
    ax->pin = nullptr;
    ax->pin_bytes = 0;
    if (cudaMallocHost(&ax->pin, UP_NSLOT * slot_b) != cudaSuccess) {
      cudaGetLastError();
      ax->pin = nullptr;
      return UP_NO_STAGING;  // no page-locked memory to be had: the caller takes the plain copy
    }
    ax->pin_bytes = UP_NSLOT * slot_b;
  }
  cudaStream_t cst = ax->s[0], gst = ax->s[1];
  const int64_t ldm = (d + 2) / 2 * 2;  // DIRECT: m = d + 1 rows of stride ((m + 1) / 2) * 2
  if (dgram) {
    CK(ctx->fac.ensure((size_t)(d + 1) * ldm));
    CK(ctx->facw.ensure(std::max<size_t>((size_t)gram_workspace_doubles(d, mb), (size_t)2 * (d + 1) * ldm)));
    CK(cudaMemsetAsync(ctx->fac.p, 0, (size_t)(d + 1) * ldm * sizeof(double), ctx->st));
  }
  CK(cudaStreamSynchronize(ctx->st));  // Zs is allocated (and its pad zeroed) on st
  std::vector<std::thread> workers;
  std::atomic<int> allowed{UP_NSLOT};
  std::unique_ptr<std::atomic<int>[]> staged(new std::atomic<int>[nblk]);
  for (int b = 0; b < nblk; ++b) staged[b].store(0, std::memory_order_relaxed);
  struct Joiner {
    std::vector<std::thread>& w;
    std::atomic<int>& allowed;
    ~Joiner() {
      allowed.store(1 << 30, std::memory_order_release);
      for (auto& t : w)
        if (t.joinable()) t.join();
    }
  } joiner{workers, allowed};
  const unsigned nthr = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const char* src0 = (const char*)samples;
  char* ring = (char*)ax->pin;
  if (!pinned)
    for (unsigned t = 0; t < nthr; ++t)
      workers.emplace_back([=, &allowed, &staged] {
        for (int b = 0; b < nblk; ++b) {
          while (allowed.load(std::memory_order_acquire) <= b) std::this_thread::yield();
          const int64_t r0 = (int64_t)b * mb, r1 = std::min<int64_t>(n, r0 + mb);
          const size_t bytes = (size_t)(r1 - r0) * row_b;
          const size_t lo = bytes * t / nthr / 64 * 64, hi = t + 1 == nthr ? bytes : bytes * (t + 1) / nthr / 64 * 64;
          memcpy(ring + (size_t)(b % UP_NSLOT) * slot_b + lo, src0 + (size_t)r0 * row_b + lo, hi - lo);
          staged[b].fetch_add(1, std::memory_order_release);
        }
      });
  for (int b = 0; b < nblk; ++b) {
    const int64_t r0 = (int64_t)b * mb, r1 = std::min<int64_t>(n, r0 + mb);
    const char* from = src0 + (size_t)r0 * row_b;
    if (!pinned) {
      while (staged[b].load(std::memory_order_acquire) < (int)nthr) std::this_thread::yield();
      from = ring + (size_t)(b % UP_NSLOT) * slot_b;
    }
    CK(cudaMemcpy2DAsync(ctx->Zs + r0 * ld, ld * sizeof(double), from, row_b, row_b, r1 - r0, cudaMemcpyHostToDevice,
                         cst));
    CK(cudaEventRecord(ax->e[b % UP_NSLOT], cst));
    if (dgram) {  // + Z~[:, block] Z~[:, block]^T, blocks in order (fixed summation order)
      CK(cudaStreamWaitEvent(gst, ax->e[b % UP_NSLOT], 0));
      CK(gram_syrk(ctx->Zs + r0 * ld, r1 - r0, d, ld, true, 1.0, 0.0, ctx->fac.p, ldm, ctx->facw.p, gst, b > 0));
    }
    if (!pinned && b + 1 >= UP_NSLOT) {  // block b + 1 reuses the slot of block b + 1 - UP_NSLOT
      CK(cudaEventSynchronize(ax->e[(b + 1 - UP_NSLOT) % UP_NSLOT]));
      allowed.store(b + 2, std::memory_order_release);
    }
  }
  CK(cudaStreamSynchronize(cst));
  if (dgram) {
    // the Gram's tail may still be running: later work on st waits for it
    CK(cudaEventRecord(ax->e[UP_NSLOT], gst));
    CK(cudaStreamWaitEvent(ctx->st, ax->e[UP_NSLOT], 0));
    ctx->dg_gen = ctx->zs_gen + 1;  // the caller bumps zs_gen for this upload
  }
  return GDWD_OK;
}

// Large pageable host array -> device through the pooled page-locked ring
// (host threads fill a slot while the DMA engine drains the ones before it);
// small ones by the plain synchronous copy.  Returns when the data has landed.
static int h2d_staged(gdwd_ctx* ctx, void* dst, const void* src, size_t bytes) {
  const size_t slot_b = (size_t)16 << 20;
  UploadAux* ax = bytes >= 2 * slot_b && !getenv("GDWD_UPLOAD") ? upload_aux_acquire(ctx->device) : nullptr;
  if (ax && ax->pin_bytes < UP_NSLOT * slot_b) {
    if (ax->pin) cudaFreeHost(ax->pin);
    ax->pin = nullptr;
    ax->pin_bytes = 0;
    if (cudaMallocHost(&ax->pin, UP_NSLOT * slot_b) == cudaSuccess) {
      ax->pin_bytes = UP_NSLOT * slot_b;
    } else {
      cudaGetLastError();
      ax->pin = nullptr;
      upload_aux_release(ax);
      ax = nullptr;
    }
  }
  if (!ax) {
    CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    CK(cudaStreamSynchronize(cudaStreamLegacy));  // staged by the driver: let it land
    return GDWD_OK;
  }
  struct Release {
    UploadAux* a;
    ~Release() { upload_aux_release(a); }
  } rel{ax};
  const int nblk = (int)((bytes + slot_b - 1) / slot_b);
  cudaStream_t cst = ax->s[0];
  std::vector<std::thread> workers;
  std::atomic<int> allowed{UP_NSLOT};
  std::unique_ptr<std::atomic<int>[]> staged(new std::atomic<int>[nblk]);
  for (int b = 0; b < nblk; ++b) staged[b].store(0, std::memory_order_relaxed);
  struct Joiner {
    std::vector<std::thread>& w;
    std::atomic<int>& allowed;
    ~Joiner() {
      allowed.store(1 << 30, std::memory_order_release);
      for (auto& t : w)
        if (t.joinable()) t.join();
    }
  } joiner{workers, allowed};
  const unsigned nthr = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const char* src0 = (const char*)src;
  char* ring = (char*)ax->pin;
  for (unsigned t = 0; t < nthr; ++t)
    workers.emplace_back([=, &allowed, &staged] {
      for (int b = 0; b < nblk; ++b) {
        while (allowed.load(std::memory_order_acquire) <= b) std::this_thread::yield();
        const size_t off = (size_t)b * slot_b, len = std::min(slot_b, bytes - off);
        const size_t lo = len * t / nthr / 64 * 64, hi = t + 1 == nthr ? len : len * (t + 1) / nthr / 64 * 64;
        memcpy(ring + (size_t)(b % UP_NSLOT) * slot_b + lo, src0 + off + lo, hi - lo);
        staged[b].fetch_add(1, std::memory_order_release);
      }
    });
  for (int b = 0; b < nblk; ++b) {
    const size_t off = (size_t)b * slot_b, len = std::min(slot_b, bytes - off);
    while (staged[b].load(std::memory_order_acquire) < (int)nthr) std::this_thread::yield();
    CK(cudaMemcpyAsync((char*)dst + off, ring + (size_t)(b % UP_NSLOT) * slot_b, len, cudaMemcpyHostToDevice, cst));
    CK(cudaEventRecord(ax->e[b % UP_NSLOT], cst));
    if (b + 1 >= UP_NSLOT) {
      CK(cudaEventSynchronize(ax->e[(b + 1 - UP_NSLOT) % UP_NSLOT]));
      allowed.store(b + 2, std::memory_order_release);
    }
  }
  CK(cudaStreamSynchronize(cst));
  return GDWD_OK;
}

int gdwd_upload_hint(gdwd_ctx* ctx, int32_t backend, double mu) {
  if (!ctx || !(mu > 0.0) || backend < GDWD_BACKEND_AUTO || backend > GDWD_BACKEND_ITERATIVE)
    return set_err(ctx, GDWD_ERR_VALUE, "bad upload hint");
  ctx->hint_backend = backend;
  ctx->hint_mu = mu;
  return GDWD_OK;
}

int gdwd_upload_dense(gdwd_ctx* ctx, const double* samples, int64_t d, int64_t n) {
  Range nvtx_range("gdwd_upload_dense");
  if (!ctx || !samples || d < 1 || n < 1) return set_err(ctx, GDWD_ERR_VALUE, "bad dense upload arguments");
  CK(cudaSetDevice(ctx->device));
  free_sparse(ctx);
  const int64_t ld = (d + 1) / 2 * 2;
  dfree(ctx->Zs, ctx->st);
  ctx->Zs = nullptr;
  CK(dmalloc((void**)&ctx->Zs, (size_t)n * ld * sizeof(double), ctx->st));
  if (ld != d) CK(cudaMemsetAsync(ctx->Zs, 0, (size_t)n * ld * sizeof(double), ctx->st));
  // Sample-space regimes (n <= 2500, n <= d: SMW2, DIRECT with 2n <= d) with
  // a page-locked source: the matrix is copied in blocks of samples
  // (contiguous rows) on a copy stream; as each block lands, a second stream
  // forms its rows of the n x n Gram K = Z~^T Z~ and of G = K/mu^2 + I, and a
  // third advances the bordered Cholesky factor and L^{-1} by that block, so
  // K, G^{-1} are ready shortly after the last byte (upload_dense_pipelined).
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, samples) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  finish_upload(ctx);
  const int hk = ctx->hint_backend == GDWD_BACKEND_AUTO ? select_kind(n, d) : ctx->hint_backend;
  // (an ITERATIVE hint -- also what a shard of a multi-GPU solve passes -- means
  // no Gram is needed at all: plain copy)
  if (n <= 2500 && n <= d && d >= 64 && !sharded(ctx) && !getenv("GDWD_UPLOAD") && hk != GDWD_BACKEND_ITERATIVE &&
      (pinned || (size_t)n * d >= ((size_t)1 << 20))) {  // pageable: worth the staging threads from ~8 MB
    const int rc = upload_dense_pipelined(ctx, samples, d, n, ld, pinned);
    if (rc != UP_NO_STAGING) return rc;
  }
  // DIRECT's own regime (and not the sample-space form of it): sum the d x d Gram during the copy
  const bool dgram = hk == GDWD_BACKEND_DIRECT && 2 * n > d && d <= 8192 && n >= 4 * d && !sharded(ctx) &&
                     getenv("GDWD_UPLOAD_FACTOR") == nullptr;
  int rc = UP_NO_STAGING;
  if (!getenv("GDWD_UPLOAD") && (size_t)n * d >= ((size_t)1 << 20) && (!pinned || dgram))
    rc = upload_rows_staged(ctx, samples, d, n, ld, pinned, dgram);
  if (rc == UP_NO_STAGING) rc = upload_rows(ctx, samples, d, n, ld);
  RC(rc);
  ctx->zs_gen++;
  ctx->n = n;
  ctx->d = d;
  ctx->ldz = ld;
  ctx->has_dense = true;
  ctx->has_problem = false;
  ctx->data_gen++;
  RC(ensure_scratch(ctx, n, d));
  return compute_fro2(ctx, ctx->Zs, n, d, ld);
}

int gdwd_upload_csc(gdwd_ctx* ctx, const int64_t* colptr, const int64_t* rowidx, const double* values, int64_t d,
                    int64_t n) {
  Range nvtx_range("gdwd_upload_csc");
  if (!ctx || !colptr || d < 1 || n < 1) return set_err(ctx, GDWD_ERR_VALUE, "bad CSC upload arguments");
  const int64_t nnz = colptr[n];
  if (colptr[0] != 0 || nnz < 0) return set_err(ctx, GDWD_ERR_VALUE, "colptr endpoints do not match stored entries");
  if (nnz >= ((int64_t)1 << 31)) return set_err(ctx, GDWD_ERR_UNSUPPORTED, "nnz >= 2^31 per shard");
  if (nnz > 0 && (!rowidx || !values)) return set_err(ctx, GDWD_ERR_VALUE, "null CSC arrays");
  const bool tmark = getenv("GDWD_SETUP_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto hmark = [&](const char* what) {
    if (!tmark) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[upload timing] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  // validate + transpose to CSR on the host (counting sort keeps sample order
  // within each feature row, so row sums accumulate like np.bincount), on
  // all host cores: threads own contiguous sample ranges, per-thread row
  // histograms give every (thread, row) its output offset, so the scatter
  // keeps sample order.  The error reported is the first one in sample order
  // (a sample's colptr before its indices), as a sequential pass finds it.
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>({16, (int64_t)std::thread::hardware_concurrency(), n / 1024 + 1}));
  auto par = [&](auto&& fn) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back([&, t]() { fn(t, n * t / T, n * (t + 1) / T); });
    for (auto& x : th) x.join();
  };
  std::vector<int64_t> bad_ptr(T, n), bad_idx(T, n);
  par([&](int t, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i)
      if (colptr[i + 1] < colptr[i]) {
        bad_ptr[t] = i;
        break;
      }
  });
  const int64_t first_ptr = *std::min_element(bad_ptr.begin(), bad_ptr.end());
  std::vector<std::vector<int64_t>> hist(T);
  RawBuf<int> ci32((size_t)nnz);
  par([&](int t, int64_t i0, int64_t i1) {
    hist[t].assign(d, 0);
    int64_t* h = hist[t].data();
    for (int64_t i = i0; i < std::min(i1, first_ptr); ++i)
      for (int64_t k = colptr[i]; k < colptr[i + 1]; ++k) {
        const int64_t r = rowidx[k];
        if (r < 0 || r >= d) {
          bad_idx[t] = i;
          return;
        }
        h[r]++;
        ci32[k] = (int)r;
      }
  });
  const int64_t first_idx = *std::min_element(bad_idx.begin(), bad_idx.end());
  if (first_idx < n && first_idx < first_ptr) return set_err(ctx, GDWD_ERR_VALUE, "row index out of bounds");
  if (first_ptr < n) return set_err(ctx, GDWD_ERR_VALUE, "colptr must be nondecreasing");
  std::vector<int64_t> rp(d + 1, 0);
  for (int64_t j = 0; j < d; ++j) {  // row starts, then each thread's offset within the row
    int64_t o = rp[j];
    for (int t = 0; t < T; ++t) {
      const int64_t c = hist[t][j];
      hist[t][j] = o;
      o += c;
    }
    rp[j + 1] = o;
  }
  RawBuf<int> cidx((size_t)nnz);
  RawBuf<double> cval((size_t)nnz);
  par([&](int t, int64_t i0, int64_t i1) {
    int64_t* fillp = hist[t].data();
    for (int64_t i = i0; i < i1; ++i)
      for (int64_t k = colptr[i]; k < colptr[i + 1]; ++k) {
        const int64_t pos = fillp[rowidx[k]]++;
        cidx[pos] = (int)i;
        cval[pos] = values[k];
      }
  });
  hmark("validate + CSR transpose");
  CK(cudaSetDevice(ctx->device));
  free_sparse(ctx);
  dfree(ctx->Zs, ctx->st);
  ctx->Zs = nullptr;
  ctx->zs_gen++;
  ctx->has_dense = false;
  const size_t nz = (size_t)std::max<int64_t>(nnz, 1);
  CK(dmalloc((void**)&ctx->csc_ptr, (n + 1) * sizeof(int64_t), ctx->st));
  CK(dmalloc((void**)&ctx->csr_ptr, (d + 1) * sizeof(int64_t), ctx->st));
  CK(dmalloc((void**)&ctx->csc_idx, nz * sizeof(int), ctx->st));
  CK(dmalloc((void**)&ctx->csr_idx, nz * sizeof(int), ctx->st));
  CK(dmalloc((void**)&ctx->csc_val, nz * sizeof(double), ctx->st));
  CK(dmalloc((void**)&ctx->csr_val, nz * sizeof(double), ctx->st));
  CK(cudaMemcpy(ctx->csc_ptr, colptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->csr_ptr, rp.data(), (d + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  if (nnz > 0) {
    RC(h2d_staged(ctx, ctx->csc_idx, ci32.data(), nnz * sizeof(int)));
    RC(h2d_staged(ctx, ctx->csr_idx, cidx.data(), nnz * sizeof(int)));
    RC(h2d_staged(ctx, ctx->csc_val, values, nnz * sizeof(double)));
    RC(h2d_staged(ctx, ctx->csr_val, cval.data(), nnz * sizeof(double)));
  }
  // feature-blocked CSC: parts of S samples (one CTA each, 2 per SM) x
  // feature blocks of FB_COLS; within (part, block) the samples in order,
  // each sample's entries in CSC order, 16-bit block-local feature indices
  hmark("CSC + CSR to device");
  // feature-blocked sliced ELL (spops.cuh FbView): parts of S samples (one
  // CTA each) x feature blocks of FB_COLS; per (part, block) the samples
  // sorted by entry count (descending, then index) in slices of 32, entries
  // column-major within a slice, 16-bit block-local indices
  const int fb_S = (int)((n + FB_PARTS - 1) / FB_PARTS);
  if (nnz > 0 && fb_S < 65535 && (size_t)(FB_COLS + fb_S) * sizeof(double) <= FB_SMEM_MAX) {
    const int parts = FB_PARTS, S = fb_S, Q = (S + 31) / 32;
    const int nb = (int)((d + FB_COLS - 1) / FB_COLS);
    std::vector<int> sbase((size_t)parts * nb * (Q + 1));
    std::vector<unsigned short> perm((size_t)parts * nb * 32 * Q, 0xffff), cnt((size_t)parts * nb * 32 * Q, 0);
    // parts are independent: built on all host cores into per-part arrays,
    // slice starts relative to the part, then concatenated
    std::vector<std::vector<unsigned short>> pidx(parts);
    std::vector<std::vector<double>> pval(parts);
    auto build_part = [&](int p) {
      const int64_t a = std::min<int64_t>(n, (int64_t)p * S), z = std::min<int64_t>(n, a + S);
      std::vector<int> start((size_t)nb * (S + 1), 0);
      for (int64_t i = a; i < z; ++i)
        for (int64_t k = colptr[i]; k < colptr[i + 1]; ++k) start[(size_t)(rowidx[k] / FB_COLS) * (S + 1) + (i - a) + 1]++;
      for (size_t t = 1; t < start.size(); ++t) start[t] += start[t - 1];
      const int64_t pn = colptr[z] - colptr[a];
      std::vector<unsigned short> lidx((size_t)pn);
      std::vector<double> lval((size_t)pn);
      {
        std::vector<int> cur(start);
        for (int64_t i = a; i < z; ++i)
          for (int64_t k = colptr[i]; k < colptr[i + 1]; ++k) {
            const int64_t r = rowidx[k], f = r / FB_COLS;
            const int at = cur[(size_t)f * (S + 1) + (i - a)]++;
            lidx[at] = (unsigned short)(r - f * FB_COLS);
            lval[at] = values[k];
          }
      }
      std::vector<int> ord(S);
      auto& sv = pval[p];
      auto& si = pidx[p];
      for (int f = 0; f < nb; ++f) {
        const int* st = &start[(size_t)f * (S + 1)];
        auto count = [&](int ls) { return ls < (int)(z - a) ? st[ls + 1] - st[ls] : 0; };
        for (int ls = 0; ls < S; ++ls) ord[ls] = ls;
        std::sort(ord.begin(), ord.end(), [&](int x, int y) {
          const int cx = count(x), cy = count(y);
          return cx != cy ? cx > cy : x < y;
        });
        const size_t pf = (size_t)p * nb + f;
        for (int q = 0; q < Q; ++q) {
          sbase[pf * (Q + 1) + q] = (int)sv.size();
          const int len = count(ord[32 * q]);
          const size_t b = sv.size();
          sv.resize(b + (size_t)32 * len, 0.0);
          si.resize(b + (size_t)32 * len, 0);
          for (int l = 0; l < 32 && 32 * q + l < S; ++l) {
            const int ls = ord[32 * q + l], c = count(ls);
            perm[pf * 32 * Q + 32 * q + l] = ls < (int)(z - a) ? (unsigned short)ls : 0xffff;
            cnt[pf * 32 * Q + 32 * q + l] = (unsigned short)c;
            for (int j = 0; j < c; ++j) {
              sv[b + (size_t)32 * j + l] = lval[st[ls] + j];
              si[b + (size_t)32 * j + l] = lidx[st[ls] + j];
            }
          }
        }
        sbase[pf * (Q + 1) + Q] = (int)sv.size();
      }
    };
    {
      const unsigned nthr = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nthr; ++t)
        th.emplace_back([&, t]() {
          for (int p = (int)t; p < parts; p += (int)nthr) build_part(p);
        });
      for (auto& x : th) x.join();
    }
    hmark("sliced ELL build (threads)");
    std::vector<size_t> poff(parts + 1, 0);
    for (int p = 0; p < parts; ++p) poff[p + 1] = poff[p] + pval[p].size();
    for (int p = 0; p < parts; ++p)
      for (size_t t = (size_t)p * nb * (Q + 1); t < (size_t)(p + 1) * nb * (Q + 1); ++t) sbase[t] += (int)poff[p];
    if (poff[parts] < ((size_t)1 << 31)) {
      const size_t ne = std::max<size_t>(poff[parts], 1);
      CK(dmalloc((void**)&ctx->fb_ptr, sbase.size() * sizeof(int), ctx->st));
      CK(dmalloc((void**)&ctx->fb_perm, perm.size() * sizeof(unsigned short), ctx->st));
      CK(dmalloc((void**)&ctx->fb_cnt, cnt.size() * sizeof(unsigned short), ctx->st));
      CK(dmalloc((void**)&ctx->fb_idx, ne * sizeof(unsigned short), ctx->st));
      CK(dmalloc((void**)&ctx->fb_val, ne * sizeof(double), ctx->st));
      CK(cudaMemcpy(ctx->fb_ptr, sbase.data(), sbase.size() * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->fb_perm, perm.data(), perm.size() * sizeof(unsigned short), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->fb_cnt, cnt.data(), cnt.size() * sizeof(unsigned short), cudaMemcpyHostToDevice));
      {
        // the parts' arrays gathered by all threads, then one staged copy each
        // (592 separate pageable copies ran at ~11 GB/s)
        RawBuf<double> allv(ne);
        RawBuf<unsigned short> alli(ne);
        par([&](int t, int64_t, int64_t) {
          for (int p = t; p < parts; p += T)
            if (!pval[p].empty()) {
              memcpy(allv.data() + poff[p], pval[p].data(), pval[p].size() * sizeof(double));
              memcpy(alli.data() + poff[p], pidx[p].data(), pidx[p].size() * sizeof(unsigned short));
            }
        });
        if (poff[parts] > 0) {
          RC(h2d_staged(ctx, ctx->fb_val, allv.data(), poff[parts] * sizeof(double)));
          RC(h2d_staged(ctx, ctx->fb_idx, alli.data(), poff[parts] * sizeof(unsigned short)));
        }
      }
      ctx->fb_nb = nb;
      ctx->fb_parts = parts;
      ctx->fb_S = S;
      ctx->fb_Q = Q;
      ctx->fb_entries = (int64_t)poff[parts];
    }
    hmark("sliced ELL concat + to device");
  }
  // sample-blocked sliced ELL for Z~ t (spops.cuh SbView): blocks of SB_S
  // samples; per block every feature, sorted by its entry count in the block
  // (descending, then index), 32 per slice, entries column-major in sample
  // order with 16-bit block-local sample indices
  if (nnz > 0 && d < ((int64_t)1 << 31) / 32) {
    const int nb = (int)((n + SB_S - 1) / SB_S);
    const int nslpb = (int)((d + 31) / 32);
    const int64_t nsl = (int64_t)nb * nslpb;
    std::vector<int> hh((size_t)nsl, 0), pp((size_t)nsl * 32, -1);
    std::vector<int64_t> bb((size_t)nsl + 1, 0);
    // per block, per feature: the entry range of row j inside the block
    std::vector<int64_t> bnd((size_t)(nb + 1) * d);
    par([&](int t, int64_t, int64_t) {
      for (int64_t j = d * t / T; j < d * (t + 1) / T; ++j) {
        int64_t k = rp[j];
        for (int b = 0; b <= nb; ++b) {
          const int64_t lim = std::min<int64_t>(n, (int64_t)b * SB_S);
          while (k < rp[j + 1] && cidx[k] < lim) ++k;
          bnd[(size_t)b * d + j] = k;
        }
      }
    });
    // slice heights and orders per block (threads over blocks)
    {
      std::vector<std::thread> th;
      const int nthr = std::max(1, std::min(nb, T));
      for (int t = 0; t < nthr; ++t)
        th.emplace_back([&, t]() {
          std::vector<int> ord(d);
          for (int b = t; b < nb; b += nthr) {
            const int64_t* lo = &bnd[(size_t)b * d];
            const int64_t* hi = &bnd[(size_t)(b + 1) * d];
            for (int64_t j = 0; j < d; ++j) ord[j] = (int)j;
            std::sort(ord.begin(), ord.end(), [&](int x, int y) {
              const int64_t cx = hi[x] - lo[x], cy = hi[y] - lo[y];
              return cx != cy ? cx > cy : x < y;
            });
            for (int q = 0; q < nslpb; ++q) {
              const int64_t sl = (int64_t)b * nslpb + q;
              hh[sl] = (int)(hi[ord[32 * q]] - lo[ord[32 * q]]);
              for (int l = 0; l < 32 && 32 * q + l < d; ++l) pp[sl * 32 + l] = ord[32 * q + l];
            }
          }
        });
      for (auto& x : th) x.join();
    }
    for (int64_t sl = 0; sl < nsl; ++sl) bb[sl + 1] = bb[sl] + 32 * (int64_t)hh[sl];
    const int64_t ne = bb[nsl];
    if (ne < ((int64_t)1 << 31)) {
      RawBuf<double> sv((size_t)std::max<int64_t>(ne, 1));
      RawBuf<unsigned short> si((size_t)std::max<int64_t>(ne, 1));
      par([&](int t, int64_t, int64_t) {  // pad entries must read as zero: cleared in parallel
        const size_t tot = sv.size(), lo = tot * t / T, hi = tot * (t + 1) / T;
        memset(sv.data() + lo, 0, (hi - lo) * sizeof(double));
        memset(si.data() + lo, 0, (hi - lo) * sizeof(unsigned short));
      });
      par([&](int t, int64_t, int64_t) {
        for (int64_t sl = nsl * t / T; sl < nsl * (t + 1) / T; ++sl) {
          const int b = (int)(sl / nslpb);
          for (int l = 0; l < 32; ++l) {
            const int j = pp[sl * 32 + l];
            if (j < 0) continue;
            const int64_t lo = bnd[(size_t)b * d + j], hi = bnd[(size_t)(b + 1) * d + j];
            for (int64_t e = 0; e < hi - lo; ++e) {
              sv[bb[sl] + 32 * e + l] = cval[lo + e];
              si[bb[sl] + 32 * e + l] = (unsigned short)(cidx[lo + e] - (int64_t)b * SB_S);
            }
          }
        }
      });
      // SB_CHUNKS chunks of consecutive slices with equal shares of entries
      // (+ 32 per slice for its fixed cost)
      std::vector<int> ch(SB_CHUNKS + 1, (int)nsl);
      {
        const double tot = (double)ne + 32.0 * (double)nsl;
        int c = 1;
        ch[0] = 0;
        double acc = 0.0;
        for (int64_t sl = 0; sl < nsl && c < SB_CHUNKS; ++sl) {
          acc += 32.0 * hh[sl] + 32.0;
          while (c < SB_CHUNKS && acc >= tot * c / SB_CHUNKS) ch[c++] = (int)(sl + 1);
        }
        for (; c < SB_CHUNKS; ++c) ch[c] = (int)nsl;
      }
      CK(dmalloc((void**)&ctx->sb_val, sv.size() * sizeof(double), ctx->st));
      CK(dmalloc((void**)&ctx->sb_idx, si.size() * sizeof(unsigned short), ctx->st));
      CK(dmalloc((void**)&ctx->sb_base, bb.size() * sizeof(int64_t), ctx->st));
      CK(dmalloc((void**)&ctx->sb_h, hh.size() * sizeof(int), ctx->st));
      CK(dmalloc((void**)&ctx->sb_perm, pp.size() * sizeof(int), ctx->st));
      CK(dmalloc((void**)&ctx->sb_chunk, ch.size() * sizeof(int), ctx->st));
      RC(h2d_staged(ctx, ctx->sb_val, sv.data(), sv.size() * sizeof(double)));
      RC(h2d_staged(ctx, ctx->sb_idx, si.data(), si.size() * sizeof(unsigned short)));
      CK(cudaMemcpy(ctx->sb_base, bb.data(), bb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->sb_h, hh.data(), hh.size() * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->sb_perm, pp.data(), pp.size() * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->sb_chunk, ch.data(), ch.size() * sizeof(int), cudaMemcpyHostToDevice));
      CK(ctx->sb_part.ensure((size_t)nb * d * 2));
      ctx->sb_nb = nb;
      ctx->sb_nslpb = nslpb;
      ctx->sb_entries = ne;
    }
    hmark("sample-blocked sliced ELL");
  }
  // the synchronous copies above are staged through the legacy stream, which
  // the (non-blocking) solve stream does not wait for: let them land
  CK(cudaStreamSynchronize(cudaStreamLegacy));
  CK(ctx->tbuf.ensure((size_t)2 * n + 2));
  ctx->n = n;
  ctx->d = d;
  ctx->ldz = (d + 1) / 2 * 2;
  ctx->nnz = nnz;
  ctx->has_sparse = true;
  ctx->has_problem = false;
  ctx->data_gen++;
  RC(ensure_scratch(ctx, n, d));
  if (nnz > 0) return compute_fro2(ctx, ctx->csc_val, 1, nnz, nnz);
  ctx->fro2_pending = false;
  ctx->fro2 = 0.0;
  return GDWD_OK;
}

// DIRECT / SMW2 on sparse input: materialise the dense sample-major copy once
// (the Gram and every product then take the dense path)
static int densify(gdwd_ctx* ctx) {
  if (ctx->has_dense) return GDWD_OK;
  const int64_t n = ctx->n, ld = ctx->ldz;
  size_t freeb = 0, totb = 0;
  CK(cudaMemGetInfo(&freeb, &totb));
  if ((double)n * ld * 8.0 > 0.8 * (double)freeb)
    return set_err(ctx, GDWD_ERR_UNSUPPORTED, "dense copy of the sparse matrix does not fit for this backend");
  CK(dmalloc((void**)&ctx->Zs, (size_t)n * ld * sizeof(double), ctx->st));
  CK(cudaMemsetAsync(ctx->Zs, 0, (size_t)n * ld * sizeof(double), ctx->st));
  SpView A{ctx->csc_ptr, ctx->csc_idx, ctx->csc_val, n, ctx->d};
  sp_densify_kernel<<<(unsigned)((n + 7) / 8), 256, 0, ctx->st>>>(A, ctx->Zs, ld);
  ctx->zs_gen++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->st));
  ctx->has_dense = true;
  return GDWD_OK;
}

int gdwd_generate_dense(gdwd_ctx* ctx, int32_t kind, uint64_t seed, int64_t d, int64_t n, int64_t offset,
                        int64_t signal_k, double shift) {
  if (!ctx || d < 1 || n < 1 || offset < 0) return set_err(ctx, GDWD_ERR_VALUE, "bad generation arguments");
  if (kind != 0) return set_err(ctx, GDWD_ERR_UNSUPPORTED, "only the two-Gaussian generator runs on the device");
  CK(cudaSetDevice(ctx->device));
  free_sparse(ctx);
  dfree(ctx->Zs, ctx->st);
  ctx->Zs = nullptr;
  const int64_t ld = (d + 1) / 2 * 2;
  CK(dmalloc((void**)&ctx->Zs, (size_t)n * ld * sizeof(double), ctx->st));
  if (ld != d) CK(cudaMemsetAsync(ctx->Zs, 0, (size_t)n * ld * sizeof(double), ctx->st));
  gen_gauss_kernel<<<NUM_SMS * 16, 256, 0, ctx->st>>>(ctx->Zs, ld, d, n, offset, seed, signal_k, shift);
  ctx->zs_gen++;
  CK(cudaGetLastError());
  ctx->n = n;
  ctx->d = d;
  ctx->ldz = ld;
  ctx->has_dense = true;
  ctx->has_problem = false;
  ctx->data_gen++;
  RC(ensure_scratch(ctx, n, d));
  return compute_fro2(ctx, ctx->Zs, n, d, ld);  // ||X||_F^2 of the raw (local) samples
}

int gdwd_scale_dense(gdwd_ctx* ctx, const double* y, double z_scale) {
  if (!ctx || !ctx->has_dense || !y || !(z_scale > 0)) return set_err(ctx, GDWD_ERR_VALUE, "bad scale arguments");
  CK(cudaSetDevice(ctx->device));
  DevBuf yd;
  CK(yd.ensure(ctx->n));
  CK(cudaMemcpy(yd.p, y, ctx->n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaStreamSynchronize(cudaStreamLegacy));  // st is non-blocking: the staged copy must have landed
  scale_rows_kernel<<<NUM_SMS * 16, 256, 0, ctx->st>>>(ctx->Zs, ctx->ldz, ctx->d, ctx->n, yd.p, z_scale);
  ctx->zs_gen++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->st));
  yd.release();
  ctx->data_gen++;
  return compute_fro2(ctx, ctx->Zs, ctx->n, ctx->d, ctx->ldz);
}

int gdwd_download_dense(gdwd_ctx* ctx, double* samples) {
  if (!ctx || !ctx->has_dense || !samples) return set_err(ctx, GDWD_ERR_VALUE, "no dense data");
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->st));
  CK(cudaMemcpy2D(samples, ctx->d * sizeof(double), ctx->Zs, ctx->ldz * sizeof(double), ctx->d * sizeof(double),
                  ctx->n, cudaMemcpyDeviceToHost));
  return GDWD_OK;
}

int gdwd_set_problem(gdwd_ctx* ctx, const double* y, const double* e, const double* weights, double C, double q,
                     double z_scale) {
  if (!ctx || !(ctx->has_dense || ctx->has_sparse)) return set_err(ctx, GDWD_ERR_VALUE, "upload Z~ before set_problem");
  if (!y || !e || !weights) return set_err(ctx, GDWD_ERR_VALUE, "null problem vector");
  if (!(C > 0 && q > 0 && z_scale > 0)) return set_err(ctx, GDWD_ERR_VALUE, "C, q and z_scale must be positive");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = ctx->n;
  double yty = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(y[i] == 1.0 || y[i] == -1.0)) return set_err(ctx, GDWD_ERR_VALUE, "labels must be a length-n vector over {-1,+1}");
    if (!(e[i] > 0)) return set_err(ctx, GDWD_ERR_VALUE, "e must be positive of length n");
    if (!(weights[i] > 0)) return set_err(ctx, GDWD_ERR_VALUE, "weights must be positive of length n");
    yty += y[i] * y[i];
  }
  CK(ctx->y.ensure(n));
  CK(ctx->e.ensure(n));
  CK(ctx->wl.ensure(n));
  CK(cudaMemcpyAsync(ctx->y.p, y, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(ctx->e.p, e, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(ctx->wl.p, weights, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  ctx->C = C;
  ctx->q = q;
  ctx->zscale = z_scale;
  ctx->yty = yty;
  ctx->has_problem = true;
  ctx->data_gen++;
  if (ctx->comm_mode) {  // a new local problem invalidates the communicator setup
    if (ctx->comm && nccl::api().ok) nccl::api().CommDestroy(ctx->comm);
    ctx->comm = nullptr;
    ctx->comm_mode = 0;
    ctx->nranks = 1;
    ctx->rank = 0;
  }
  ctx->n_global = n;
  return GDWD_OK;
}

int gdwd_matvec(gdwd_ctx* ctx, const double* v_n, double* out_d) {
  if (!ctx || !(ctx->has_dense || ctx->has_sparse) || !v_n || !out_d) return set_err(ctx, GDWD_ERR_VALUE, "matvec: no data or null pointer");
  CK(cudaSetDevice(ctx->device));
  double *dv = nullptr, *dout = nullptr;
  CK(dmalloc((void**)&dv, ctx->n * sizeof(double), ctx->st));
  CK(dmalloc((void**)&dout, ctx->d * sizeof(double), ctx->st));
  CK(cudaMemcpyAsync(dv, v_n, ctx->n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  OpPlainZ op{dv, nullptr, dout, nullptr};
  run_zmv(ctx, op, zview(ctx));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_d, dout, ctx->d * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  dfree(dv, ctx->st);
  dfree(dout, ctx->st);
  return GDWD_OK;
}

int gdwd_matvec_t(gdwd_ctx* ctx, const double* v_d, double* out_n) {
  if (!ctx || !(ctx->has_dense || ctx->has_sparse) || !v_d || !out_n) return set_err(ctx, GDWD_ERR_VALUE, "matvec_t: no data or null pointer");
  CK(cudaSetDevice(ctx->device));
  double *dv = nullptr, *dout = nullptr;
  CK(dmalloc((void**)&dv, ctx->d * sizeof(double), ctx->st));
  CK(dmalloc((void**)&dout, ctx->n * sizeof(double), ctx->st));
  CK(cudaMemcpyAsync(dv, v_d, ctx->d * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  OpPlainZt op{dv, dout};
  run_zt(ctx, op, zview(ctx));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_n, dout, ctx->n * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  dfree(dv, ctx->st);
  dfree(dout, ctx->st);
  return GDWD_OK;
}

int gdwd_score(gdwd_ctx* ctx, const double* w, double beta, const double* y, double* scores, int64_t* wrong) {
  if (!ctx || !(ctx->has_dense || ctx->has_sparse) || !w)
    return set_err(ctx, GDWD_ERR_VALUE, "score: no data or null weights");
  if (y && !wrong) return set_err(ctx, GDWD_ERR_VALUE, "score: y given without a count output");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = ctx->n, d = ctx->d;
  // [w (d) | scores (n) | y (n) | count]
  double* buf = nullptr;
  CK(dmalloc((void**)&buf, (size_t)(d + 2 * n + 2) * sizeof(double), ctx->st));
  double *dw = buf, *dout = buf + d, *dy = buf + d + n, *dcnt = buf + d + 2 * n;
  CK(cudaMemcpyAsync(dw, w, d * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  if (y) CK(cudaMemcpyAsync(dy, y, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  RC(ensure_scratch(ctx, n, d));
  const int comm_mode = ctx->comm_mode;
  ctx->comm_mode = 0;  // local samples only
  OpScore op{dw, beta, y ? dy : nullptr, scores ? dout : nullptr, dcnt};
  run_zt(ctx, op, zview(ctx), "ztmv_score");
  ctx->comm_mode = comm_mode;
  CK(cudaGetLastError());
  double cnt = 0.0;
  if (scores) CK(cudaMemcpyAsync(scores, dout, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  if (y) CK(cudaMemcpyAsync(&cnt, dcnt, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  dfree(buf, ctx->st);
  if (wrong) *wrong = y ? (int64_t)cnt : 0;
  return GDWD_OK;
}

int gdwd_kkt_residuals(gdwd_ctx* ctx, const double* r, const double* xi, const double* alpha, const double* w,
                       const double* u, double beta, double mu, double* out11) {
  if (!ctx || !ctx->has_problem) return set_err(ctx, GDWD_ERR_VALUE, "kkt_residuals: no problem uploaded");
  if (!r || !xi || !alpha || !w || !u || !out11) return set_err(ctx, GDWD_ERR_VALUE, "kkt_residuals: null argument");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = ctx->n, d = ctx->d;
  double* buf = nullptr;  // [r | xi | alpha (n each) | w | u (d each) | sums (13)]
  CK(dmalloc((void**)&buf, (size_t)(3 * n + 2 * d + 16) * sizeof(double), ctx->st));
  KktArgs K{buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 3 * n + d, ctx->y.p, ctx->e.p, ctx->wl.p, beta, ctx->C,
            ctx->q, ctx->q + 1.0, 1.0 / (ctx->q + 1.0), ctx->q / (ctx->q + 1.0), buf + 3 * n + 2 * d};
  CK(cudaMemcpyAsync(buf, r, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(buf + n, xi, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(buf + 2 * n, alpha, n * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(buf + 3 * n, w, d * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(buf + 3 * n + d, u, d * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  RC(ensure_scratch(ctx, n, d));
  const int comm_mode = ctx->comm_mode;
  ctx->comm_mode = 0;  // a local iterate
  MatView Z = zview(ctx);
  run_zt(ctx, OpKktZt{K}, Z, "ztmv_kkt");
  run_zmv(ctx, OpKktZa{K}, Z, "zmv_kkt");
  run_vm(ctx, OpKktD{K}, d, "vmap_kkt");
  ctx->comm_mode = comm_mode;
  CK(cudaGetLastError());
  double t[13];
  CK(cudaMemcpyAsync(t, K.out, sizeof(t), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  dfree(buf, ctx->st);
  if (t[9] > 0.0) return set_err(ctx, GDWD_ERR_ASSERT, "margin iterate left the positive orthant");
  // the reference's scalar assembly (solver.py:323-340)
  const double C = ctx->C, oc = 1.0 + C, q = ctx->q;
  const double kappa = (q + 1.0) / q * pow(q, 1.0 / (q + 1.0));
  out11[0] = fabs(t[0]) / oc;
  out11[1] = fabs(t[1]) / oc;
  out11[2] = t[2] / oc;
  out11[3] = sqrt(t[3]) / oc;
  out11[4] = mu * sqrt(t[11]) / oc;
  out11[5] = std::max(sqrt(t[12]) - ctx->zscale, 0.0) / oc;
  out11[6] = sqrt(t[4]) / oc;
  out11[7] = sqrt(t[5]) / oc;
  const double op = t[6] + C * t[7];
  const double od = kappa * t[8] - ctx->zscale * sqrt(t[10]);
  out11[8] = fabs(op - od) / (1.0 + fabs(op) + fabs(od));
  out11[9] = op;
  out11[10] = od;
  return GDWD_OK;
}

int gdwd_between_class_median(gdwd_ctx* ctx, const int64_t* ia, int64_t na, const int64_t* ib, int64_t nb,
                              double* median, int64_t* positives) {
  if (!ctx || !(ctx->has_dense || ctx->has_sparse) || !ia || !ib || !median || !positives || na < 1 || nb < 1)
    return set_err(ctx, GDWD_ERR_VALUE, "between_class_median: bad arguments");
  for (int64_t t = 0; t < na; ++t)
    if (ia[t] < 0 || ia[t] >= ctx->n) return set_err(ctx, GDWD_ERR_VALUE, "sample index out of range");
  for (int64_t t = 0; t < nb; ++t)
    if (ib[t] < 0 || ib[t] >= ctx->n) return set_err(ctx, GDWD_ERR_VALUE, "sample index out of range");
  CK(cudaSetDevice(ctx->device));
  const int64_t d = ctx->d, ldd = (d + 1) / 2 * 2, ldg = (nb + 1) / 2 * 2, tot = na * nb;
  // [A (na x ldd) | B (nb x ldd) | G (na x ldg) | dist (tot) | sqa | sqb] + index / counter block
  const size_t nd = (size_t)(na + nb) * ldd + (size_t)na * ldg + (size_t)tot + na + nb;
  double* buf = nullptr;
  CK(dmalloc((void**)&buf, nd * sizeof(double), ctx->st));
  double *A = buf, *B = A + na * ldd, *Gm = B + nb * ldd, *dist = Gm + na * ldg, *sqa = dist + tot, *sqb = sqa + na;
  int64_t* idx = nullptr;
  CK(dmalloc((void**)&idx, (size_t)(na + nb + 2 + 256 + 1) * sizeof(int64_t), ctx->st));
  int64_t *dia = idx, *dib = idx + na;
  unsigned long long* state = reinterpret_cast<unsigned long long*>(idx + na + nb);
  unsigned long long* hist = state + 2;
  unsigned long long* zeros = hist + 256;
  CK(cudaMemcpyAsync(dia, ia, na * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(dib, ib, nb * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemsetAsync(state, 0, (2 + 256 + 1) * sizeof(unsigned long long), ctx->st));
  CK(cudaMemsetAsync(A, 0, (size_t)(na + nb) * ldd * sizeof(double), ctx->st));
  if (ctx->has_dense) {
    gather_rows_kernel<<<(unsigned)((na + 7) / 8), 256, 0, ctx->st>>>(ctx->Zs, ctx->ldz, dia, na, d, A, ldd);
    gather_rows_kernel<<<(unsigned)((nb + 7) / 8), 256, 0, ctx->st>>>(ctx->Zs, ctx->ldz, dib, nb, d, B, ldd);
  } else {
    SpView S{ctx->csc_ptr, ctx->csc_idx, ctx->csc_val, ctx->n, d};
    gather_csc_kernel<<<(unsigned)((na + 7) / 8), 256, 0, ctx->st>>>(S, dia, na, A, ldd);
    gather_csc_kernel<<<(unsigned)((nb + 7) / 8), 256, 0, ctx->st>>>(S, dib, nb, B, ldd);
  }
  row_sq_kernel<<<(unsigned)((na + 7) / 8), 256, 0, ctx->st>>>(A, ldd, na, d, sqa);
  row_sq_kernel<<<(unsigned)((nb + 7) / 8), 256, 0, ctx->st>>>(B, ldd, nb, d, sqb);
  CK(cudaGetLastError());
  CK(gemm_f64(A, ldd, 1, B, ldd, 1, na, nb, d, 1.0, 0.0, Gm, ldg, ctx->st));  // G = A B^T (DMMA)
  between_dist_kernel<<<NUM_SMS * 8, 256, 0, ctx->st>>>(Gm, ldg, sqa, sqb, na, nb, dist, zeros);
  CK(cudaGetLastError());
  unsigned long long z = 0;
  CK(cudaMemcpyAsync(&z, zeros, sizeof(z), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  const int64_t m = tot - (int64_t)z;
  *positives = m;
  *median = 0.0;
  if (m > 0) {
    // zeros are the smallest values, so the j-th positive is order statistic z + j
    const int64_t ks[2] = {(int64_t)z + (m - 1) / 2, (int64_t)z + m / 2};
    double v[2] = {0.0, 0.0};
    for (int q = 0; q < (ks[0] == ks[1] ? 1 : 2); ++q) {
      const unsigned long long st0[2] = {0ull, (unsigned long long)ks[q]};
      CK(cudaMemcpyAsync(state, st0, sizeof(st0), cudaMemcpyHostToDevice, ctx->st));
      for (int shift = 56; shift >= 0; shift -= 8) {
        radix_hist_kernel<<<NUM_SMS * 4, 256, 0, ctx->st>>>(dist, tot, state, shift, hist);
        radix_pick_kernel<<<1, 32, 0, ctx->st>>>(hist, state, shift);
      }
      CK(cudaGetLastError());
      unsigned long long bits = 0;
      CK(cudaMemcpyAsync(&bits, state, sizeof(bits), cudaMemcpyDeviceToHost, ctx->st));
      CK(cudaStreamSynchronize(ctx->st));
      memcpy(&v[q], &bits, sizeof(double));
    }
    // np.median: the middle value, or the mean of the two middle values
    *median = (ks[0] == ks[1]) ? v[0] : (v[0] + v[1]) / 2.0;
  }
  dfree(buf, ctx->st);
  dfree(idx, ctx->st);
  return GDWD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// solver internals
// ---------------------------------------------------------------------------
static int select_kind(int64_t n, int64_t d) {  // subsolvers.py:42-55
  if (d > 5000 && 5 * n < d && n <= 2500) return GDWD_BACKEND_SMW2;
  if (d > 5000) return GDWD_BACKEND_ITERATIVE;
  return GDWD_BACKEND_DIRECT;
}

// One-time factorisation (cached per data generation / kind / mu^2).
// Diagnostics (GDWD_SETUP_TIMING): stream-ordered marks through the setup,
// printed as deltas when the solve begins.
struct SetupTimer {
  cudaStream_t st;
  bool on;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  explicit SetupTimer(cudaStream_t s) : st(s), on(getenv("GDWD_SETUP_TIMING") != nullptr) { mark("start"); }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.emplace_back(name, e);
  }
  ~SetupTimer() {
    if (!on) return;
    cudaStreamSynchronize(st);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      fprintf(stderr, "[setup timing] %-22s %8.3f ms\n", ev[i].first, ms);
    }
    for (auto& p : ev) cudaEventDestroy(p.second);
  }
};

static int build_factor(gdwd_ctx* ctx, int kind, double mu2) {
  Range nvtx_range("build_factor");
  if (ctx->fac_gen == ctx->data_gen && ctx->fac_kind == kind && ctx->fac_mu2 == mu2 &&
      ctx->fac_iter_gram == (int)ctx->iter_gram)
    return GDWD_OK;
  Dev& D = ctx->D;
  const int64_t n = ctx->n, d = ctx->d;
  MatView Z = zview(ctx);
  SetupTimer T(ctx->st);
  if (kind == GDWD_BACKEND_DIRECT || kind == GDWD_BACKEND_SMW2) {
    RC(densify(ctx));
    T.mark("densify");
    const int64_t m = (kind == GDWD_BACKEND_DIRECT) ? d + 1 : n;
    const int64_t ld = (m + 1) / 2 * 2;
    // G^{-1} already formed block by block during the upload (same data, same mu)
    const bool pf = kind == GDWD_BACKEND_SMW2 && ctx->pf_gen == ctx->zs_gen && ctx->pf_mu2 == mu2 &&
                    ctx->k_gen == ctx->zs_gen;
    // DIRECT: Z~ Z~^T already summed block by block during the upload (in fac)
    const bool dg = kind == GDWD_BACKEND_DIRECT && !sharded(ctx) && ctx->dg_gen == ctx->zs_gen;
    if (!pf && !dg) {
      CK(ctx->fac.ensure((size_t)m * ld));
      CK(cudaMemsetAsync(ctx->fac.p, 0, (size_t)m * ld * sizeof(double), ctx->st));
    }
    const int64_t K = (kind == GDWD_BACKEND_DIRECT) ? n : d;
    const int64_t M = (kind == GDWD_BACKEND_DIRECT) ? d : n;
    size_t ws = std::max<size_t>((size_t)gram_workspace_doubles(M, K), (size_t)2 * m * ld);
    if (!pf) CK(ctx->facw.ensure(ws));
    if (kind == GDWD_BACKEND_DIRECT) {
      if (sharded(ctx)) {
        // local Z_p Z_p^T, summed over the shards once (8 MB at d=1000), then + mu^2 I
        CK(gram_syrk(ctx->Zs, n, d, ctx->ldz, true, 1.0, 0.0, ctx->fac.p, ld, ctx->facw.p, ctx->st));
        allreduce(ctx, ctx->fac.p, (int64_t)m * ld);
        add_diag_kernel<<<(unsigned)((d + 255) / 256), 256, 0, ctx->st>>>(ctx->fac.p, ld, d, mu2);
      } else if (dg) {
        add_diag_kernel<<<(unsigned)((d + 255) / 256), 256, 0, ctx->st>>>(ctx->fac.p, ld, d, mu2);
      } else {
        CK(gram_syrk(ctx->Zs, n, d, ctx->ldz, true, 1.0, mu2, ctx->fac.p, ld, ctx->facw.p, ctx->st));
      }
      ctx->dg_gen = -1;  // fac is overwritten by the inverse below
      assemble_direct_kernel<<<(unsigned)((d + 256) / 256), 256, 0, ctx->st>>>(ctx->fac.p, ld, d, D.zy, ctx->yty);
    } else {
      // keep K = Z^T Z for the Gram-space iteration; G = K/mu^2 + I
      if (ctx->k_gen != ctx->zs_gen) {
        CK(ctx->kmat.ensure((size_t)m * ld));
        // zero pad columns: the persistent kernel's paired loads read them (times 0)
        CK(cudaMemsetAsync(ctx->kmat.p, 0, (size_t)m * ld * sizeof(double), ctx->st));
      }
      if (ctx->k_gen == ctx->zs_gen) {
        // K was formed during the upload, chunk by chunk as the rows landed
      } else {
        CK(gram_syrk(ctx->Zs, n, d, ctx->ldz, false, 1.0, 0.0, ctx->kmat.p, ld, ctx->facw.p, ctx->st));
      }
      T.mark("gram K = Z^T Z");
      if (!pf) {
        g_from_k_kernel<<<vm_grid(m * m), 256, 0, ctx->st>>>(ctx->kmat.p, ctx->fac.p, m, ld, mu2);
        CK(cudaGetLastError());
        T.mark("G = K/mu^2 + I");
      }
    }
    if (!pf) {
      CK(cudaMemsetAsync(ctx->dinfo, 0, sizeof(int), ctx->st));
      CK(chol_inverse(ctx->fac.p, ctx->facw.p, ctx->facw.p + (size_t)m * ld, ld, m, ctx->dinfo, ctx->st));
      T.mark("cholesky inverse");
    }
    ctx->pf_gen = -1;  // fac now belongs to this factorisation (a later refactor overwrites it)
    int info = 0;
    CK(cudaMemcpyAsync(&info, ctx->dinfo, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (info != 0) return set_err(ctx, GDWD_ERR_INDEFINITE, "non-positive pivot in Cholesky factorisation");
    ctx->ldm = ld;
    ctx->fac_rows = m;
    if (kind == GDWD_BACKEND_SMW2) {
      // GK = G^{-1} K for the persistent Gram-space loop, = mu^2 (I - G^{-1})
      CK(ctx->gkmat.ensure((size_t)m * ld));
      CK(cudaMemsetAsync(ctx->gkmat.p, 0, (size_t)m * ld * sizeof(double), ctx->st));
      gk_from_ginv_kernel<<<vm_grid(m * m), 256, 0, ctx->st>>>(ctx->fac.p, ctx->gkmat.p, m, ld, mu2);
      CK(cudaGetLastError());
      T.mark("GK = mu^2 (I - G^-1)");
      OpJyG op{ctx->y.p, D.ynorm, const_cast<double*>(D.jy), ctx->S};
      RC(ensure_scratch(ctx, m, m));
      run_zt(ctx, op, MatView{ctx->fac.p, m, m, ld});
      CK(cudaGetLastError());
      // fixed vectors of the 3-barrier persistent kernel (persist3.cuh)
      run_zt(ctx, OpGemvStore{D.jy, 1.0, const_cast<double*>(D.kap)}, MatView{ctx->kmat.p, m, m, ld});
      run_zt(ctx, OpGemvStore{ctx->y.p, D.ynorm, const_cast<double*>(D.gam)}, MatView{ctx->gkmat.p, m, m, ld});
      CK(cudaGetLastError());
      RC(ensure_scratch(ctx, n, d));
      T.mark("G^-1 y, K G^-1 y, GK y");
    }
  } else {
    if (Z.a && n >= 65536) {
      const int comm_mode = ctx->comm_mode;
      ctx->comm_mode = 0;  // local sums; all-reduced below
      run_zmv(ctx, OpColSq{ctx->colsq.p}, Z, "zmv_colsq");
      ctx->comm_mode = comm_mode;
    } else if (Z.a) {
      colsq_kernel<OpColSqPrep><<<(unsigned)((d + 255) / 256), 256, 0, ctx->st>>>(Z, ctx->colsq.p);
    } else {
      SpView A{ctx->csr_ptr, ctx->csr_idx, ctx->csr_val, d, n};
      sp_rowsq_kernel<<<(unsigned)((d + 255) / 256), 256, 0, ctx->st>>>(A, ctx->colsq.p);
    }
    if (sharded(ctx)) allreduce(ctx, ctx->colsq.p, d);
    jacobi_kernel<<<(unsigned)((d + 256) / 256), 256, 0, ctx->st>>>(ctx->colsq.p, d, mu2, ctx->yty,
                                                                     const_cast<double*>(D.jac));
    CK(cudaGetLastError());
    if (ctx->iter_gram) {
      // PSQMR operator block Z~ Z~^T, once (sharded: local Gram, summed once)
      const int64_t ld = (d + 1) / 2 * 2;
      CK(ctx->gdmat.ensure((size_t)d * ld));
      CK(ctx->facw.ensure((size_t)gram_workspace_doubles(d, n)));
      CK(gram_syrk(ctx->Zs, n, d, ctx->ldz, true, 1.0, 0.0, ctx->gdmat.p, ld, ctx->facw.p, ctx->st));
      if (sharded(ctx)) allreduce(ctx, ctx->gdmat.p, d * ld);
      ctx->ldg = ld;
      T.mark("iterative Gram Z Z^T");
    }
  }
  CK(cudaStreamSynchronize(ctx->st));
  ctx->fac_gen = ctx->data_gen;
  ctx->fac_kind = kind;
  ctx->fac_mu2 = mu2;
  ctx->fac_iter_gram = (int)ctx->iter_gram;
  return GDWD_OK;
}

// enqueue one normal-system solve: out = A^{-1} hv (DIRECT / SMW2)
static void enqueue_solve(gdwd_ctx* ctx, int kind, const double* hv, double* out, int pred) {
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  MatView F{ctx->fac.p, ctx->fac_rows, ctx->fac_rows, ctx->ldm};
  if (kind == GDWD_BACKEND_DIRECT) {
    run_zt(ctx, OpGemvSolve{D, hv, out, pred}, F, pred ? "gemv_Ainv_2" : "gemv_Ainv");
  } else {
    run_zt(ctx, OpSmwS1{D, hv, pred}, Z, pred ? "ztmv_smw_s1_2" : "ztmv_smw_s1");
    run_zt(ctx, OpSmwG{D, hv, pred}, F, pred ? "gemv_Ginv_2" : "gemv_Ginv");
    run_zmv(ctx, OpSmwP{D, hv, out, pred}, Z, pred ? "zmv_smw_p_2" : "zmv_smw_p");
  }
}

// host-driven PSQMR solve (ITERATIVE): out ~ A^{-1} b from x0
static int psqmr_solve(gdwd_ctx* ctx, const double* b, const double* x0, double* out, int pred, double tolmul,
                       int max_steps, int* steps, int* conv, int* active_run) {
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  const MatView Gd{ctx->gdmat.p, ctx->d, ctx->d, ctx->ldg};
  if (ctx->iter_gram) {
    run_zt(ctx, OpInitResidualGram{D, x0, b, pred}, Gd, "gemv_gram_psqmr_init");
  } else {
    run_zt(ctx, OpApplyZt{D, x0, pred, 0}, Z, "ztmv_psqmr_init");
    run_zmv(ctx, OpInitResidual{D, x0, b, pred}, Z, "zmv_psqmr_init");
  }
  run_vm(ctx, OpPsInit{D, x0, out, pred, tolmul}, D.m, "vmap_psqmr_init");
  CK(cudaGetLastError());
  *steps = 0;
  *conv = 1;
  *active_run = 0;
  for (int it = 0; it <= max_steps; ++it) {
    CK(cudaMemcpyAsync(ctx->Sh, ctx->S, sizeof(Scal), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    const Scal& s = *ctx->Sh;
    if (s.stopped) return GDWD_OK;
    if (it == 0) {
      if (pred && s.reuse) return GDWD_OK;  // skipped by the Step-1c predicate
      *active_run = 1;
    }
    if (!s.ps_active) {
      *steps = s.ps_iters;
      *conv = s.ps_conv;
      return GDWD_OK;
    }
    if (it == max_steps) break;
    if (ctx->iter_gram) {
      run_zt(ctx, OpPsApplyGram{D}, Gd, "gemv_gram_psqmr_apply");
    } else {
      run_zt(ctx, OpApplyZt{D, D.pq, 0, 1}, Z, "ztmv_psqmr_apply");
      run_zmv(ctx, OpPsApply{D}, Z, "zmv_psqmr_apply");
    }
    run_vm(ctx, OpPsV1{D}, D.m, "vmap_psqmr_v1");
    run_vm(ctx, OpPsV2{D, out, tolmul, max_steps}, D.m, "vmap_psqmr_v2");
    CK(cudaGetLastError());
  }
  *steps = ctx->Sh->ps_iters;
  *conv = ctx->Sh->ps_conv;
  return GDWD_OK;
}

// ---------------------------------------------------------------------------
// Device-resident PSQMR: the step loop is a CUDA-graph WHILE node whose
// condition a one-thread kernel sets from the device scalars (active and not
// stopped) -- no host synchronisation inside a solve.  Same kernels, same
// order, same recurrence as psqmr_solve (psqmr.py:65-93).
// ---------------------------------------------------------------------------
__global__ void ps_cond_kernel(const Scal* S, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, (!S->stopped && S->ps_active) ? 1u : 0u);
}

// Append WHILE(h) { body() } to the capture on ctx->st; body() enqueues on
// ctx->st, which is pointed at a capture-to-graph stream meanwhile.
template <class F>
static int capture_while(gdwd_ctx* ctx, cudaGraphConditionalHandle h, F&& body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(ctx->st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(ctx->st, &node, 1, cudaStreamSetCaptureDependencies));
  cudaStream_t outer = ctx->st;
  ctx->st = ctx->cap_st;
  const int64_t before = ctx->launches;
  cudaError_t e = cudaStreamBeginCaptureToGraph(ctx->cap_st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    body();
    cudaGraph_t tmp = nullptr;
    e = cudaStreamEndCapture(ctx->cap_st, &tmp);
  }
  ctx->ps_step_nodes = ctx->launches - before + 1;  // + the condition kernel
  ctx->launches = before;
  ctx->st = outer;
  CK(e);
  return GDWD_OK;
}

static int psqmr_dev(gdwd_ctx* ctx, const double* b, const double* x0, double* out, int pred, double tolmul,
                     int which) {
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  const MatView Gd{ctx->gdmat.p, ctx->d, ctx->d, ctx->ldg};
  if (ctx->iter_gram) {
    run_zt(ctx, OpInitResidualGram{D, x0, b, pred}, Gd, "gemv_gram_psqmr_init");
  } else {
    run_zt(ctx, OpApplyZt{D, x0, pred, 0}, Z, "ztmv_psqmr_init");
    run_zmv(ctx, OpInitResidual{D, x0, b, pred}, Z, "zmv_psqmr_init");
  }
  run_vm(ctx, OpPsInit{D, x0, out, pred, tolmul}, D.m, "vmap_psqmr_init");
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  CK(cudaStreamGetCaptureInfo(ctx->st, &cs, nullptr, &g, nullptr, nullptr));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
  ps_cond_kernel<<<1, 1, 0, ctx->st>>>(ctx->S, h);
  ctx->launches++;
  const int max_steps = ctx->max_steps;
  RC(capture_while(ctx, h, [&]() {
    if (ctx->iter_gram) {
      run_zt(ctx, OpPsApplyGram{D}, Gd, "gemv_gram_psqmr_apply");
    } else {
      run_zt(ctx, OpApplyZt{D, D.pq, 0, 1}, Z, "ztmv_psqmr_apply");
      run_zmv(ctx, OpPsApply{D}, Z, "zmv_psqmr_apply");
    }
    run_vm(ctx, OpPsV1{D}, D.m, "vmap_psqmr_v1");
    run_vm(ctx, OpPsV2{D, out, tolmul, max_steps}, D.m, "vmap_psqmr_v2");
    ps_cond_kernel<<<1, 1, 0, ctx->st>>>(ctx->S, h);
  }));
  run_vm(ctx, OpPsEnd{D, pred, which}, 1, "vmap_psqmr_end");
  return GDWD_OK;
}

// the tail shared by every backend: w/ztw commit, Steps 2-3, KKT sample terms
static void enqueue_tail(gdwd_ctx* ctx) {
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  run_vm(ctx, OpCopyIfReuse{D, D.xb, D.x}, D.m, "vmap_copy_x");
  if (ctx->ft) {
    // Step 2 (d-space), then Z~^T w, Step 3 and Z~ [xi - r, alpha] in one pass
    run_vm(ctx, OpStep2a{D}, D.d, "vmap_step2a");
    run_vm(ctx, OpStep2b{D}, D.d, "vmap_step2b");
    run_ft(ctx, OpTail{D}, Z, "zft_tail");
    run_vm(ctx, OpKktTail{D}, D.n, "vmap_kkt_tail", true);
    return;
  }
  run_zt(ctx, OpZtStore{D, D.x, D.ztw, 1}, Z, "ztmv_ztw_2");
  run_vm(ctx, OpCopyIfReuse{D, D.ztwb, D.ztw}, D.n, "vmap_copy_ztw");
  run_vm(ctx, OpStep2a{D}, D.d, "vmap_step2a");
  run_vm(ctx, OpStep2b{D}, D.d, "vmap_step2b");
  run_vm(ctx, OpStep3{D}, D.n, "vmap_step3_kkt", true);
}

// h of this iteration and the completion of the previous one (dual
// objective, gap, stopping test): one X pass, or a d-space map after a fused tail
static void enqueue_rhs(gdwd_ctx* ctx) {
  const Dev& D = ctx->D;
  if (ctx->ft) run_vm(ctx, OpRhsParts{D}, D.d, "vmap_rhs_parts");
  else run_zmv(ctx, OpRhsAlpha{D}, zview(ctx), "zmv_rhs_alpha");
}

static void enqueue_body_fixed(gdwd_ctx* ctx, int kind, bool use_sgs) {
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  enqueue_rhs(ctx);
  enqueue_solve(ctx, kind, D.h, D.xb, 0);
  run_zt(ctx, OpZtNewton{D}, Z, "ztmv_newton");
  if (use_sgs) run_zmv(ctx, OpDrZtwb{D}, Z, "zmv_dr_ztwb");
  else run_vm(ctx, OpSetReuse{D}, 1, "vmap_set_reuse");
  enqueue_solve(ctx, kind, D.h2, D.x, 1);
  enqueue_tail(ctx);
}

// Gram-space SMW2 body (see solver_ops.cuh): no pass over X
static void enqueue_solve_gram(gdwd_ctx* ctx, const double* hv, double* out, int pred) {
  const Dev& D = ctx->D;
  MatView K{ctx->kmat.p, ctx->n, ctx->n, ctx->ldm};
  MatView F{ctx->fac.p, ctx->fac_rows, ctx->fac_rows, ctx->ldm};
  run_zt(ctx, OpSmwS1{D, hv, pred}, K, pred ? "gemv_K_s1_2" : "gemv_K_s1");
  run_zt(ctx, OpSmwG{D, hv, pred}, F, pred ? "gemv_Ginv_2" : "gemv_Ginv");
  run_vm(ctx, GsX{D, hv, out, pred}, ctx->n, pred ? "vmap_gs_x_2" : "vmap_gs_x");
}

static void enqueue_body_gram(gdwd_ctx* ctx, bool use_sgs) {
  const Dev& D = ctx->D;
  const int64_t n = ctx->n;
  MatView K{ctx->kmat.p, n, n, ctx->ldm};
  run_zt(ctx, GsKAlpha{D}, K, "gemv_K_alpha");
  run_vm(ctx, GsRhs{D}, n, "vmap_gs_rhs");
  enqueue_solve_gram(ctx, D.h, D.xb, 0);
  run_zt(ctx, OpZtNewton{D}, K, "gemv_K_newton");
  if (use_sgs) {
    run_vm(ctx, GsResid1{D}, n, "vmap_gs_resid");
    run_zt(ctx, GsResid2{D}, K, "gemv_K_resid");
  } else {
    run_vm(ctx, OpSetReuse{D}, 1, "vmap_set_reuse");
  }
  enqueue_solve_gram(ctx, D.h2, D.x, 1);
  run_vm(ctx, OpCopyIfReuse{D, D.xb, D.x}, n + 1, "vmap_copy_x");
  run_zt(ctx, OpZtStore{D, D.x, D.ztw, 1}, K, "gemv_K_ztw_2");
  run_vm(ctx, OpCopyIfReuse{D, D.ztwb, D.ztw}, n, "vmap_copy_ztw");
  run_zt(ctx, GsStep2a{D}, K, "gemv_K_step2a");
  run_vm(ctx, GsStep2b{D}, n, "vmap_gs_step2b");
  run_zt(ctx, GsStep2c{D}, K, "gemv_K_step2c");
  run_vm(ctx, OpStep3{D}, n, "vmap_step3_kkt");
}

// w, u, rho back in feature space (one pass over X for w,u and one for rho)
static void enqueue_materialize(gdwd_ctx* ctx) {
  if (!ctx->gram) return;
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  run_zmv(ctx, GsMaterialize2{D}, Z, "zmv_materialize");
  run_zmv(ctx, GsMaterialize1{D}, Z, "zmv_materialize");
}

// ---------------------------------------------------------------------------
// proximal fallback
// ---------------------------------------------------------------------------
// eigen-decomposition of a symmetric tridiagonal (k <= ~100) by cyclic
// Jacobi rotations; eigenvalues in `ev`, eigenvectors as columns of S (k x k)
static void tridiag_eig(const std::vector<double>& a, const std::vector<double>& b, std::vector<double>& ev,
                        std::vector<double>& S) {
  const int k = (int)a.size();
  std::vector<double> M((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) M[i * k + i] = a[i];
  for (int i = 0; i + 1 < k; ++i) M[i * k + i + 1] = M[(i + 1) * k + i] = b[i];
  S.assign((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) S[i * k + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {
        tot += M[i * k + j] * M[i * k + j];
        if (i != j) off += M[i * k + j] * M[i * k + j];
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = M[p * k + q];
        if (fabs(apq) < 1e-300) continue;
        const double theta = (M[q * k + q] - M[p * k + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int r = 0; r < k; ++r) {  // columns p, q
          const double mrp = M[r * k + p], mrq = M[r * k + q];
          M[r * k + p] = c * mrp - sn * mrq;
          M[r * k + q] = sn * mrp + c * mrq;
        }
        for (int r = 0; r < k; ++r) {  // rows p, q
          const double mpr = M[p * k + r], mqr = M[q * k + r];
          M[p * k + r] = c * mpr - sn * mqr;
          M[q * k + r] = sn * mpr + c * mqr;
        }
        for (int r = 0; r < k; ++r) {
          const double srp = S[r * k + p], srq = S[r * k + q];
          S[r * k + p] = c * srp - sn * srq;
          S[r * k + q] = sn * srp + c * srq;
        }
      }
  }
  ev.resize(k);
  for (int i = 0; i < k; ++i) ev[i] = M[i * k + i];
}

static double hdot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// lanczos_topk (lanczos.py:47-133) on v -> Z~(Z~^T v) with device applies,
// then the ProximalFactor (subsolvers.py:204-240) uploaded to the device.
static int build_prox(gdwd_ctx* ctx) {
  Dev& D = ctx->D;
  const int64_t d = ctx->d, n = ctx->n;
  if (d < 2) return set_err(ctx, GDWD_ERR_VALUE, "proximal backend needs d >= 2");
  const int k = (int)std::min<int64_t>(ctx->ell, d - 1);
  if (k - 1 > PX_MAXL) return set_err(ctx, GDWD_ERR_UNSUPPORTED, "ell > 17 not supported by the proximal kernels");
  const int cap = (int)std::min<int64_t>(d, std::max(10 * k, 100));
  const double tol = 1e-12;
  if ((int64_t)ctx->lz_start.size() != d) return set_err(ctx, GDWD_ERR_VALUE, "no Lanczos start vector");
  MatView Z = zview(ctx);
  DevBuf dv, dw, dt;
  CK(dv.ensure(d));
  CK(dw.ensure(d));
  CK(dt.ensure(n));
  auto apply = [&](const std::vector<double>& v, std::vector<double>& w) -> int {
    CK(cudaMemcpyAsync(dv.p, v.data(), d * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
    run_zt(ctx, OpPlainZt{dv.p, dt.p}, Z, "ztmv_lanczos");
    run_zmv(ctx, OpPlainZ{dt.p, nullptr, dw.p, nullptr}, Z, "zmv_lanczos");
    CK(cudaMemcpyAsync(w.data(), dw.p, d * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return GDWD_OK;
  };
  std::vector<std::vector<double>> basis;
  std::vector<double> al, be, v(ctx->lz_start), w(d), ev, Sm;
  {
    const double nv = sqrt(hdot(v.data(), v.data(), d));
    for (auto& x : v) x /= nv;
  }
  double nest = 0.0;
  std::vector<double> lam_best;
  std::vector<std::vector<double>> vec_best;
  bool ok = false;
  uint64_t rs = 0x9E3779B97F4A7C15ull;
  for (int it = 0; it < cap; ++it) {
    RC(apply(v, w));
    const double a = hdot(v.data(), w.data(), d);
    for (int64_t j = 0; j < d; ++j) w[j] = w[j] - a * v[j];
    if (!basis.empty() && !be.empty() && be.back() != 0.0)
      for (int64_t j = 0; j < d; ++j) w[j] -= be.back() * basis.back()[j];
    basis.push_back(v);
    al.push_back(a);
    for (int rep = 0; rep < 2; ++rep) {  // full reorthogonalisation, twice
      std::vector<double> c(basis.size());
      for (size_t m = 0; m < basis.size(); ++m) c[m] = hdot(basis[m].data(), w.data(), d);
      for (int64_t j = 0; j < d; ++j) {
        double s = 0.0;
        for (size_t m = 0; m < basis.size(); ++m) s += basis[m][j] * c[m];
        w[j] -= s;
      }
    }
    const double bn = sqrt(hdot(w.data(), w.data(), d));
    tridiag_eig(al, be, ev, Sm);
    const int kk = (int)al.size();
    double mx = 0.0;
    for (double x : ev) mx = std::max(mx, fabs(x));
    nest = std::max(nest, mx);
    std::vector<int> order(kk);
    for (int i = 0; i < kk; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return ev[x] > ev[y]; });
    const int top = std::min(k, kk);
    bool conv = true;
    lam_best.assign(top, 0.0);
    vec_best.assign(top, std::vector<double>(d, 0.0));
    for (int t = 0; t < top; ++t) {
      const int c = order[t];
      lam_best[t] = ev[c];
      if (fabs(bn * Sm[(size_t)(kk - 1) * kk + c]) > tol * std::max(nest, 1e-300)) conv = false;
      for (int m = 0; m < kk; ++m) {
        const double sm = Sm[(size_t)m * kk + c];
        for (int64_t j = 0; j < d; ++j) vec_best[t][j] += basis[m][j] * sm;
      }
    }
    if (kk >= k && (conv || kk == d)) {
      ok = true;
      break;
    }
    if (bn <= std::max(nest, 1.0) * 1e-14) {
      if (kk == d) {
        ok = true;
        break;
      }
      // invariant subspace: restart orthogonal to the basis (fresh direction)
      for (int64_t j = 0; j < d; ++j) {
        rs = rs * 6364136223846793005ull + 1442695040888963407ull;
        v[j] = ((double)(rs >> 11) / 9007199254740992.0) - 0.5;
      }
      for (int rep = 0; rep < 2; ++rep)
        for (auto& q : basis) {
          const double c = hdot(q.data(), v.data(), d);
          for (int64_t j = 0; j < d; ++j) v[j] -= c * q[j];
        }
      const double nv = sqrt(hdot(v.data(), v.data(), d));
      for (auto& x : v) x /= nv;
      be.push_back(0.0);
    } else {
      for (int64_t j = 0; j < d; ++j) v[j] = w[j] / bn;
      be.push_back(bn);
    }
  }
  if (!ok) return set_err(ctx, GDWD_ERR_LANCZOS, "no convergence to tol=1e-12 within " + std::to_string(cap) + " iterations");
  // ProximalFactor: inv / fwd coefficients, V[:, :-1], Schur scalar
  const double mu2 = D.mu2;
  const int L = k - 1;
  const double lamk = lam_best[k - 1];
  const double base = 1.0 / (mu2 + lamk);
  std::vector<double> cinv(PX_MAXL, 0.0), cfwd(PX_MAXL, 0.0);
  for (int i = 0; i < L; ++i) {
    cinv[i] = 1.0 / (mu2 + lam_best[i]) - base;
    cfwd[i] = lam_best[i] - lamk;
  }
  std::vector<double> zy(d);
  CK(cudaMemcpy(zy.data(), D.zy, d * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<double> iv(d);
  {
    std::vector<double> p(L);
    for (int i = 0; i < L; ++i) p[i] = hdot(vec_best[i].data(), zy.data(), d);
    for (int64_t j = 0; j < d; ++j) {
      double s = 0.0;
      for (int i = 0; i < L; ++i) s += vec_best[i][j] * (cinv[i] * p[i]);
      iv[j] = base * zy[j] + s;
    }
  }
  const double schur = ctx->yty - hdot(zy.data(), iv.data(), d);
  if (!(schur > 1e-14)) return set_err(ctx, GDWD_ERR_SCHUR, "Schur scalar is not safely positive");
  const size_t need = (size_t)PX_MAXL * d + 2 * PX_MAXL + 5 * (size_t)(d + 2);
  CK(ctx->pxbuf.ensure(need));
  double* px = ctx->pxbuf.p;
  for (int i = 0; i < L; ++i)
    CK(cudaMemcpy(px + (size_t)i * d, vec_best[i].data(), d * sizeof(double), cudaMemcpyHostToDevice));
  double* cb = px + (size_t)PX_MAXL * d;
  CK(cudaMemcpy(cb, cinv.data(), PX_MAXL * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(cb + PX_MAXL, cfwd.data(), PX_MAXL * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaStreamSynchronize(cudaStreamLegacy));  // st is non-blocking: the staged copies must have landed
  double* vb = cb + 2 * PX_MAXL;
  D.pxV = px;
  D.px_cinv = cb;
  D.px_cfwd = cb + PX_MAXL;
  D.px_sa = vb;
  D.px_hp = vb + (d + 2);
  D.px_tmp = vb + 2 * (d + 2);
  D.px_zaz = vb + 3 * (d + 2);
  D.px_base = base;
  D.px_fwd0 = mu2 + lamk;
  D.px_schur = schur;
  D.px_L = L;
  ctx->prox = true;
  return GDWD_OK;
}

// anchor w kept across the Step-1c PSQMR call (a free (d+1)-slot of mvec)
static double* px_wold(gdwd_ctx* ctx) { return ctx->mvec.p + 13 * ((ctx->d + 3) / 2 * 2); }

// solve_system in proximal mode (solver.py:484-491) -> out = [w; beta]
static void prox_solve(gdwd_ctx* ctx, const double* hv, double* out, int pred, bool compute_sa, const double* aw,
                       const double* aztw) {
  const Dev& D = ctx->D;
  const int64_t d = ctx->d;
  MatView Z = zview(ctx);
  if (compute_sa) {
    run_zmv(ctx, OpZtwStore{D, aztw, pred}, Z, "zmv_prox_anchor");
    run_vm(ctx, OpPxDot{D, aw, pred}, d, "vmap_prox");
    run_vm(ctx, OpPxShift{D, aw, hv, pred}, d, "vmap_prox");
  } else {
    run_vm(ctx, OpPxShifted{D, hv, pred}, d, "vmap_prox");
  }
  run_vm(ctx, OpPxDot{D, D.px_hp, pred}, d, "vmap_prox");
  run_vm(ctx, OpPxBeta{D, hv, pred}, d, "vmap_prox");
  run_vm(ctx, OpPxRhs2{D, pred}, d, "vmap_prox");
  run_vm(ctx, OpPxDot{D, D.px_tmp, pred}, d, "vmap_prox");
  run_vm(ctx, OpPxW{D, out, pred}, d, "vmap_prox");
}

static int body_iterative(gdwd_ctx* ctx, bool use_sgs, int max_steps, int* psqmr_steps) {
  Dev& D = ctx->D;
  MatView Z = zview(ctx);
  enqueue_rhs(ctx);
  int steps = 0, conv = 1, ran = 0;
  *psqmr_steps = 0;
  bool sa_ready = false;  // shift anchor of this iteration computed
  if (!ctx->prox) {
    RC(psqmr_solve(ctx, D.h, D.x, D.xb, 0, 1.0, max_steps, &steps, &conv, &ran));
    if (ctx->Sh->stopped) return GDWD_OK;
    *psqmr_steps += steps;
    if (ran && !conv) {  // solver.py:479-483: permanent switch to the proximal backend
      RC(build_prox(ctx));
      prox_solve(ctx, D.h, D.xb, 0, true, D.x, D.ztw);
      sa_ready = true;
    }
  } else {
    prox_solve(ctx, D.h, D.xb, 0, true, D.x, D.ztw);
    sa_ready = true;
  }
  run_zt(ctx, OpZtNewton{D}, Z, "ztmv_newton");
  if (use_sgs) {
    if (ctx->prox) {
      run_zmv(ctx, OpPxH2{D}, Z, "zmv_prox_h2");
      run_vm(ctx, OpPxDot{D, D.xb, 0}, ctx->d, "vmap_prox");
      run_vm(ctx, OpPxResid{D}, ctx->d, "vmap_prox_resid");
    } else {
      run_zmv(ctx, OpDrZtwb{D}, Z, "zmv_dr_ztwb");
    }
  } else {
    run_vm(ctx, OpSetReuse{D}, 1, "vmap_set_reuse");
  }
  if (ctx->prox) {
    prox_solve(ctx, D.h2, D.x, 1, !sa_ready, D.x, D.ztw);
  } else {
    // keep the anchor w of this iteration in case PSQMR gives up below
    run_vm(ctx, OpCopy{D, D.x, px_wold(ctx)}, D.m, "vmap_copy_x");
    RC(psqmr_solve(ctx, D.h2, D.xb, D.x, 1, 5.0, max_steps, &steps, &conv, &ran));
    *psqmr_steps += ran ? steps : 0;
    if (ran && !conv) {
      RC(build_prox(ctx));
      prox_solve(ctx, D.h2, D.x, 1, true, px_wold(ctx), D.ztw);
    }
  }
  enqueue_tail(ctx);
  CK(cudaGetLastError());
  return GDWD_OK;
}

// ITERATIVE body with both PSQMR solves device-resident (captured once per
// solve; the proximal switch is handled by the host, prox_resume)
static int body_iterative_dev(gdwd_ctx* ctx, bool use_sgs) {
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  enqueue_rhs(ctx);
  RC(psqmr_dev(ctx, D.h, D.x, D.xb, 0, 1.0, 1));
  run_zt(ctx, OpZtNewton{D}, Z, "ztmv_newton");
  if (use_sgs) run_zmv(ctx, OpDrZtwb{D}, Z, "zmv_dr_ztwb");
  else run_vm(ctx, OpSetReuse{D}, 1, "vmap_set_reuse");
  run_vm(ctx, OpCopy{D, D.x, px_wold(ctx)}, D.m, "vmap_copy_x");
  RC(psqmr_dev(ctx, D.h2, D.xb, D.x, 1, 5.0, 2));
  enqueue_tail(ctx);
  return GDWD_OK;
}

// A device-resident PSQMR solve of iteration k did not converge (OpPsEnd:
// error 7, need_prox = which solve): build the proximal backend and finish
// iteration k on the host path exactly as body_iterative does after its
// switch (solver.py:479-491).  Returns 1 when it resumed, 0 when the stop
// had another cause.
static int prox_resume(gdwd_ctx* ctx, bool use_sgs, int* resumed) {
  *resumed = 0;
  CK(cudaMemcpyAsync(ctx->Sh, ctx->S, sizeof(Scal), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  Scal& s = *ctx->Sh;
  if (s.error != 7) return GDWD_OK;
  const int k = s.k, which = s.need_prox;
  s.error = 0;
  s.need_prox = 0;
  s.stopped = 0;
  CK(cudaMemcpyAsync(ctx->S, ctx->Sh, sizeof(Scal), cudaMemcpyHostToDevice, ctx->st));
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  RC(build_prox(ctx));
  if (which == 1) {
    prox_solve(ctx, D.h, D.xb, 0, true, D.x, D.ztw);
    run_zt(ctx, OpZtNewton{D}, Z, "ztmv_newton");
    if (use_sgs) {
      run_zmv(ctx, OpPxH2{D}, Z, "zmv_prox_h2");
      run_vm(ctx, OpPxDot{D, D.xb, 0}, ctx->d, "vmap_prox");
      run_vm(ctx, OpPxResid{D}, ctx->d, "vmap_prox_resid");
    } else {
      run_vm(ctx, OpSetReuse{D}, 1, "vmap_set_reuse");
    }
    prox_solve(ctx, D.h2, D.x, 1, false, D.x, D.ztw);
  } else {
    prox_solve(ctx, D.h2, D.x, 1, true, px_wold(ctx), D.ztw);
  }
  enqueue_tail(ctx);
  CK(cudaGetLastError());
  ctx->k_host = k + 1;
  ctx->stopped = false;
  *resumed = 1;
  return GDWD_OK;
}

static void end_session(gdwd_ctx* ctx) {
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  ctx->gexec = nullptr;
  ctx->in_solve = false;
}

// Finish a persistent launch: wait for it and read its stop flag back.
static int pk_settle(gdwd_ctx* ctx) {
  if (!ctx->pk_pending) return GDWD_OK;
  ctx->pk_pending = false;
  CK(cudaMemcpyAsync(ctx->Sh, ctx->S, sizeof(Scal), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  if (ctx->pk_ts) {
    pk_timing_report(ctx->pk_ts, ctx->pk_tsn, 3);  // (frees the buffer)
    ctx->pk_ts = nullptr;
  }
  ctx->k_host = ctx->Sh->stopped ? ctx->Sh->iters_done : ctx->pk_kend;
  ctx->stopped = ctx->Sh->stopped != 0;
  return GDWD_OK;
}

extern "C" int gdwd_solve_begin(gdwd_ctx* ctx, const gdwd_config* cfg, const double* sched, int64_t sched_len) {
  Range nvtx_range("gdwd_solve_begin (setup)");
  if (!ctx || !cfg) return set_err(ctx, GDWD_ERR_VALUE, "null argument");
  if (!(ctx->has_dense || ctx->has_sparse) || !ctx->has_problem)
    return set_err(ctx, GDWD_ERR_VALUE, "no problem uploaded");
  if (!(cfg->steplength > 0.0 && cfg->steplength <= 1.618034))
    return set_err(ctx, GDWD_ERR_VALUE, "steplength must lie in (0, 1.618034)");
  if (std::min({cfg->tol_feas, cfg->tol_cgap, cfg->tol_cap}) <= 0)
    return set_err(ctx, GDWD_ERR_VALUE, "tolerances must be positive");
  if (cfg->mu <= 0 || cfg->ell < 1 || cfg->max_iter < 1)
    return set_err(ctx, GDWD_ERR_VALUE, "q, mu must be positive; ell, max_iter at least 1");
  CK(cudaSetDevice(ctx->device));
  RC(pk_settle(ctx));
  end_session(ctx);
  const int64_t n = ctx->n, d = ctx->d, m = d + 1;
  const int64_t ng = ctx->n_global > 0 ? ctx->n_global : n;  // sharded: the global sample count
  int kind = cfg->backend == GDWD_BACKEND_AUTO ? select_kind(ng, d) : cfg->backend;
  if (kind < 1 || kind > 3) return set_err(ctx, GDWD_ERR_VALUE, "bad backend");
  if (sharded(ctx) && kind == GDWD_BACKEND_SMW2)
    return set_err(ctx, GDWD_ERR_UNSUPPORTED,
                   "SMW2 couples all samples through the n x n Gram: run it unsharded (replicas)");
  const double mu = cfg->mu, mu2 = mu * mu, q = ctx->q, C = ctx->C;
  const int max_iter = cfg->max_iter;

  // ---- buffers ------------------------------------------------------------
  const int NV = 13, MV = 18;
  // Gram space pays off (and keeps w exactly representable) only when n <= d,
  // SMW2's own regime; an explicitly requested SMW2 with d < n iterates over X.
  // DIRECT with few samples (2n <= d, unsharded, n within the persistent
  // kernel's shared-memory budget): the same exact solve done in sample space
  // with SMW2's Gram-space machinery; still reported as DIRECT.  The (d+1)^2
  // factor becomes an n x n one and the iteration runs in one cooperative
  // kernel (c1: n = 1000, d = 2000).
  int skind = kind;
  if (kind == GDWD_BACKEND_DIRECT && cfg->smw_gram_space && !sharded(ctx) && 2 * n <= d && n <= 2500) skind = GDWD_BACKEND_SMW2;
  const bool gram = (skind == GDWD_BACKEND_SMW2) && cfg->smw_gram_space && n <= d;
  CK(ctx->nvec.ensure((size_t)NV * ((n + 1) / 2 * 2)));
  CK(ctx->mvec.ensure((size_t)MV * ((m + 2) / 2 * 2)));
  CK(ctx->tabs.ensure((size_t)2 * (max_iter + 2) + (size_t)std::max<int64_t>(sched_len, 1)));
  CK(ctx->histb.ensure((size_t)(max_iter + 1) * HIST_W));
  if (!ctx->poll_flag) CK(cudaMallocHost(&ctx->poll_flag, 2 * sizeof(int)));
  for (int i = 0; i < 2; ++i)
    if (!ctx->poll_ev[i]) CK(cudaEventCreateWithFlags(&ctx->poll_ev[i], cudaEventDisableTiming));
  for (cudaEvent_t* e : {&ctx->ev_begin, &ctx->ev_loop, &ctx->ev_end})
    if (!*e) CK(cudaEventCreate(e));
  Dev& D = ctx->D;
  D = Dev{};
  D.n = n; D.d = d; D.m = m;
  D.C = C; D.q = q; D.mu = mu; D.mu2 = mu2; D.zscale = ctx->zscale; D.tau = cfg->steplength;
  D.yty = ctx->yty; D.ynorm = sqrt(ctx->yty);
  D.kappa = (q + 1.0) / q * pow(q, 1.0 / (q + 1.0));
  D.e1 = 1.0 / (q + 1.0); D.e2 = q / (q + 1.0); D.qp1 = q + 1.0; D.one_c = 1.0 + C;
  D.tol_feas = cfg->tol_feas; D.tol_cgap = cfg->tol_cgap; D.tol_cap = cfg->tol_cap;
  D.max_iter = max_iter;
  D.y = ctx->y.p; D.e = ctx->e.p; D.wl = ctx->wl.p;
  // every vector slot starts 16-byte aligned (even strides): double2 loads
  // and bulk (TMA) copies of whole vectors
  const int64_t nst = (n + 1) / 2 * 2;
  double* nv = ctx->nvec.p;
  D.r = nv; D.xi = nv + nst; D.al = nv + 2 * nst; D.ztw = nv + 3 * nst; D.rnew = nv + 4 * nst;
  D.dr = nv + 5 * nst; D.ztwb = nv + 6 * nst; D.s1 = nv + 7 * nst; D.g = nv + 8 * nst; D.tq = nv + 9 * nst;
  double* mv = ctx->mvec.p;
  const int64_t ms = (m + 2) / 2 * 2;
  D.u = mv; D.rho = mv + ms; D.h = mv + 2 * ms; D.h2 = mv + 3 * ms; D.xb = mv + 4 * ms; D.x = mv + 5 * ms;
  D.pr = mv + 6 * ms; D.pres = mv + 7 * ms; D.pq = mv + 8 * ms; D.pu = mv + 9 * ms; D.pd = mv + 10 * ms;
  D.pAd = mv + 11 * ms; D.pAq = mv + 12 * ms;
  D.cres = nv + 10 * nst; D.cdiff = nv + 11 * nst; D.aln = nv + 12 * nst;
  D.zp0 = mv + 16 * ms; D.zp1 = mv + 17 * ms;  // fused tail products, zero before iteration 1
  D.bot = d;
  D.wd = D.x; D.ud = D.u; D.rhod = D.rho;
  if (gram) {
    // coefficient vectors (n + 1 <= d + 2 slots) in the same buffers; the
    // d-space outputs get their own slots
    D.bot = n;
    D.wd = mv + 13 * ms; D.ud = mv + 14 * ms; D.rhod = mv + 15 * ms;
  }
  // persistent per-problem vectors: [colsq (d) | zy (d) | jac (m) | jy (n)],
  // each segment at an even (16-byte aligned) offset
  const int64_t dst2 = (d + 1) / 2 * 2, mst2 = (m + 1) / 2 * 2;
  CK(ctx->colsq.ensure((size_t)2 * dst2 + mst2 + 3 * nst + 8));
  D.zy = ctx->colsq.p + dst2;
  D.jac = ctx->colsq.p + 2 * dst2;
  D.jy = ctx->colsq.p + 2 * dst2 + mst2;
  D.kap = D.jy + nst;
  D.gam = D.jy + 2 * nst;
  D.S = ctx->S;
  D.hist = ctx->histb.p;

  // ---- tables (host pow == Python's float pow) -------------------------------
  // eps constant (solver.py:441-445): 1 / max(1, ||Z~||_F), norm reduced on
  // the device at upload
  const double eps_c = isnan(cfg->epsilon_c) ? 1.0 / std::max(1.0, sqrt(get_fro2(ctx))) : cfg->epsilon_c;
  std::vector<double> tab(2 * (size_t)(max_iter + 2) + (size_t)std::max<int64_t>(sched_len, 1), 0.0);
  const double sqrt_n = sqrt((double)ng);
  for (int k = 0; k < max_iter + 2; ++k) {
    tab[k] = eps_c / pow(k + 1.0, 1.5);
    tab[(max_iter + 2) + k] = tab[k] / sqrt_n;
  }
  if (sched && sched_len > 0) std::copy(sched, sched + sched_len, tab.begin() + 2 * (max_iter + 2));
  CK(cudaMemcpyAsync(ctx->tabs.p, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  D.eps_tab = ctx->tabs.p;
  D.tol_tab = ctx->tabs.p + (max_iter + 2);
  D.sched = (sched && sched_len > 0) ? ctx->tabs.p + 2 * (max_iter + 2) : nullptr;
  D.sched_len = (int)sched_len;

  double sigma0 = cfg->sigma0;
  if (isnan(sigma0)) sigma0 = pow(std::min(10.0 * C, (double)ng), q);

  // ---- setup: zy, factor / preconditioner ------------------------------------
  CK(cudaEventRecord(ctx->ev_begin, ctx->st));
  RC(ensure_scratch(ctx, n, d));
  MatView Z = zview(ctx);
  // Z~ y: the border of A in feature space; the Gram-space iteration carries
  // it as the coefficient vector y itself (no pass over X)
  if (!gram) run_zmv(ctx, OpPlainZ{ctx->y.p, nullptr, const_cast<double*>(D.zy), nullptr}, Z, "zmv_zy");
  CK(cudaGetLastError());
  // ITERATIVE on dense data: the d x d Gram as PSQMR's operator when it is
  // much smaller than X (d <= n/4, n the global count) and fits in memory
  ctx->iter_gram = false;
  if (kind == GDWD_BACKEND_ITERATIVE && ctx->has_dense && cfg->iter_gram >= 0) {
    bool want = cfg->iter_gram == 1 || 4 * d <= ng;
    if (want && !(ctx->gdmat.p && ctx->fac_gen == ctx->data_gen)) {
      size_t freeb = 0, totb = 0;
      CK(cudaMemGetInfo(&freeb, &totb));
      const double need = 8.0 * ((double)d * ((d + 1) / 2 * 2) + (double)gram_workspace_doubles(d, n)) * 1.05;
      want = need < (double)freeb;
    }
    ctx->iter_gram = want;
  }
  RC(build_factor(ctx, skind, mu2));
  if (kind != GDWD_BACKEND_ITERATIVE) RC(ensure_scratch(ctx, ctx->fac_rows, ctx->fac_rows + 2));
  RC(ensure_scratch(ctx, n, d));
  // initial iterates (solver.py:447-454); padding slots zeroed first
  CK(cudaMemsetAsync(ctx->nvec.p, 0, (size_t)NV * nst * sizeof(double), ctx->st));
  fill(ctx, D.r, n, 1.0);
  fill(ctx, D.xi, n, 1.0);
  fill(ctx, D.al, n, 0.0);
  fill(ctx, D.ztw, n, 0.0);
  CK(cudaMemsetAsync(ctx->mvec.p, 0, (size_t)MV * ms * sizeof(double), ctx->st));
  CK(cudaMemsetAsync(ctx->histb.p, 0, (size_t)(max_iter + 1) * HIST_W * sizeof(double), ctx->st));
  {
    CK(cudaMemcpyAsync(ctx->Sh, ctx->S, sizeof(Scal), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    const double ys = ctx->Sh->ys, yjy = ctx->Sh->yjy;  // computed by build_factor (SMW2)
    Scal s0;
    memset(&s0, 0, sizeof(s0));
    s0.sigma = sigma0;
    s0.sigma_next = sigma0;
    s0.ys = ys;
    s0.yjy = yjy;
    *ctx->Sh = s0;
    CK(cudaMemcpyAsync(ctx->S, ctx->Sh, sizeof(Scal), cudaMemcpyHostToDevice, ctx->st));
  }
  CK(cudaEventRecord(ctx->ev_loop, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  float setup = 0.f;
  cudaEventElapsedTime(&setup, ctx->ev_begin, ctx->ev_loop);

  ctx->ps_per_iter.assign(max_iter + 1, 0.0);
  ctx->kind = kind;
  ctx->gram = gram;
  ctx->prox = false;  // every solve starts on PSQMR (solver.py:422)
  ctx->ell = cfg->ell;
  ctx->persistent = gram && cfg->persistent && !ctx->prof && !sharded(ctx);
  // fused tail over dense X (zft.cuh): iterates start at r = xi = 1, alpha = 0
  // (solver.py:447-454), so the products it hands to iteration 1 are exactly 0
  ctx->ft = !gram && ctx->has_dense && ft_enabled() && ft_plan(d).cs > 0;
  if (ctx->ft) run_ft(ctx, OpTail{D}, Z, "zft_tail", true);
  ctx->use_sgs = cfg->use_sgs != 0;
  ctx->poll = std::max(1, cfg->poll_every);
  ctx->max_iter = max_iter;
  ctx->max_steps = cfg->psqmr_switch_steps;
  ctx->k_host = 0;
  ctx->psqmr_total = 0;
  ctx->stopped = false;
  ctx->eps_c = eps_c;
  ctx->setup_ms = setup;
  ctx->poll_pending = 0;
  if (ctx->persistent) {
    int nb = 0;
    // 11 vector slots: 3 staged, 6 bulk-copied inputs, y and G^{-1} y/|y|
    const size_t sm = (size_t)(11 * ((n + 3) / 2 * 2)) * sizeof(double);
    const void* kfn = (const void*)gram_smw_persistent3<0>;
    if (sm > 220 * 1024 || cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
      cudaGetLastError();
      ctx->persistent = false;
    }
    if (ctx->persistent) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kfn, PK_THREADS, sm));
    if (nb < 1 || n > (int64_t)PK_MAX_OWN * NUM_SMS) ctx->persistent = false;
    else CK(ctx->pk_part.ensure((size_t)2 * NUM_SMS * PK_NPART + 8));  // + barrier counter
  }
  if (ctx->persistent) {
    // own rows of K and GK resident in tensor memory when n <= 1024 (<= 7
    // rows per CTA, 8 ceil(n/64) words per lane and row); K alone up to
    // n = 2048, GK streamed from L2 in 8-chunk groups whose loads overlap
    // the group's TMEM words (c2: 24.9 vs 27.0 us/iteration streaming both;
    // a fused 16-load variant spilled in-flight registers and was slower).
    int tmem = n <= 1024 ? 2 : (n <= 2048 ? 1 : 0);
    if (getenv("GDWD_PK_TMEM")) {  // diagnostics: 0 L2 only, 1 K in TMEM (n <= 2048), 2 K and GK (n <= 1024)
      const int want = atoi(getenv("GDWD_PK_TMEM"));
      tmem = want >= 2 && n <= 1024 ? 2 : (want >= 1 && n <= 2048 ? 1 : 0);
    }
    const void* kfn = tmem == 2   ? (const void*)gram_smw_persistent3<2>
                      : tmem == 1 ? (const void*)gram_smw_persistent3<1>
                                  : (const void*)gram_smw_persistent3<0>;
    const size_t sm = (size_t)(11 * ((n + 3) / 2 * 2)) * sizeof(double);
    // the TMEM variants allocate all 512 columns per CTA while spinning on
    // grid barriers: a second CTA on the same SM would block in tcgen05.alloc
    // forever.  One CTA per SM holds today by register pressure; enforce it by
    // padding the dynamic shared memory past half an SM if that ever changes.
    size_t sm_launch = sm;
    if (tmem) {
      int nb_tm = 0;
      CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb_tm, kfn, PK_THREADS, sm));
      if (nb_tm > 1) sm_launch = std::max(sm, (size_t)120 * 1024);
    }
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_launch));
    ctx->pk_kfn = kfn;
    ctx->pk_smem = sm_launch;
    CK(cudaMemsetAsync(ctx->pk_part.p + (size_t)2 * NUM_SMS * PK_NPART, 0, sizeof(unsigned), ctx->st));
  }
  // ITERATIVE: the whole body with device-resident PSQMR (graph WHILE nodes),
  // unsharded (an NCCL all-reduce inside a conditional body is not relied on)
  ctx->ps_graph = kind == GDWD_BACKEND_ITERATIVE && cfg->use_graph && !ctx->prof && !sharded(ctx) &&
                  env_int("GDWD_PSQMR_GRAPH", 1) != 0;
  if ((kind != GDWD_BACKEND_ITERATIVE || ctx->ps_graph) && cfg->use_graph && !ctx->prof && !ctx->persistent &&
      ctx->comm_mode != 2) {
    cudaGraph_t graph;
    const int64_t before = ctx->launches;
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    int rc = GDWD_OK;
    if (kind == GDWD_BACKEND_ITERATIVE) rc = body_iterative_dev(ctx, ctx->use_sgs);
    else if (gram) enqueue_body_gram(ctx, ctx->use_sgs);
    else enqueue_body_fixed(ctx, kind, ctx->use_sgs);
    const cudaError_t ce = cudaStreamEndCapture(ctx->st, &graph);
    RC(rc);
    CK(ce);
    ctx->body_nodes = ctx->launches - before;
    ctx->launches = before;
    CK(cudaGraphInstantiate(&ctx->gexec, graph, 0));
    cudaGraphDestroy(graph);
  }
  ctx->in_solve = true;
  return GDWD_OK;
}

// Run up to `count` more iterations (fewer if the stopping rule fires).
extern "C" int gdwd_solve_iterate(gdwd_ctx* ctx, int32_t count, gdwd_iter_cb cb, void* user, int32_t* iters_done,
                                  int32_t* stopped_out) {
  Range nvtx_range("gdwd_solve_iterate (loop)");
  if (!ctx || !ctx->in_solve) return set_err(ctx, GDWD_ERR_VALUE, "no solve in progress");
  CK(cudaSetDevice(ctx->device));
  RC(pk_settle(ctx));
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  int status = GDWD_OK;
  const int kend = std::min(ctx->max_iter, ctx->k_host + std::max(0, count));
  if (ctx->persistent && !cb && ctx->k_host < kend && !ctx->stopped) {
    // one cooperative launch runs all requested iterations (persist3.cuh)
    if (getenv("GDWD_PK_TIMING")) {
      ctx->pk_tsn = (size_t)PK_TS_ITERS * NUM_SMS * 32;
      CK(cudaMalloc(&ctx->pk_ts, ctx->pk_tsn * sizeof(unsigned long long)));
      CK(cudaMemset(ctx->pk_ts, 0, ctx->pk_tsn * sizeof(unsigned long long)));
    }
    const int diag = getenv("GDWD_PK_DIAG") ? atoi(getenv("GDWD_PK_DIAG")) : 0;
    // 3 grid barriers per iteration (persist3.cuh)
    unsigned* ctr = nullptr;  // zeroed at solve_begin; Scal.pk_bar carries its value between launches
    if (!(getenv("GDWD_PK_BAR") && atoi(getenv("GDWD_PK_BAR")) == 0))
      ctr = reinterpret_cast<unsigned*>(ctx->pk_part.p + (size_t)2 * NUM_SMS * PK_NPART);
    PK3Args pa{D, ctx->kmat.p, ctx->gkmat.p, D.kap, D.gam, ctx->ldm, ctx->pk_part.p, kend - ctx->k_host,
               diag, ctx->pk_ts, ctx->use_sgs ? 1 : 0, ctr};
    void* args[] = {&pa};
    Launch L(ctx, "persistent_gram_smw2");
    CK(cudaLaunchCooperativeKernel(ctx->pk_kfn, dim3(NUM_SMS), dim3(PK_THREADS), args, ctx->pk_smem, ctx->st));
    ctx->pk_pending = true;
    ctx->pk_kend = kend;
    ctx->k_host = kend;  // tentative until pk_settle reads the stop flag back
    if (!ctx->pk_defer) RC(pk_settle(ctx));
  }
  // the callback of iteration k: complete its KKT record (dual objective,
  // gap, stop test), materialise w/u/rho, hand the row to the host
  auto callback = [&](int k, bool* stop) -> int {
    *stop = false;
    if (ctx->gram) run_zt(ctx, GsKAlpha{D}, MatView{ctx->kmat.p, ctx->n, ctx->n, ctx->ldm}, "gemv_K_alpha");
    else enqueue_rhs(ctx);
    enqueue_materialize(ctx);
    CK(cudaMemcpyAsync(ctx->Sh, ctx->S, sizeof(Scal), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    const Scal& s = *ctx->Sh;
    if (s.error) {
      *stop = true;
      return GDWD_OK;
    }
    if (s.iters_done == k + 1) {
      double hrow[HIST_W];
      CK(cudaMemcpy(hrow, D.hist + (int64_t)k * HIST_W, sizeof(hrow), cudaMemcpyDeviceToHost));
      double res11[11];
      for (int f = 0; f < 11; ++f)
        res11[f] = (f < 8) ? hrow[f] : (f == 8 ? hrow[H_GAP] : (f == 9 ? hrow[H_OBJP] : hrow[H_OBJD]));
      if (cb(user, k + 1, res11, hrow[H_SIGMA], hrow[H_BETA]) != 0)
        return set_err(ctx, GDWD_ERR_ABORTED, "callback requested abort");
    }
    *stop = s.stopped != 0;
    return GDWD_OK;
  };
  for (;;) {
    while (ctx->k_host < kend && !ctx->stopped) {
      const int k = ctx->k_host;
      const bool iter_host = ctx->kind == GDWD_BACKEND_ITERATIVE && (!ctx->ps_graph || !ctx->gexec || ctx->prox);
      if (iter_host) {
        int steps = 0;
        status = body_iterative(ctx, ctx->use_sgs, ctx->max_steps, &steps);
        if (status) break;
        ctx->psqmr_total += steps;
        ctx->ps_per_iter[k] = steps;
      } else if (ctx->gexec) {
        CK(cudaGraphLaunch(ctx->gexec, ctx->st));
        ctx->launches += ctx->body_nodes;
      } else if (ctx->gram) {
        enqueue_body_gram(ctx, ctx->use_sgs);
      } else {
        enqueue_body_fixed(ctx, ctx->kind, ctx->use_sgs);
      }
      CK(cudaGetLastError());
      ctx->k_host = k + 1;
      if (ctx->prof) prof_flush(ctx);
      if (cb) {
        bool stop = false;
        status = callback(k, &stop);
        if (status) break;
        ctx->stopped = stop;
      } else if (iter_host && !ctx->prox) {
        ctx->stopped = ctx->Sh->stopped != 0;  // synced inside the PSQMR loop
      } else if ((k + 1) % ctx->poll == 0) {
        // lagged poll: read the flag copied one poll interval ago (the GPU
        // still has this interval queued, so it never idles on the host)
        const int sl = ctx->poll_slot;
        CK(cudaMemcpyAsync(ctx->poll_flag + sl, &ctx->S->stopped, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaEventRecord(ctx->poll_ev[sl], ctx->st));
        if (ctx->poll_pending) {
          CK(cudaEventSynchronize(ctx->poll_ev[sl ^ 1]));
          if (ctx->poll_flag[sl ^ 1]) ctx->stopped = true;
        }
        ctx->poll_pending = 1;
        ctx->poll_slot = sl ^ 1;
      }
    }
    // a device-resident PSQMR solve that needs the proximal switch stopped
    // the graph iterations: finish that iteration on the host and go on
    if (status || !ctx->ps_graph || ctx->prox || !(ctx->stopped || ctx->k_host >= kend)) break;
    int resumed = 0;
    status = prox_resume(ctx, ctx->use_sgs, &resumed);
    if (status || !resumed) break;
    ctx->poll_pending = 0;
    if (cb) {
      bool stop = false;
      status = callback(ctx->k_host - 1, &stop);
      if (status) break;
      ctx->stopped = stop;
    }
  }
  if (ctx->prof) prof_flush(ctx);
  if (iters_done) *iters_done = ctx->k_host;
  if (stopped_out) *stopped_out = ctx->stopped ? 1 : 0;
  if (status) end_session(ctx);
  return status;
}

// GDWD_FT_TIMING: median per-tile intervals of the fused pass's roles (CTA 0, last launch)
static void ft_timing_report(gdwd_ctx* ctx) {
  std::vector<unsigned long long> h((size_t)FT_TS_TILES * FT_TS_PTS);
  cudaMemcpy(h.data(), ctx->ft_ts, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  struct Iv { const char* name; int a, b; bool next; };
  const Iv ivs[] = {{"prod: wait empty", 0, 1, false}, {"dot: wait xfree", 2, 13, false}, {"dot: fma loop", 13, 14, false},
                    {"dot: shuffle sums", 14, 15, false}, {"dot: publish", 15, 3, false},
                    {"axpy: wait full", 4, 5, false}, {"axpy: wait ts", 5, 6, false}, {"axpy: axpy", 6, 7, false},
                    {"sw: wait dots", 8, 9, false}, {"sw: combine+input", 9, 10, false}, {"sw: prefetch+wait tsfree", 10, 11, false},
                    {"sw: ts handoff", 11, 12, false}, {"sw: period", 8, 8, true}, {"axpy: period", 4, 4, true},
                    {"prod: period", 0, 0, true}};
  for (const Iv& iv : ivs) {
    std::vector<double> v;
    for (int t = 4; t + 1 < FT_TS_TILES; ++t) {
      const unsigned long long* a = &h[(size_t)t * FT_TS_PTS];
      const unsigned long long* b = iv.next ? &h[(size_t)(t + 1) * FT_TS_PTS] : a;
      if (!a[iv.a] || !b[iv.b]) continue;
      v.push_back((double)(b[iv.b] - a[iv.a]));
    }
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    fprintf(stderr, "zft timing %-26s median %7.0f ns  p90 %7.0f ns  (n=%zu)\n", iv.name, v[v.size() / 2],
            v[v.size() * 9 / 10], v.size());
  }
}

extern "C" int gdwd_solve_end(gdwd_ctx* ctx, gdwd_result* out) {
  Range nvtx_range("gdwd_solve_end");
  if (!ctx || !ctx->in_solve || !out) return set_err(ctx, GDWD_ERR_VALUE, "no solve in progress");
  CK(cudaSetDevice(ctx->device));
  RC(pk_settle(ctx));
  if (ctx->ft_ts) {
    cudaDeviceSynchronize();
    ft_timing_report(ctx);
  }
  memset(out, 0, sizeof(*out));
  const Dev& D = ctx->D;
  MatView Z = zview(ctx);
  // final pass: dual objective / gap / stop test of the last iteration
  if (ctx->gram) run_zt(ctx, GsKAlpha{D}, MatView{ctx->kmat.p, ctx->n, ctx->n, ctx->ldm}, "gemv_K_alpha");
  else enqueue_rhs(ctx);
  enqueue_materialize(ctx);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev_end, ctx->st));
  CK(cudaMemcpyAsync(ctx->Sh, ctx->S, sizeof(Scal), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  if (ctx->prof) prof_flush(ctx);
  const Scal s = *ctx->Sh;
  float ms_loop = 0;
  cudaEventElapsedTime(&ms_loop, ctx->ev_loop, ctx->ev_end);
  end_session(ctx);
  if (s.error == 6) return set_err(ctx, GDWD_ERR_ASSERT, "margin iterate left the positive orthant");
  ctx->hist_rows = s.iters_done;
  ctx->hist_ps_dev = ctx->ps_graph;
  ctx->last_kind = ctx->kind;
  out->iterations = s.iters_done;
  out->converged = s.converged;
  out->backend = ctx->kind;
  out->psqmr_total = ctx->psqmr_total + s.ps_total;  // host-driven + device-resident PSQMR steps
  if (ctx->ps_graph) ctx->launches += (int64_t)s.ps_total * ctx->ps_step_nodes;
  out->double_count = s.double_count;
  out->status = 0;
  out->sigma = s.sigma;
  out->eps_c = ctx->eps_c;
  out->setup_ms = ctx->setup_ms;
  out->loop_ms = ms_loop;
  double bet = 0.0;
  CK(cudaMemcpy(&bet, D.wd + ctx->d, sizeof(double), cudaMemcpyDeviceToHost));
  out->beta = bet;
  for (int f = 0; f < 11; ++f) out->resid[f] = s.eta[f];
  return GDWD_OK;
}

extern "C" int gdwd_solve(gdwd_ctx* ctx, const gdwd_config* cfg, const double* sched, int64_t sched_len,
                          gdwd_iter_cb cb, void* user, gdwd_result* out) {
  if (!out) return set_err(ctx, GDWD_ERR_VALUE, "null result");
  RC(gdwd_solve_begin(ctx, cfg, sched, sched_len));
  RC(gdwd_solve_iterate(ctx, cfg->max_iter, cb, user, nullptr, nullptr));
  return gdwd_solve_end(ctx, out);
}

extern "C" int gdwd_set_lanczos_start(gdwd_ctx* ctx, const double* v, int64_t d) {
  if (!ctx || !v || d != ctx->d) return set_err(ctx, GDWD_ERR_VALUE, "start vector must have length d");
  ctx->lz_start.assign(v, v + d);
  return GDWD_OK;
}

extern "C" int gdwd_frobenius_sq(gdwd_ctx* ctx, double* out) {
  if (!ctx || !out || get_fro2(ctx) < 0) return set_err(ctx, GDWD_ERR_VALUE, "no data uploaded");
  *out = ctx->fro2;
  return GDWD_OK;
}

// ---------------------------------------------------------------------------
// sample sharding
// ---------------------------------------------------------------------------
static int comm_finish_init(gdwd_ctx* ctx, int32_t nranks, int32_t rank, int64_t n_global) {
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->n_global = n_global;
  ctx->data_gen++;  // factors depend on the global data
  // global ||Z~||_F^2 and check of the global sample count
  DevBuf tmp;
  CK(tmp.ensure(2));
  double hv[2] = {get_fro2(ctx), (double)ctx->n};
  // on st (non-blocking): a legacy-stream copy is not ordered before the all-reduce's reads
  CK(cudaMemcpyAsync(tmp.p, hv, sizeof(hv), cudaMemcpyHostToDevice, ctx->st));
  allreduce(ctx, tmp.p, 2);
  CK(cudaMemcpyAsync(hv, tmp.p, sizeof(hv), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  tmp.release();
  if (ctx->comm_err) return set_err(ctx, GDWD_ERR_CUDA, "all-reduce failed during communicator setup");
  if ((int64_t)hv[1] != n_global)
    return set_err(ctx, GDWD_ERR_VALUE, "shard sizes do not add up to n_global (sum " + std::to_string(hv[1]) +
                                            ", n_global " + std::to_string(n_global) + ", local " +
                                            std::to_string(ctx->n) + ")");
  ctx->fro2 = hv[0];
  ctx->yty = (double)n_global;  // labels are +-1 (validated in set_problem)
  return GDWD_OK;
}

extern "C" int gdwd_comm_unique_id(uint8_t* out128) {
  if (!out128) return GDWD_ERR_VALUE;
  if (!nccl::api().ok) return GDWD_ERR_UNSUPPORTED;
  nccl::UniqueId id;
  if (nccl::api().GetUniqueId(&id) != 0) return GDWD_ERR_CUDA;
  memcpy(out128, id.internal, 128);
  return GDWD_OK;
}

extern "C" int gdwd_comm_init_nccl(gdwd_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id128,
                                   int64_t n_global) {
  if (!ctx || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return set_err(ctx, GDWD_ERR_VALUE, "bad comm arguments");
  if (!ctx->has_problem) return set_err(ctx, GDWD_ERR_VALUE, "set the local problem before the communicator");
  if (!nccl::api().ok) return set_err(ctx, GDWD_ERR_UNSUPPORTED, "libnccl.so.2 not found");
  CK(cudaSetDevice(ctx->device));
  nccl::UniqueId id;
  memcpy(id.internal, id128, 128);
  const nccl::Result r = nccl::api().CommInitRank(&ctx->comm, nranks, id, rank);
  if (r != 0) return set_err(ctx, GDWD_ERR_CUDA, std::string("ncclCommInitRank: ") + nccl::api().GetErrorString(r));
  ctx->comm_mode = 1;
  return comm_finish_init(ctx, nranks, rank, n_global);
}

extern "C" int gdwd_comm_init_host(gdwd_ctx* ctx, int32_t nranks, int32_t rank, gdwd_allreduce_cb cb, void* user,
                                   int64_t n_global) {
  if (!ctx || !cb || nranks < 1 || rank < 0 || rank >= nranks) return set_err(ctx, GDWD_ERR_VALUE, "bad comm arguments");
  if (!ctx->has_problem) return set_err(ctx, GDWD_ERR_VALUE, "set the local problem before the communicator");
  CK(cudaSetDevice(ctx->device));
  ctx->host_ar = cb;
  ctx->host_ar_user = user;
  ctx->comm_mode = 2;
  return comm_finish_init(ctx, nranks, rank, n_global);
}

// Sum of a host vector over the shards of the attached communicator (the
// identity without one): the host side's n-sums, e.g. the global train error.
extern "C" int gdwd_allreduce_host(gdwd_ctx* ctx, double* buf, int64_t count) {
  if (!ctx || (!buf && count > 0) || count < 0) return set_err(ctx, GDWD_ERR_VALUE, "bad all-reduce arguments");
  if (!ctx->comm_mode || count == 0) return GDWD_OK;
  CK(cudaSetDevice(ctx->device));
  DevBuf tmp;
  CK(tmp.ensure(count));
  CK(cudaMemcpyAsync(tmp.p, buf, count * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  allreduce(ctx, tmp.p, count);
  CK(cudaMemcpyAsync(buf, tmp.p, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  tmp.release();
  if (ctx->comm_err) return set_err(ctx, GDWD_ERR_CUDA, "all-reduce failed");
  return GDWD_OK;
}

extern "C" int gdwd_set_profile(gdwd_ctx* ctx, int32_t enable) {
  if (!ctx) return GDWD_ERR_VALUE;
  ctx->prof = enable != 0;
  if (!ctx->prof) ctx->prof_acc.clear();
  return GDWD_OK;
}

extern "C" int gdwd_get_profile(gdwd_ctx* ctx, char* buf, int64_t buflen, int64_t* launches) {
  if (!ctx) return GDWD_ERR_VALUE;
  if (launches) *launches = ctx->launches;
  if (buf && buflen > 0) {
    std::string txt;
    char line[256];
    for (auto& kv : ctx->prof_acc) {
      snprintf(line, sizeof(line), "%s %lld %.6f\n", kv.first.c_str(), (long long)kv.second.first, kv.second.second);
      txt += line;
    }
    strncpy(buf, txt.c_str(), (size_t)buflen - 1);
    buf[buflen - 1] = 0;
  }
  return GDWD_OK;
}

extern "C" int gdwd_reset_counters(gdwd_ctx* ctx) {
  if (!ctx) return GDWD_ERR_VALUE;
  ctx->launches = 0;
  ctx->prof_acc.clear();
  return GDWD_OK;
}

// Device time (ms) of `count` iterations of the current solve, CUDA events on
// the solve's stream, with a synchronize on both sides.
extern "C" int gdwd_time_iterations(gdwd_ctx* ctx, int32_t count, double* ms, int32_t* iters_done) {
  if (!ctx || !ctx->in_solve || !ms) return set_err(ctx, GDWD_ERR_VALUE, "no solve in progress");
  CK(cudaSetDevice(ctx->device));  // events belong to the context's device (one host thread per GPU)
  CK(cudaStreamSynchronize(ctx->st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, ctx->st));
  int32_t st = 0;
  ctx->pk_defer = true;  // a persistent launch is read back after the end event
  const int rc = gdwd_solve_iterate(ctx, count, nullptr, nullptr, iters_done, &st);
  ctx->pk_defer = false;
  RC(rc);
  CK(cudaEventRecord(b, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  RC(pk_settle(ctx));
  if (iters_done) *iters_done = ctx->k_host;
  float f = 0.f;
  cudaEventElapsedTime(&f, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms = f;
  return GDWD_OK;
}

extern "C" int gdwd_get_state(gdwd_ctx* ctx, double* r, double* xi, double* alpha, double* w, double* u,
                              double* rho, double* ztw, double* beta) {
  Range nvtx_range("gdwd_get_state (download)");
  if (!ctx || !ctx->nvec.p) return set_err(ctx, GDWD_ERR_VALUE, "no solve state");
  CK(cudaSetDevice(ctx->device));
  const Dev& D = ctx->D;
  const int64_t n = ctx->n, d = ctx->d;
  struct P { double* h; const double* dp; int64_t len; } items[] = {
      {r, D.r, n}, {xi, D.xi, n}, {alpha, D.al, n}, {ztw, D.ztw, n}, {w, D.wd, d}, {u, D.ud, d}, {rho, D.rhod, d}, {beta, D.wd + d, 1}};
  // through the context's page-locked staging block when everything fits:
  // the copies run back to back without a staged (synchronous) transfer each
  double* stage = ctx->aux ? ((CtxAux*)ctx->aux)->stage : nullptr;
  size_t tot = 0;
  for (auto& it : items)
    if (it.h) tot += (size_t)it.len;
  if (stage && tot <= CTX_STAGE_DOUBLES) {
    size_t off = 0;
    for (auto& it : items)
      if (it.h) {
        CK(cudaMemcpyAsync(stage + off, it.dp, it.len * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
        off += (size_t)it.len;
      }
    CK(cudaStreamSynchronize(ctx->st));
    off = 0;
    for (auto& it : items)
      if (it.h) {
        memcpy(it.h, stage + off, it.len * sizeof(double));
        off += (size_t)it.len;
      }
    return GDWD_OK;
  }
  for (auto& it : items)
    if (it.h) CK(cudaMemcpyAsync(it.h, it.dp, it.len * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return GDWD_OK;
}

extern "C" int gdwd_get_history(gdwd_ctx* ctx, double* hist, int64_t max_rows, int64_t* rows) {
  if (!ctx || !hist || !rows) return set_err(ctx, GDWD_ERR_VALUE, "null argument");
  int64_t nr = std::min(max_rows, ctx->hist_rows);
  if (nr > 0) {
    double* stage = ctx->aux ? ((CtxAux*)ctx->aux)->stage : nullptr;
    if (stage && (size_t)nr * HIST_W <= CTX_STAGE_DOUBLES) {
      CK(cudaMemcpyAsync(stage, ctx->histb.p, nr * HIST_W * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
      CK(cudaStreamSynchronize(ctx->st));
      memcpy(hist, stage, nr * HIST_W * sizeof(double));
    } else {
      CK(cudaMemcpy(hist, ctx->histb.p, nr * HIST_W * sizeof(double), cudaMemcpyDeviceToHost));
    }
    // host-driven PSQMR counts its steps on the host; the device-resident
    // one records them in the history itself (OpPsEnd)
    if (!ctx->hist_ps_dev)
      for (int64_t k = 0; k < nr && k < (int64_t)ctx->ps_per_iter.size(); ++k) hist[k * HIST_W + H_PSQMR] = ctx->ps_per_iter[k];
  }
  *rows = nr;
  return GDWD_OK;
}

// ---------------------------------------------------------------------------
// standalone seams
// ---------------------------------------------------------------------------
namespace {
struct Tmp {
  std::vector<void*> ptrs;
  ~Tmp() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return (T*)p;
  }
};

// Dense symmetric operator for standalone PSQMR: Aq = A q, fused q.Aq
struct OpDenseApply {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return !D.S->ps_active; }
  GDWD_DEV double wval(int64_t j) const { return D.pq[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const {
    D.pAq[i] = dot;
    na[0] += D.pq[i] * dot;
  }
  GDWD_DEV void fin(const double (&ns)[NN]) const {
    Scal* S = D.S;
    if (fabs(ns[0]) < TINY) {
      S->ps_brk = 1;
      S->ps_active = 0;
      return;
    }
    S->ps_alpha = S->ps_rho / ns[0];
  }
};
struct OpDenseInitRes {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  const double* x0;
  const double* b;
  double* r;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV double wval(int64_t j) const { return x0[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const { r[i] = b[i] - dot; }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};
}  // namespace

extern "C" int gdwd_newton_sweep(int32_t device, int64_t n, const double* a, double sigma, double q,
                                 const double* w, const double* r0, double tol, int32_t max_newton,
                                 int32_t scalar_form, double* out, int32_t* iters) {
  gdwd_ctx* ctx = nullptr;
  if (n < 0 || !a || !w || !r0 || !out) return GDWD_ERR_VALUE;
  if (!(sigma > 0 && q > 0)) return GDWD_ERR_VALUE;
  if (n == 0) return GDWD_OK;
  if (cudaSetDevice(device) != cudaSuccess) return GDWD_ERR_CUDA;
  Tmp t;
  double *da = t.alloc<double>(n), *dw = t.alloc<double>(n), *dr = t.alloc<double>(n), *dout = t.alloc<double>(n);
  int* dit = t.alloc<int>(n);
  if (!da || !dw || !dr || !dout || !dit) return GDWD_ERR_CUDA;
  CK(cudaMemcpy(da, a, n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, w, n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dr, r0, n * 8, cudaMemcpyHostToDevice));
  OpNewtonSweep op{da, dw, dr, dout, dit, sigma, q, tol, max_newton, scalar_form};
  if (scalar_form & 2) newton_warp_kernel<<<(unsigned)std::min<int64_t>((n + 7) / 8, 4 * NUM_SMS), 256>>>(op, n);
  else vmap_kernel<OpNewtonSweep><<<vm_grid(n), VM_THREADS>>>(op, n, Scratch{});
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost));
  if (iters) CK(cudaMemcpy(iters, dit, n * 4, cudaMemcpyDeviceToHost));
  return GDWD_OK;
}

extern "C" int gdwd_chol_inverse(int32_t device, const double* Sm, int64_t m, double* inv_out) {
  gdwd_ctx* ctx = nullptr;
  if (m < 1 || !Sm || !inv_out) return GDWD_ERR_VALUE;
  if (cudaSetDevice(device) != cudaSuccess) return GDWD_ERR_CUDA;
  Tmp t;
  const int64_t ld = (m + 1) / 2 * 2;
  double* A = t.alloc<double>((size_t)m * ld);
  double* W = t.alloc<double>((size_t)2 * m * ld);
  int* info = t.alloc<int>(1);
  if (!A || !W || !info) return GDWD_ERR_CUDA;
  CK(cudaMemcpy2D(A, ld * 8, Sm, m * 8, m * 8, m, cudaMemcpyHostToDevice));
  CK(cudaMemset(info, 0, sizeof(int)));
  CK(chol_inverse(A, W, W + (size_t)m * ld, ld, m, info, 0));
  int h = 0;
  CK(cudaMemcpy(&h, info, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) return GDWD_ERR_INDEFINITE;
  CK(cudaMemcpy2D(inv_out, m * 8, A, ld * 8, m * 8, m, cudaMemcpyDeviceToHost));
  return GDWD_OK;
}

// Test seam: the n x n Gram K = Z~^T Z~ and (when the upload also factored)
// G^{-1} = (K/mu^2 + I)^{-1} that a page-locked upload in the sample-space
// regimes formed block by block.  *have: bit 0 = K, bit 1 = G^{-1}.
extern "C" int gdwd_get_upload_factor(gdwd_ctx* ctx, double* K_out, double* Ginv_out, int32_t* have) {
  if (!ctx || !have) return set_err(ctx, GDWD_ERR_VALUE, "null argument");
  CK(cudaSetDevice(ctx->device));
  *have = 0;
  const int64_t n = ctx->n, ldk = (n + 1) / 2 * 2;
  CK(cudaStreamSynchronize(ctx->st));
  if (ctx->has_dense && ctx->k_gen == ctx->zs_gen && ctx->kmat.p) {
    *have |= 1;
    if (K_out) CK(cudaMemcpy2D(K_out, n * 8, ctx->kmat.p, ldk * 8, n * 8, n, cudaMemcpyDeviceToHost));
  }
  if (ctx->has_dense && ctx->pf_gen == ctx->zs_gen && ctx->fac.p) {
    *have |= 2;
    if (Ginv_out) CK(cudaMemcpy2D(Ginv_out, n * 8, ctx->fac.p, ldk * 8, n * 8, n, cudaMemcpyDeviceToHost));
  }
  return GDWD_OK;
}

// The same inverse by the bordered (row-block) chain the pipelined upload
// runs: blocks of `block` rows, three streams as in upload_dense_pipelined.
extern "C" int gdwd_chol_inverse_bordered(int32_t device, const double* Sm, int64_t m, int32_t block,
                                          double* inv_out) {
  gdwd_ctx* ctx = nullptr;
  if (m < 1 || block < 1 || !Sm || !inv_out) return GDWD_ERR_VALUE;
  if (cudaSetDevice(device) != cudaSuccess) return GDWD_ERR_CUDA;
  Tmp t;
  const int64_t ld = (m + 1) / 2 * 2;
  double* A = t.alloc<double>((size_t)m * ld);
  const int64_t bws = bordered_workspace(m, block);
  double* W = t.alloc<double>((size_t)3 * m * ld + (size_t)bws);
  int* info = t.alloc<int>(1);
  if (!A || !W || !info) return GDWD_ERR_CUDA;
  double* Wi = W;
  double* T = W + (size_t)m * ld;
  double* Ginv = W + (size_t)2 * m * ld;
  CK(cudaMemcpy2D(A, ld * 8, Sm, m * 8, m * 8, m, cudaMemcpyHostToDevice));
  CK(cudaMemset(info, 0, sizeof(int)));
  CK(cudaMemset(W, 0, (size_t)3 * m * ld * 8));
  CK(cudaStreamSynchronize(cudaStreamLegacy));  // the streams below are non-blocking: inputs must have landed
  cudaStream_t s3[3];
  for (auto& x : s3) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  cudaError_t e = cudaSuccess;
  for (int64_t r0 = 0; r0 < m && e == cudaSuccess; r0 += block)
    e = bordered_chol_step(A, Wi, T, Ginv, ld, r0, std::min<int64_t>(m, r0 + block), info, s3[0], s3[1], s3[2],
                           W + (size_t)3 * m * ld, bws);
  if (e == cudaSuccess) e = mirror_lower(Ginv, ld, m, s3[2]);
  for (auto& x : s3) {
    cudaStreamSynchronize(x);
    cudaStreamDestroy(x);
  }
  CK(e);
  int h = 0;
  CK(cudaMemcpy(&h, info, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) return GDWD_ERR_INDEFINITE;
  CK(cudaMemcpy2D(inv_out, m * 8, Ginv, ld * 8, m * 8, m, cudaMemcpyDeviceToHost));
  return GDWD_OK;
}

extern "C" int gdwd_gram(int32_t device, const double* X, int64_t rows, int64_t cols, int32_t sum_over_rows,
                         double div, double shift, double* outp) {
  gdwd_ctx* ctx = nullptr;
  if (rows < 1 || cols < 1 || !X || !outp) return GDWD_ERR_VALUE;
  if (cudaSetDevice(device) != cudaSuccess) return GDWD_ERR_CUDA;
  Tmp t;
  const int64_t ld = (cols + 1) / 2 * 2;
  const int64_t M = sum_over_rows ? cols : rows, K = sum_over_rows ? rows : cols;
  double* dX = t.alloc<double>((size_t)rows * ld);
  double* C = t.alloc<double>((size_t)M * M);
  double* W = t.alloc<double>((size_t)gram_workspace_doubles(M, K));
  if (!dX || !C || !W) return GDWD_ERR_CUDA;
  CK(cudaMemset(dX, 0, (size_t)rows * ld * 8));
  CK(cudaMemcpy2D(dX, ld * 8, X, cols * 8, cols * 8, rows, cudaMemcpyHostToDevice));
  CK(gram_syrk(dX, rows, cols, ld, sum_over_rows != 0, div, shift, C, M, W, 0));
  CK(cudaMemcpy(outp, C, (size_t)M * M * 8, cudaMemcpyDeviceToHost));
  return GDWD_OK;
}

// Device time of the one-time Gram of the resident dense Z~ (the FP64
// tensor-core SYRK the DIRECT / SMW2 / Gram-operator setups run): the smaller
// side's Gram, averaged over `reps` launches after one warm-up (CUDA events).
extern "C" int gdwd_time_gram(gdwd_ctx* ctx, int32_t reps, double* ms) {
  if (!ctx || !ms || reps < 1) return set_err(ctx, GDWD_ERR_VALUE, "bad arguments");
  if (!ctx->has_dense) return set_err(ctx, GDWD_ERR_VALUE, "no dense data");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = ctx->n, d = ctx->d;
  const bool rows = n >= d;  // Z~ Z~^T (d x d) when samples dominate, else Z~^T Z~ (n x n)
  const int64_t M = rows ? d : n, K = rows ? n : d, ld = (M + 1) / 2 * 2;
  DevBuf c, w;
  CK(c.ensure((size_t)M * ld));
  CK(w.ensure((size_t)gram_workspace_doubles(M, K)));
  CK(gram_syrk(ctx->Zs, n, d, ctx->ldz, rows, 1.0, 0.0, c.p, ld, w.p, ctx->st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, ctx->st));
  for (int r = 0; r < reps; ++r) CK(gram_syrk(ctx->Zs, n, d, ctx->ldz, rows, 1.0, 0.0, c.p, ld, w.p, ctx->st));
  CK(cudaEventRecord(b, ctx->st));
  CK(cudaEventSynchronize(b));
  float f = 0.f;
  cudaEventElapsedTime(&f, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  c.release();
  w.release();
  *ms = f / reps;
  return GDWD_OK;
}

extern "C" int gdwd_psqmr_dense(int32_t device, const double* A, int64_t m, const double* b, const double* M,
                                double tol, int32_t max_iter, const double* x0, double* x_out, int32_t* info,
                                double* resnorm) {
  if (m < 1 || !A || !b || !x_out || !info) return GDWD_ERR_VALUE;
  if (cudaSetDevice(device) != cudaSuccess) return GDWD_ERR_CUDA;
  gdwd_ctx* ctx = nullptr;
  Tmp t;
  const int64_t ld = (m + 1) / 2 * 2;
  double* dA = t.alloc<double>((size_t)m * ld);
  double* vec = t.alloc<double>((size_t)12 * (m + 1));
  Scal* S = t.alloc<Scal>(1);
  size_t npn = (size_t)NUM_SMS * 32 * 16 + 64;
  double* npart = t.alloc<double>(npn);
  double* part = t.alloc<double>((size_t)8 * (m + 1));
  unsigned* tk = t.alloc<unsigned>(NUM_SMS * 32 + 8);
  if (!dA || !vec || !S || !npart || !part || !tk) return GDWD_ERR_CUDA;
  CK(cudaMemset(dA, 0, (size_t)m * ld * 8));
  CK(cudaMemcpy2D(dA, ld * 8, A, m * 8, m * 8, m, cudaMemcpyHostToDevice));
  CK(cudaMemset(vec, 0, (size_t)12 * (m + 1) * 8));
  CK(cudaMemset(tk, 0, (NUM_SMS * 32 + 8) * sizeof(unsigned)));
  const int64_t s = m + 1;
  Dev D{};
  D.m = m;
  double* bb = vec;
  double* x0d = vec + s;
  double* jac = vec + 2 * s;
  D.pr = vec + 3 * s; D.pres = vec + 4 * s; D.pq = vec + 5 * s; D.pu = vec + 6 * s; D.pd = vec + 7 * s;
  D.pAd = vec + 8 * s; D.pAq = vec + 9 * s;
  double* xo = vec + 10 * s;
  double* epsd = vec + 11 * s;
  D.jac = jac;
  D.S = S;
  D.eps_tab = epsd;
  CK(cudaMemcpy(bb, b, m * 8, cudaMemcpyHostToDevice));
  if (x0) CK(cudaMemcpy(x0d, x0, m * 8, cudaMemcpyHostToDevice));
  std::vector<double> jh(m, 1.0);
  if (M) std::copy(M, M + m, jh.begin());
  CK(cudaMemcpy(jac, jh.data(), m * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(epsd, &tol, 8, cudaMemcpyHostToDevice));
  Scal s0;
  memset(&s0, 0, sizeof(s0));
  CK(cudaMemcpy(S, &s0, sizeof(Scal), cudaMemcpyHostToDevice));
  Scratch scr{part, npart, npart + (npn - 32), tk};
  MatView Av{dA, m, m, ld};
  ZtGeom g = zt_geom(m, ld, NUM_SMS);
  size_t sm = (size_t)(g.cw + ZT_BATCH) * 8;
  ztmv_kernel<OpDenseInitRes><<<dim3(g.chunks, g.ranges), ZT_THREADS, sm>>>(OpDenseInitRes{x0d, bb, D.pr}, Av, g, scr);
  vmap_kernel<OpPsInit><<<vm_grid(m), VM_THREADS>>>(OpPsInit{D, x0d, xo, 0, 1.0}, m, scr);
  CK(cudaGetLastError());
  Scal h;
  for (int it = 0; it <= max_iter; ++it) {
    CK(cudaMemcpy(&h, S, sizeof(Scal), cudaMemcpyDeviceToHost));
    if (!h.ps_active || it == max_iter) break;
    ztmv_kernel<OpDenseApply><<<dim3(g.chunks, g.ranges), ZT_THREADS, sm>>>(OpDenseApply{D}, Av, g, scr);
    vmap_kernel<OpPsV1><<<vm_grid(m), VM_THREADS>>>(OpPsV1{D}, m, scr);
    vmap_kernel<OpPsV2><<<vm_grid(m), VM_THREADS>>>(OpPsV2{D, xo, 1.0, max_iter}, m, scr);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpy(x_out, xo, m * 8, cudaMemcpyDeviceToHost));
  info[0] = h.ps_iters;
  info[1] = h.ps_conv;
  info[2] = h.ps_brk;
  info[3] = 0;
  if (resnorm) *resnorm = h.ps_resn;
  return GDWD_OK;
}
