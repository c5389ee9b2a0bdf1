// api.cu -- the C ABI of include/srl.h: validation, the model context, the step schedule
// and the NCCL plumbing (a6).  Every compute step runs in this library's kernels.
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include "internal.h"
#include "srl.h"

namespace srl {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

// SRL_TANH=accurate: rational tanh (rel. err ~2e-7) instead of MUFU.TANH (~5e-4)
static bool ar_overlap() {
  static int on = -1;
  if (on < 0) { const char* e = getenv("SRL_AR_OVERLAP"); on = (e && e[0] == '1') ? 1 : 0; }
  return on == 1;
}

// SRL_P2P_AR=0: gradient allreduce through NCCL instead of the NVLink peer-memory kernel
static bool p2p_ar_enabled() {
  const char* e = getenv("SRL_P2P_AR");
  return !(e && e[0] == '0');
}

static bool tanh_accurate() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SRL_TANH");
    on = (e && e[0] == 'a') ? 1 : 0;
  }
  return on == 1;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SRL_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace srl

using namespace srl;

#define FAIL(code, msg)            \
  do {                             \
    set_error(msg);                \
    return code;                   \
  } while (0)
#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess)                                                          \
      FAIL(SRL_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));              \
  } while (0)
#define CKN(x)                                                                      \
  do {                                                                              \
    ncclResult_t r_ = (x);                                                          \
    if (r_ != ncclSuccess) FAIL(SRL_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

static srl_status require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    FAIL(SRL_ECUDA, "no CUDA device (libsrl has no CPU fallback)");
  return SRL_OK;
}

extern "C" const char* srl_last_error(void) { return g_err.c_str(); }
extern "C" int srl_abi_version(void) { return 3; }

// ------------------------------------------------------------------ a1
extern "C" srl_status srl_gae(int T, int B, int ld, const float* rewards, const float* values,
                              const uint8_t* dones, const float* trunc_values,
                              const uint8_t* valid, float gamma, float lambda, float* adv_out,
                              float* ret_out, double* stats_out, srl_stream_t stream) {
  if (T < 1 || B < 1 || ld < B) FAIL(SRL_EINVAL, "srl_gae: need T >= 1, B >= 1, ld >= B");
  if (!rewards || !values || !dones || !adv_out) FAIL(SRL_EINVAL, "srl_gae: null pointer");
  if (srl_status st = require_device()) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* part = nullptr;
  const int nb = gae_num_blocks(B);
  if (stats_out) {
    // the per-call moment partials come from the device's stream-ordered pool; keep its memory
    // (release threshold = max) so steady-state calls neither map nor unmap pages
    static std::atomic<uint64_t> pool_set{0};
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64 &&
        !(pool_set.load(std::memory_order_relaxed) & (1ull << dev))) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      pool_set.fetch_or(1ull << dev, std::memory_order_relaxed);
    }
    CK(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * 3 * nb, s));
  }
  CK(launch_gae(T, B, ld, rewards, values, dones, trunc_values, valid, gamma, lambda, adv_out,
                ret_out, part, s));
  if (stats_out) {
    CK(launch_merge_moments(part, nb, stats_out, nullptr, 0, s));
    CK(cudaFreeAsync(part, s));
  }
  return SRL_OK;
}

// ------------------------------------------------------------------ context
struct Lay {
  int in, out;             // out = A+1 for the head
  int64_t w_off, b_off;    // flat offsets
  __half* w16;
  int w16_ld, w16_rows;
  int bn_fwd, cg_fwd;      // N tile / CTA-group of the GEMM producing this layer's output
  int bn_dx, cg_dx;        // same for the dX GEMM that produces dZ of this layer's INPUT
  int bn_dw, cg_dw, dw_n_tiles, dw_m_tiles, splits_max;
  float* part;             // dW partials [splits][out or in][ld_part]
  int64_t part_rows, ld_part;
  float* colsum;           // db partials of this layer: [sms][out] (hidden) / [sms][64] (head)
  int colsum_ld;
  int t = 0, l = 0;        // trunk (0 actor / shared, 1 critic) and layer index
  float* dz_colsum = nullptr;   // head only: column sums of dZ_L [sms][T*h_L] (db of layer L)
};

struct srl_ctx {
  int device = 0, rank = 0, world = 1, sms = 148;
  srl_ppo_config cfg{};
  std::vector<int> hidden, heads, dims;
  int L = 0, A = 0;
  // NEXT-3 separate trunks (DESIGN.md §3.5 R-AC): T = 2 trunks side by side in every activation
  // buffer (trunk t owns columns [t*h, (t+1)*h)); lay[t*L + l] = hidden layer l of trunk t,
  // lay[T*L] = the head over both trunks' last layer (block-structured fp16 weights)
  int T = 1;
  int64_t pi_w = 0, pi_b = 0, v_w = 0, v_b = 0;   // R-AC flat offsets of the two heads
  float* hbias = nullptr;                          // R-AC: contiguous fp32 head bias mirror [64]
  Lay& hid(int t, int l) { return lay[t * L + l]; }
  Lay& head() { return lay[T * L]; }
  int hidx(int t, int l) const { return t * L + l; }
  int64_t P = 0, max_n = 0;
  uint64_t digest = 0;
  std::vector<Lay> lay;
  float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr;
  int64_t* t_dev = nullptr;
  std::vector<__half*> Y;
  __half* G16 = nullptr;
  __half* dZ[2] = {nullptr, nullptr};
  double* stats_part = nullptr;
  unsigned long long* counters = nullptr;
  double* norm_scratch = nullptr;   // [world*3] gathered + [3] merged
  ncclComm_t comm = nullptr;
  std::vector<void*> allocs;
  // profiling (srl_prof_*): an event pair around every kernel srl_ppo_step launches
  struct ProfRec { const char* name; cudaEvent_t a, b; double flops, bytes; };
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  // tensor-map cache: encoding is host work; the maps depend only on pointer + shape
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t>, CUtensorMap> tmaps;
  // train-step buffers (srl_ppo_train_step): adv, ret [max_n] f32; gae partials; mean/std
  float *adv = nullptr, *ret = nullptr;
  // NEXT-1 pre-fetch slots (srl_batch_upload / srl_ppo_train_step_slot)
  struct Slot {
    float *rewards = nullptr, *values = nullptr, *logp_old = nullptr;
    uint8_t* dones = nullptr;
    __half* obs = nullptr;
    int32_t* actions = nullptr;
    float* trunc_values = nullptr;   // NEXT-3, allocated on first use
    uint8_t* valid = nullptr;
    bool has_tv = false, has_valid = false;
    int T = 0, B = 0;
    bool ready = false;
    cudaEvent_t uploaded = nullptr, released = nullptr;
  } slot[2];
  cudaStream_t copy_stream = nullptr;
  // a6 overlap (world > 1): bucket allreduce of the upper layers runs on comm_stream while the
  // rest of the backward computes
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_early = nullptr, ev_late = nullptr, ev_comm = nullptr;
  // a2's peer exchange on comm_stream during a3 (srl_ppo_train_step): the loss waits on ev_ms
  cudaEvent_t ev_gae = nullptr, ev_ms = nullptr;
  bool ms_pending = false;
  double *gae_part = nullptr, *gae_stats = nullptr, *mean_std = nullptr;
  unsigned int* gae_counter = nullptr;
  int gae_part_cap = 0;
  // NEXT-3 global-norm clipping: [kGradNormBlocks] partials, norm, coef (float in a double slot)
  double* gn = nullptr;
  unsigned int* gn_counter = nullptr;
  double* gn_norm() const { return gn + kGradNormBlocks; }
  // a6 over NVLink peer memory (world > 1): exposed double-buffered bucket + flags, peers' maps
  bool p2p = false;
  float* xbuf = nullptr;                       // [2][P + 8]
  unsigned long long* xflags = nullptr;        // [kMaxPeers]
  P2PPeers peers{};
  std::vector<void*> ipc_opened;
  unsigned long long epoch = 0, mepoch = 0;
  int64_t xstride() const { return (P + 8 + 63) / 64 * 64; }   // 256-B aligned halves
  float* gn_coef() const { return reinterpret_cast<float*>(gn + kGradNormBlocks + 1); }
  // bounded exchange waits (SPEC.md S:L532 ReduceTimeout): device + host-mapped error words
  CommCtl cc{};
  int* err_pinned = nullptr;                   // host view of cc.err_host
  bool failed = false;                         // a peer wait timed out or NCCL failed: no more steps
  unsigned* gbar = nullptr;                    // grid-barrier words of update_kernel
};

static unsigned long long comm_timeout_ns() {
  const char* e = getenv("SRL_COMM_TIMEOUT_S");
  double s = e ? atof(e) : 30.0;
  if (!(s > 0.0)) s = 30.0;
  return (unsigned long long)(s * 1e9);
}

// every call on a multi-rank context first looks at the exchange error words (no device sync:
// the host-mapped word is read directly) and at NCCL's asynchronous error state
static srl_status comm_check(srl_ctx* c, const char* who) {
  if (c->world == 1) return SRL_OK;
  if (!c->failed && c->err_pinned && *reinterpret_cast<volatile int*>(c->err_pinned)) c->failed = true;
  if (!c->failed && c->comm) {
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      c->failed = true;
    }
  }
  if (c->failed)
    FAIL(SRL_ENCCL, std::string(who) + ": the context's cross-rank exchange failed (a peer wait "
                    "exceeded SRL_COMM_TIMEOUT_S or NCCL reported an error); destroy the context");
  return SRL_OK;
}

static bool get_tmap(srl_ctx* c, CUtensorMap* out, const void* base, uint64_t inner,
                     uint64_t outer, uint64_t row_bytes, uint32_t bi, uint32_t bo,
                     int swizzle = 128) {
  auto key = std::make_tuple(base, inner, outer, row_bytes, bi, bo * 1000 + swizzle);
  auto it = c->tmaps.find(key);
  if (it != c->tmaps.end()) { *out = it->second; return true; }
  if (!make_tmap_2d(out, base, inner, outer, row_bytes, bi, bo, swizzle)) return false;
  if (c->tmaps.size() > 4096) c->tmaps.clear();
  c->tmaps.emplace(key, *out);
  return true;
}

static cudaEvent_t prof_event(srl_ctx* c) {
  if (c->pool_used == c->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->pool.push_back(e);
  }
  return c->pool[c->pool_used++];
}

struct ProfScope {
  srl_ctx* c; cudaStream_t s; const char* name; double flops, bytes; cudaEvent_t a = nullptr;
  ProfScope(srl_ctx* c_, cudaStream_t s_, const char* n, double f, double b)
      : c(c_), s(s_), name(n), flops(f), bytes(b) {
    if (c->prof) { a = prof_event(c); cudaEventRecord(a, s); }
  }
  ~ProfScope() {
    if (c->prof) {
      cudaEvent_t b2 = prof_event(c);
      cudaEventRecord(b2, s);
      c->recs.push_back({name, a, b2, flops, bytes});
    }
  }
};

// SRL_HEAD_FUSED=0: the head block as three kernels (head GEMM + loss, dX, split-K dW)
static bool head_fused_enabled() {
  const char* e = getenv("SRL_HEAD_FUSED");
  return !(e && e[0] == '0');
}

// opt-in (SRL_DW_FIXUP=1): the split-K sum inside each dW launch (gemm_tc.cuh part_fixup).
// Measured slower on the Atari step (0.480 vs 0.473 ms): the grid barrier holds every CTA
// until the slowest split is done, so the next launch no longer overlaps the dW tail (PDL),
// which costs more than the ~8 us the update launch saves.
static bool dw_fixup_enabled() {
  const char* e = getenv("SRL_DW_FIXUP");
  return e && e[0] == '1';
}

// SRL_XFUSED=0: the peer-path exchange as its own launch between two update launches
static bool xfused_enabled() {
  const char* e = getenv("SRL_XFUSED");
  return !(e && e[0] == '0');
}

static bool dw_discard_enabled() {
  const char* e = getenv("SRL_DW_DISCARD");
  return !(e && e[0] == '0');
}

static bool dw512_enabled() {   // opt-in: measured ~5% slower dW + finalize on the Atari shape
  const char* e = getenv("SRL_DW512");
  return e && e[0] == '1';
}

static int pick_bn(int n) {
  if (n % 256 == 0) return 256;
  if (n <= 64) return 64;
  if (n % 128 == 0 || n <= 128) return 128;
  return 128;
}

static uint64_t fnv1a(const std::vector<int>& xs) {
  uint64_t h = 1469598103934665603ull;
  for (int x : xs) {
    int32_t v = x;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(&v);
    for (int i = 0; i < 4; ++i) { h ^= b[i]; h *= 1099511628211ull; }
  }
  return h;
}

template <class T>
static srl_status dalloc(srl_ctx* c, T** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) FAIL(SRL_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  cudaMemset(q, 0, bytes ? bytes : 16);
  c->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return SRL_OK;
}

static void free_ctx(srl_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto& sl : c->slot) {
    if (sl.uploaded) cudaEventDestroy(sl.uploaded);
    if (sl.released) cudaEventDestroy(sl.released);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  for (cudaEvent_t e : {c->ev_early, c->ev_late, c->ev_comm, c->ev_gae, c->ev_ms})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->err_pinned) cudaFreeHost(c->err_pinned);
  if (c->comm) {
    if (c->failed) ncclCommAbort(c->comm);   // a failed exchange: do not wait on any peer
    else ncclCommDestroy(c->comm);
  }
  for (void* p : c->allocs) cudaFree(p);
  delete c;
}

extern "C" srl_status srl_nccl_unique_id(uint8_t out[128]) {
  if (!out) FAIL(SRL_EINVAL, "srl_nccl_unique_id: null");
  ncclUniqueId id;
  CKN(ncclGetUniqueId(&id));
  std::memcpy(out, id.internal, 128);
  return SRL_OK;
}

// the flat parameter vector as segments with their gradient sources (split-K / per-CTA
// partials and column sums, indexed like c->lay) and fp16 shadows
static SegTable make_segs(srl_ctx* c, const std::vector<int>& splits,
                          const std::vector<int>& colsum_parts, int dz_parts,
                          const std::vector<int>& reduced = {}) {
  SegTable t{};
  t.n = 0;
  const int L = c->L, T = c->T;
  const Lay& hd = c->head();
  const int hL = c->dims[L];
  const int hi = T * L;                                   // head index in c->lay
  auto nsp = [&](int i) { return splits.empty() ? 0 : splits[i]; };
  auto ncs = [&](int i) { return colsum_parts.empty() ? 0 : colsum_parts[i]; };
  for (int tr = 0; tr < T; ++tr)
    for (int l = 0; l < L; ++l) {
      const Lay& y = c->hid(tr, l);
      const int i = c->hidx(tr, l);
      Segment w{};
      w.off = y.w_off; w.rows = y.out; w.cols = y.in; w.is_bias = 0;
      w.part = y.part; w.splits = nsp(i); w.ld_part = y.ld_part;
      w.split_stride = y.part_rows * y.ld_part; w.transposed = 0; w.prow_cap = (int)y.ld_part;
      w.w16 = y.w16; w.w16_ld = y.w16_ld;
      w.done = reduced.empty() ? 0 : reduced[i];
      t.s[t.n++] = w;
      Segment b{};
      b.off = y.b_off; b.rows = 1; b.cols = y.out; b.is_bias = 1;
      if (l + 1 < L) {           // db_l from the dX epilogue of layer l+1 of this trunk
        b.colsum = y.colsum; b.nparts = ncs(i); b.colsum_ld = y.colsum_ld;
      } else {                   // db_L from the head's dX (this trunk's columns of dZ_L)
        b.colsum = hd.dz_colsum + tr * hL; b.nparts = dz_parts; b.colsum_ld = T * hL;
      }
      t.s[t.n++] = b;
    }
  // head: the dW^T partial [T*hL][64] (transposed) and the per-CTA column sums of g [64]
  auto head_w = [&](int64_t off, int rows, int row0, int col0) {
    Segment w{};
    w.off = off; w.rows = rows; w.cols = hL; w.is_bias = 0;
    w.part = hd.part + (int64_t)row0 * hd.ld_part + col0; w.splits = nsp(hi);
    w.ld_part = hd.ld_part; w.split_stride = hd.part_rows * hd.ld_part; w.transposed = 1;
    w.prow_cap = (int)hd.ld_part - col0;
    w.w16 = hd.w16 + (int64_t)col0 * hd.w16_ld + row0; w.w16_ld = hd.w16_ld;
    t.s[t.n++] = w;
  };
  auto head_b = [&](int64_t off, int cols, int col0) {
    Segment b{};
    b.off = off; b.rows = 1; b.cols = cols; b.is_bias = 1;
    b.colsum = hd.colsum + col0; b.nparts = ncs(hi); b.colsum_ld = hd.colsum_ld;
    b.b32 = T > 1 ? c->hbias + col0 : nullptr;
    t.s[t.n++] = b;
  };
  if (T == 1) {
    head_w(hd.w_off, hd.out, 0, 0);
    head_b(hd.b_off, hd.out, 0);
  } else {                       // policy head on the actor's columns, value on the critic's
    head_w(c->pi_w, c->A, 0, 0);
    head_b(c->pi_b, c->A, 0);
    head_w(c->v_w, 1, hL, c->A);
    head_b(c->v_b, 1, c->A);
  }
  return t;
}

extern "C" srl_status srl_ppo_create(const srl_ppo_config* cfg, int rank, int world,
                                     const uint8_t* nccl_id, int device, srl_ctx** out) {
  if (!cfg || !out) FAIL(SRL_EINVAL, "srl_ppo_create: null");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) FAIL(SRL_EINVAL, "srl_ppo_create: bad rank/world");
  if (world > 1 && !nccl_id) FAIL(SRL_EINVAL, "srl_ppo_create: world > 1 needs nccl_id");
  if (cfg->obs_dim < 1 || cfg->ld_obs < cfg->obs_dim || cfg->ld_obs % 8)
    FAIL(SRL_EINVAL, "srl_ppo_create: need 1 <= obs_dim <= ld_obs, ld_obs % 8 == 0");
  if (cfg->n_hidden < 1 || cfg->n_hidden > 8 || !cfg->hidden)
    FAIL(SRL_EINVAL, "srl_ppo_create: need 1 <= n_hidden <= 8");
  for (int l = 0; l < cfg->n_hidden; ++l)
    if (cfg->hidden[l] < 64 || cfg->hidden[l] % 64 || cfg->hidden[l] > 1024)
      FAIL(SRL_EINVAL, "srl_ppo_create: hidden widths must be multiples of 64 in [64, 1024]");
  if (cfg->n_heads < 1 || cfg->n_heads > kMaxHeads || !cfg->head_sizes)
    FAIL(SRL_EINVAL, "srl_ppo_create: need 1 <= n_heads <= 8");
  int A = 0;
  for (int h = 0; h < cfg->n_heads; ++h) {
    if (cfg->head_sizes[h] < 1) FAIL(SRL_EINVAL, "srl_ppo_create: head size < 1");
    A += cfg->head_sizes[h];
  }
  if (A + 1 > kHeadCols) FAIL(SRL_EINVAL, "srl_ppo_create: sum(head_sizes) + 1 must be <= 64");
  if (cfg->max_local_n < 1 || cfg->max_local_n > (int64_t)INT32_MAX)
    FAIL(SRL_EINVAL, "srl_ppo_create: need 1 <= max_local_n <= 2^31 - 1");
  if (cfg->precision != SRL_PREC_F16_SCALED) FAIL(SRL_EUNSUPPORTED, "srl_ppo_create: precision");
  if (!(cfg->value_clip >= 0.f) || !(cfg->max_grad_norm >= 0.f) || cfg->epochs > 1000 ||
      cfg->minibatches > 4096)
    FAIL(SRL_EINVAL, "srl_ppo_create: need value_clip >= 0, max_grad_norm >= 0, epochs <= 1000, "
                     "minibatches <= 4096");
  if (srl_status st = require_device()) return st;
  CK(cudaSetDevice(device));
  if (!tmap_init()) FAIL(SRL_ECUDA, "cuTensorMapEncodeTiled unavailable");

  srl_ctx* c = new srl_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->cfg = *cfg;
  if (c->cfg.epochs < 1) c->cfg.epochs = 1;
  if (c->cfg.minibatches < 1) c->cfg.minibatches = 1;
  c->hidden.assign(cfg->hidden, cfg->hidden + cfg->n_hidden);
  c->heads.assign(cfg->head_sizes, cfg->head_sizes + cfg->n_heads);
  c->cfg.hidden = c->hidden.data();
  c->cfg.head_sizes = c->heads.data();
  c->L = cfg->n_hidden;
  c->A = A;
  c->max_n = cfg->max_local_n;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  c->dims.push_back(cfg->obs_dim);
  for (int h : c->hidden) c->dims.push_back(h);
  c->dims.push_back(A + 1);
  std::vector<int> dig(c->dims);
  dig.insert(dig.end(), c->heads.begin(), c->heads.end());
  if (cfg->separate_critic) dig.push_back(-2);     // R-AC: a different flat layout
  c->digest = fnv1a(dig);

  auto bail = [&](srl_status st) { free_ctx(c); return st; };
  c->T = cfg->separate_critic ? 2 : 1;
  const int T = c->T, L = c->L, hL = c->dims[L];
  int64_t off = 0;
  int max_h = 0;
  c->lay.resize(T * L + 1);
  for (int tr = 0; tr < T; ++tr) {
    for (int l = 0; l < L; ++l) {
      Lay& y = c->hid(tr, l);
      y.t = tr; y.l = l;
      y.in = c->dims[l];
      y.out = c->dims[l + 1];
      y.w_off = off;
      y.b_off = off + (int64_t)y.out * y.in;
      off = y.b_off + y.out;
      y.w16_ld = (l == 0) ? (y.in + 7) / 8 * 8 : y.in;
      y.w16_rows = y.out;
      max_h = std::max(max_h, T * y.out);
    }
    if (T == 1) {
      Lay& y = c->head();
      y.w_off = off;
      y.b_off = off + (int64_t)(A + 1) * hL;
      off = y.b_off + A + 1;
    } else if (tr == 0) {        // R-AC: W_pi [A][h_L], b_pi [A] after the actor trunk
      c->pi_w = off; c->pi_b = off + (int64_t)A * hL; off = c->pi_b + A;
    } else {                     // w_v [1][h_L], b_v [1] after the critic trunk
      c->v_w = off; c->v_b = off + hL; off = c->v_b + 1;
    }
  }
  {
    Lay& y = c->head();
    y.t = 0; y.l = L;
    y.in = T * hL;               // the head reads both trunks' last layer
    y.out = A + 1;
    y.w16_ld = y.in;
    y.w16_rows = kHeadCols;
  }
  c->P = off;
  srl_status st;
  if ((st = dalloc(c, &c->params, sizeof(float) * c->P))) return bail(st);
  if ((st = dalloc(c, &c->grads, sizeof(float) * (c->P + 8)))) return bail(st);
  if ((st = dalloc(c, &c->m, sizeof(float) * c->P))) return bail(st);
  if ((st = dalloc(c, &c->v, sizeof(float) * c->P))) return bail(st);
  if ((st = dalloc(c, &c->t_dev, sizeof(int64_t)))) return bail(st);
  if ((st = dalloc(c, &c->counters, sizeof(unsigned long long) * 4))) return bail(st);
  if ((st = dalloc(c, &c->stats_part, sizeof(double) * 8 * c->sms))) return bail(st);
  if ((st = dalloc(c, &c->norm_scratch, sizeof(double) * (3 * kMomentBlocks + 3 * world + 8)))) return bail(st);
  if ((st = dalloc(c, &c->hbias, sizeof(float) * kHeadCols))) return bail(st);
  const int64_t n = c->max_n;
  for (size_t li = 0; li < c->lay.size(); ++li) {
    Lay& y = c->lay[li];
    const bool is_head = li + 1 == c->lay.size();
    if ((st = dalloc(c, &y.w16, sizeof(__half) * (size_t)y.w16_rows * y.w16_ld))) return bail(st);
    // epilogue-heavy GEMMs (fwd tanh, dX dtanh) use 128-wide tiles: 4 TMEM accumulators
    // 256-wide outputs run on CTA pairs (tcgen05 cta_group::2, 256 x 256 tiles): half the
    // shared-memory operand traffic per FLOP of a 1-SM 128 x 128 tile
    if (is_head) { y.bn_fwd = kHeadCols; y.cg_fwd = 1; }
    else if (y.out % 256 == 0) { y.bn_fwd = 256; y.cg_fwd = 2; }
    else { y.bn_fwd = (y.out % 128 == 0) ? 128 : 64; y.cg_fwd = 1; }
    if (y.in % 256 == 0) { y.bn_dx = 256; y.cg_dx = 2; }
    else { y.bn_dx = (y.in % 128 == 0) ? 128 : 64; y.cg_dx = 1; }
    // dW: hidden layer: D[out][in] = dZ^T X; head: D^T[in][64] = Y^T g
    const int dM = is_head ? y.in : y.out;
    const int dN = is_head ? kHeadCols : y.in;
    y.bn_dw = is_head ? kHeadCols : pick_bn(dN);
    // 512-wide dW tiles (two N = 256 MMAs sharing the dZ tile): the layer's dZ is read once
    // per split instead of once per 256 columns (SRL_DW512=1 enables)
    if (!is_head && dN % 512 == 0 && dM >= 256 && dw512_enabled()) y.bn_dw = 512;
    y.cg_dw = (!is_head && dM >= 256 && y.bn_dw >= 128) ? 2 : 1;
    y.dw_m_tiles = (dM + 128 * y.cg_dw - 1) / (128 * y.cg_dw);
    y.dw_n_tiles = (dN + y.bn_dw - 1) / y.bn_dw;
    y.splits_max = std::max(1, (c->sms / y.cg_dw) / (y.dw_m_tiles * y.dw_n_tiles));
    y.part_rows = dM;
    y.ld_part = (int64_t)y.dw_n_tiles * y.bn_dw;
    // the fused head kernel writes one dW_h^T partial per CTA (up to one per SM)
    const int part_splits = is_head ? std::max(y.splits_max, c->sms) : y.splits_max;
    if ((st = dalloc(c, &y.part, sizeof(float) * part_splits * y.part_rows * y.ld_part))) return bail(st);
    y.colsum_ld = is_head ? kHeadCols : y.out;
    if ((st = dalloc(c, &y.colsum, sizeof(float) * c->sms * y.colsum_ld))) return bail(st);
    if (is_head && (st = dalloc(c, &y.dz_colsum, sizeof(float) * c->sms * y.in))) return bail(st);
  }
  c->Y.resize(c->L);
  for (int l = 0; l < c->L; ++l)
    if ((st = dalloc(c, &c->Y[l], sizeof(__half) * (size_t)n * T * c->dims[l + 1]))) return bail(st);
  if ((st = dalloc(c, &c->G16, sizeof(__half) * (size_t)n * kHeadCols))) return bail(st);
  for (int k = 0; k < 2; ++k)
    if ((st = dalloc(c, &c->dZ[k], sizeof(__half) * (size_t)n * max_h))) return bail(st);
  if (world > 1) {
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_early, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_late, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_gae, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_ms, cudaEventDisableTiming) != cudaSuccess) {
      set_error("srl_ppo_create: stream/event creation failed");
      free_ctx(c);
      return SRL_ECUDA;
    }
  }
  if ((st = dalloc(c, &c->adv, sizeof(float) * n))) return bail(st);
  if ((st = dalloc(c, &c->ret, sizeof(float) * n))) return bail(st);
  c->gae_part_cap = (int)((n + 7) / 8) + 1;   // >= gae_num_blocks(B) for any B <= n
  if ((st = dalloc(c, &c->gae_part, sizeof(double) * 3 * c->gae_part_cap))) return bail(st);
  if ((st = dalloc(c, &c->gae_stats, sizeof(double) * 4))) return bail(st);
  if ((st = dalloc(c, &c->mean_std, sizeof(double) * 2))) return bail(st);
  if ((st = dalloc(c, &c->gae_counter, sizeof(unsigned int) * 4))) return bail(st);
  if ((st = dalloc(c, &c->gn, sizeof(double) * (kGradNormBlocks + 2)))) return bail(st);
  if ((st = dalloc(c, &c->gn_counter, sizeof(unsigned int) * 4))) return bail(st);
  if ((st = dalloc(c, &c->cc.err_dev, sizeof(int) * 4))) return bail(st);
  if ((st = dalloc(c, &c->gbar, sizeof(unsigned) * 8))) return bail(st);   // [0..3] update, [4..5] dW
  if (cudaHostAlloc(reinterpret_cast<void**>(&c->err_pinned), sizeof(int) * 4, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->cc.err_host), c->err_pinned, 0) != cudaSuccess) {
    c->err_pinned = nullptr;
    set_error("srl_ppo_create: mapped host allocation failed");
    free_ctx(c);
    return SRL_ENOMEM;
  }
  std::memset(c->err_pinned, 0, sizeof(int) * 4);
  c->cc.timeout_ns = comm_timeout_ns();
  if (world > 1) {
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
      set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      c->comm = nullptr;
      free_ctx(c);
      return SRL_ENCCL;
    }
  }
  if (world > 1 && world <= kMaxPeers && p2p_ar_enabled()) {
    // exchange CUDA IPC handles of the exposed bucket and flags (one NCCL all-gather)
    if ((st = dalloc(c, &c->xbuf, sizeof(float) * 2 * c->xstride()))) return bail(st);
    if ((st = dalloc(c, &c->xflags, kSyncBytes))) return bail(st);
    cudaIpcMemHandle_t h[2];
    bool ok = cudaIpcGetMemHandle(&h[0], c->xbuf) == cudaSuccess &&
              cudaIpcGetMemHandle(&h[1], c->xflags) == cudaSuccess;
    uint8_t* dh = nullptr;
    std::vector<uint8_t> all((size_t)world * sizeof(h));
    if (ok) ok = cudaMalloc(&dh, all.size() + sizeof(h)) == cudaSuccess;
    if (ok) ok = cudaMemcpy(dh + all.size(), h, sizeof(h), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) ok = ncclAllGather(dh + all.size(), dh, sizeof(h), ncclUint8, c->comm, 0) == ncclSuccess;
    if (ok) ok = cudaMemcpy(all.data(), dh, all.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (dh) cudaFree(dh);
    for (int r = 0; ok && r < world; ++r) {
      if (r == rank) { c->peers.x[r] = c->xbuf; c->peers.flag[r] = c->xflags; continue; }
      cudaIpcMemHandle_t ph[2];
      std::memcpy(ph, all.data() + (size_t)r * sizeof(h), sizeof(h));
      void *px = nullptr, *pf = nullptr;
      ok = cudaIpcOpenMemHandle(&px, ph[0], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (ok) c->ipc_opened.push_back(px);
      if (ok) ok = cudaIpcOpenMemHandle(&pf, ph[1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (ok) c->ipc_opened.push_back(pf);
      c->peers.x[r] = static_cast<float*>(px);
      c->peers.flag[r] = static_cast<unsigned long long*>(pf);
    }
    // every rank must agree: the peer path is used only if it could be set up everywhere
    int mine = ok ? 1 : 0, *dflag = nullptr, every = 0;
    if (cudaMalloc(&dflag, sizeof(int)) == cudaSuccess) {
      cudaMemcpy(dflag, &mine, sizeof(int), cudaMemcpyHostToDevice);
      if (ncclAllReduce(dflag, dflag, 1, ncclInt32, ncclMin, c->comm, 0) == ncclSuccess)
        cudaMemcpy(&every, dflag, sizeof(int), cudaMemcpyDeviceToHost);
      cudaFree(dflag);
    }
    cudaGetLastError();
    c->p2p = every == 1;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    set_error(std::string("srl_ppo_create: ") + cudaGetErrorString(e));
    free_ctx(c);
    return SRL_ECUDA;
  }
  *out = c;
  return SRL_OK;
}

extern "C" int srl_ppo_comm_path(srl_ctx* c) {
  if (!c) return -1;
  if (c->world == 1) return 0;
  return (c->p2p && !ar_overlap()) ? 2 : 1;
}

extern "C" srl_status srl_ppo_destroy(srl_ctx* ctx) {
  free_ctx(ctx);
  return SRL_OK;
}

extern "C" srl_status srl_ppo_params(srl_ctx* c, float** params_dev, float** grads_dev,
                                     int64_t* P, uint64_t* digest) {
  if (!c) FAIL(SRL_EINVAL, "srl_ppo_params: null ctx");
  if (params_dev) *params_dev = c->params;
  if (grads_dev) *grads_dev = c->grads;
  if (P) *P = c->P;
  if (digest) *digest = c->digest;
  return SRL_OK;
}

extern "C" srl_status srl_ppo_adam_state(srl_ctx* c, float** m_dev, float** v_dev,
                                         int64_t* step) {
  if (!c) FAIL(SRL_EINVAL, "srl_ppo_adam_state: null ctx");
  CK(cudaSetDevice(c->device));
  if (m_dev) *m_dev = c->m;
  if (v_dev) *v_dev = c->v;
  if (step) CK(cudaMemcpy(step, c->t_dev, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return SRL_OK;
}

extern "C" srl_status srl_ppo_load_params(srl_ctx* c, const float* params_dev,
                                          srl_stream_t stream) {
  if (!c || !params_dev) FAIL(SRL_EINVAL, "srl_ppo_load_params: null");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaMemcpyAsync(c->params, params_dev, sizeof(float) * c->P, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(c->m, 0, sizeof(float) * c->P, s));
  CK(cudaMemsetAsync(c->v, 0, sizeof(float) * c->P, s));
  CK(cudaMemsetAsync(c->t_dev, 0, sizeof(int64_t), s));
  SegTable t = make_segs(c, {}, {}, 0);
  CK(launch_shadow(t, c->params, s));
  return SRL_OK;
}

// ------------------------------------------------------------------ a2
extern "C" srl_status srl_adv_norm(srl_ctx* ctx, float* adv, int64_t n, const double* local_stats,
                                   float eps, int unbiased, int apply, double* mean_std_out,
                                   srl_stream_t stream) {
  if (n < 1) FAIL(SRL_EINVAL, "srl_adv_norm: n < 1");
  if (!adv && (!local_stats || apply)) FAIL(SRL_EINVAL, "srl_adv_norm: null adv");
  if (srl_status st = require_device()) return st;
  if (ctx) {
    CK(cudaSetDevice(ctx->device));
    if (srl_status st = comm_check(ctx, "srl_adv_norm")) return st;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* scratch = nullptr;   // [kMomentBlocks*3] partials, [3] local, [world*3] gathered, [2] ms
  const int world = ctx ? ctx->world : 1;
  const size_t cnt = 3 * kMomentBlocks + 3 + 3 * world + 2;
  if (ctx) scratch = ctx->norm_scratch;   // context-owned: no allocation on the hot path
  else CK(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(double) * cnt, s));
  double* local = scratch + 3 * kMomentBlocks;
  double* gathered = local + 3;
  double* ms = gathered + 3 * world;
  if (!local_stats) {
    CK(launch_moments(adv, n, scratch, s));
    CK(launch_merge_moments(scratch, kMomentBlocks, local, nullptr, 0, s));
    local_stats = local;
  }
  if (world > 1 && ctx->p2p) {
    // the same NVLink peer-memory exchange srl_ppo_train_step uses (rank-order merge)
    CK(launch_p2p_moments(ctx->peers, world, ctx->rank, ++ctx->mepoch, local_stats, ms, unbiased,
                          ctx->cc, 3, s));
  } else if (world > 1) {
    CKN(ncclAllGather(local_stats, gathered, 3, ncclDouble, ctx->comm, s));
    CK(launch_merge_moments(gathered, world, nullptr, ms, unbiased, s));
  } else {
    CK(launch_merge_moments(local_stats, 1, nullptr, ms, unbiased, s));
  }
  if (apply) CK(launch_normalize(adv, n, ms, eps, s));
  if (mean_std_out)
    CK(cudaMemcpyAsync(mean_std_out, ms, sizeof(double) * 2, cudaMemcpyDeviceToDevice, s));
  if (!ctx) CK(cudaFreeAsync(scratch, s));
  return SRL_OK;
}

// ------------------------------------------------------------------ a6
static __global__ void scale_kernel(float* x, int64_t n, float a) {
  griddep_wait();
  griddep_launch();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= a;
}

extern "C" srl_status srl_allreduce_grads(srl_ctx* c, float* buf, int64_t count, int op,
                                          srl_stream_t stream) {
  if (!c || !buf || count < 0 || (op != 0 && op != 1)) FAIL(SRL_EINVAL, "srl_allreduce_grads: bad args");
  if (c->world == 1 || count == 0) return SRL_OK;
  CK(cudaSetDevice(c->device));
  if (srl_status st = comm_check(c, "srl_allreduce_grads")) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float scale = op == 1 ? 1.f / (float)c->world : 1.f;
  if (c->p2p && count <= c->xstride()) {
    // the step's two-shot peer-memory exchange: stage into this rank's exposed buffer of the
    // next epoch's parity, reduce in rank order, result back into buf (identical on all ranks)
    const unsigned long long epoch = c->epoch + 1;
    const int64_t xoff = (int64_t)(epoch & 1ull) * c->xstride();
    CK(cudaMemcpyAsync(c->xbuf + xoff, buf, sizeof(float) * count, cudaMemcpyDeviceToDevice, s));
    c->epoch = epoch;
    CK(launch_p2p_allreduce(c->peers, c->world, c->rank, xoff, count, epoch, scale, buf, c->cc, 3, s));
    return SRL_OK;
  }
  CKN(ncclAllReduce(buf, buf, (size_t)count, ncclFloat, ncclSum, c->comm, s));
  if (op == 1) {
    int64_t blocks = std::min<int64_t>((count + 255) / 256, 4 * c->sms);
    CK(launch_k(scale_kernel, dim3((unsigned)blocks), dim3(256), 0, s, 1, buf, count, scale));
  }
  return SRL_OK;
}

// ------------------------------------------------------------------ a3..a7
static srl_status gemm(int bn, bool a_mn, bool b_mn, int epi, int cg, const CUtensorMap& ta,
                       const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& ty,
                       GemmArgs& g, int sms, cudaStream_t s, int* grid_out = nullptr) {
  const int units = g.m_tiles * g.n_tiles * g.k_splits;   // m_tiles of 128 * cg rows
  const int grid = cg * std::min(units, sms / cg);
  if (grid_out) *grid_out = grid;
  cudaError_t e = launch_gemm(bn, a_mn, b_mn, epi, cg, ta, tb, to, ty, g, grid, s);
  if (e != cudaSuccess) FAIL(SRL_ECUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  return SRL_OK;
}

#define TM(map, ...)                                                             \
  do {                                                                           \
    if (!make_tmap_2d(&(map), __VA_ARGS__)) FAIL(SRL_ECUDA, "tensor map encode failed"); \
  } while (0)
#define TMC(map, ...)                                                            \
  do {                                                                           \
    if (!get_tmap(c, &(map), __VA_ARGS__)) FAIL(SRL_ECUDA, "tensor map encode failed"); \
  } while (0)

// a3: the hidden layers of the forward pass, Y_l = tanh(Y_{l-1} W_l^T + b_l), into c->Y
// a3: the hidden layers of the forward pass, Y_l = tanh(Y_{l-1} W_l^T + b_l), into c->Y; with
// separate trunks each layer runs once per trunk on that trunk's column half (both read obs)
static srl_status forward_hidden(srl_ctx* c, int n, const __half* X0, cudaStream_t s) {
  const int L = c->L, T = c->T;
  const int sms = c->sms;
  const int ld_obs = c->cfg.ld_obs;
  for (int l = 0; l < L; ++l)
    for (int tr = 0; tr < T; ++tr) {
      const Lay& y = c->hid(tr, l);
      CUtensorMap ta, tb;
      const __half* X = l == 0 ? X0 : c->Y[l - 1] + (size_t)tr * y.in;
      const int ldx = l == 0 ? ld_obs : T * y.in;
      TMC(ta, X, y.in, n, (uint64_t)ldx * 2, 64, 128);
      TMC(tb, y.w16, y.in, y.out, (uint64_t)y.w16_ld * 2, 64, y.bn_fwd / y.cg_fwd);
      CUtensorMap to;
      TMC(to, c->Y[l] + (size_t)tr * y.out, y.out, n, (uint64_t)T * y.out * 2, 32, 32, 64);
      GemmArgs g{};
      g.M = n; g.N = y.out;
      g.m_tiles = (n + 128 * y.cg_fwd - 1) / (128 * y.cg_fwd); g.n_tiles = y.out / y.bn_fwd; g.k_splits = 1;
      g.kb_total = (y.in + 63) / 64; g.kb_per_split = g.kb_total;
      g.bias = c->params + y.b_off;
      ProfScope ps(c, s, l == 0 ? "fwd_l1" : "fwd_hidden", 2.0 * n * y.in * y.out,
                   2.0 * n * (y.in + y.out) + 2.0 * y.in * y.out + 4.0 * y.out);
      if (srl_status st = gemm(y.bn_fwd, false, false, tanh_accurate() ? EPI_TANH_ACC : EPI_TANH, y.cg_fwd,
                               ta, tb, to, to, g, sms, s)) return st;
    }
  return SRL_OK;
}

extern "C" srl_status srl_ppo_step(srl_ctx* c, int64_t n_local, int64_t n_global,
                                   const uint16_t* obs, const int32_t* actions,
                                   const float* logp_old, const float* adv, const float* ret,
                                   const float* v_old, const uint8_t* valid,
                                   const double* adv_mean_std, int apply,
                                   srl_ppo_stats* stats_out, srl_stream_t stream) {
  if (!c) FAIL(SRL_EINVAL, "srl_ppo_step: null ctx");
  if (srl_status st = comm_check(c, "srl_ppo_step")) return st;
  if (n_local < 1 || n_local > c->max_n || n_global < (valid ? 1 : n_local))
    FAIL(SRL_EINVAL, "srl_ppo_step: need 1 <= n_local <= max_local_n, n_global >= n_local "
                     "(>= 1 with a valid mask)");
  if (!obs || !actions || !logp_old || !adv || !ret) FAIL(SRL_EINVAL, "srl_ppo_step: null input");
  const bool vclip = c->cfg.value_clip > 0.f;
  if (vclip && !v_old) FAIL(SRL_EINVAL, "srl_ppo_step: value_clip > 0 needs v_old");
  if ((reinterpret_cast<uintptr_t>(obs) & 15) != 0) FAIL(SRL_EINVAL, "srl_ppo_step: obs must be 16-byte aligned");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int n = (int)n_local;
  const int L = c->L;
  const int sms = c->sms;
  const float inv_n = (float)(1.0 / (double)n_global);
  const __half* X0 = reinterpret_cast<const __half*>(obs);
  const int ld_obs = c->cfg.ld_obs;
  // c->counters are zero here: zeroed at create, re-zeroed by the stats kernel of every step

  // ---------------- a3: forward hidden layers Y_l = tanh(Y_{l-1} W_l^T + b_l)
  if (srl_status st = forward_hidden(c, n, X0, s)) return st;
  // ---------------- a4: head GEMM + fused PPO loss -> per-sample dlogits G16
  const int T = c->T;
  const int HI = T * L;                                 // the head's index in c->lay
  const Lay& hd = c->head();
  int grid_loss = 0, dz_parts = 0;
  const int hL = hd.in;                                 // T * h_L: both trunks' last layer
  const float* hbias = T == 1 ? c->params + hd.b_off : c->hbias;
  const int zcols = c->A + 1 + (int)c->heads.size();
  const bool fused = head_fused_enabled() && hL % 128 == 0 && hL <= 512 && c->A + 1 <= 32 &&
                     head_fused_smem(hL, zcols, (int)c->heads.size()) + 512 <= kSmemLimit;
  std::vector<int> splits(HI + 1, 1), colsum_parts(HI + 1, 0), reduced(HI + 1, 0);
  int cur = 0;
  auto loss_args = [&](GemmArgs& g) {
    g.bias = hbias;
    g.colsum = hd.colsum; g.colsum_ld = kHeadCols;
    g.counters = c->counters;
    g.actions = actions; g.logp_old = logp_old; g.adv = adv; g.ret = ret;
    g.mean_std = adv_mean_std; g.stats = c->stats_part;
    g.n_heads = (int)c->heads.size(); g.A = c->A;
    for (int h = 0; h < g.n_heads; ++h) g.head_size[h] = c->heads[h];
    g.clip_eps = c->cfg.clip_eps; g.value_coef = c->cfg.value_coef;
    g.entropy_coef = c->cfg.entropy_coef; g.adv_eps = c->cfg.adv_eps;
    g.v_old = vclip ? v_old : nullptr; g.value_clip = c->cfg.value_clip;
    g.valid = valid;
  };
  if (c->ms_pending) {                                  // mean/std from the a2 exchange
    CK(cudaStreamWaitEvent(s, c->ev_ms, 0));
    c->ms_pending = false;
  }
  if (fused) {
    // a4 + the head's a5 in one kernel: loss, dZ_L, db_L / db_h column sums, dW_h^T partials
    CUtensorMap ty, tw, to;
    TMC(ty, c->Y[L - 1], hL, n, (uint64_t)hL * 2, 64, 128);
    TMC(tw, hd.w16, hL, kHeadCols, (uint64_t)hd.w16_ld * 2, 64, 32);   // the 32 real head rows
    TMC(to, c->dZ[cur], hL, n, (uint64_t)hL * 2, 32, 32, 64);
    GemmArgs g{};
    g.M = n; g.N = kHeadCols;
    g.m_tiles = (n + 127) / 128; g.n_tiles = 1; g.k_splits = 1;
    loss_args(g);
    g.part = hd.part; g.ld_part = hd.ld_part; g.part_split_stride = hd.part_rows * hd.ld_part;
    const int grid = std::min(g.m_tiles, sms);
    const double Ap1 = (double)hd.out;
    ProfScope ps(c, s, "head_fused", 6.0 * n * hL * Ap1,
                 4.0 * n * hL + (16.0 + 4.0 * g.n_heads) * n + 2.0 * kHeadCols * hL);
    cudaError_t e = launch_head_fused(ty, tw, to, g, hL, hd.dz_colsum, grid, s);
    if (e != cudaSuccess) FAIL(SRL_ECUDA, std::string("head_fused launch: ") + cudaGetErrorString(e));
    grid_loss = grid;
    splits[HI] = grid;
    colsum_parts[HI] = grid;
    dz_parts = grid;
  } else {
    CUtensorMap ta, tb;
    TMC(ta, c->Y[L - 1], hd.in, n, (uint64_t)hd.in * 2, 64, 128);
    TMC(tb, hd.w16, hd.in, kHeadCols, (uint64_t)hd.w16_ld * 2, 64, 64);
    CUtensorMap to;
    TMC(to, c->G16, kHeadCols, n, (uint64_t)kHeadCols * 2, 32, 32, 64);
    GemmArgs g{};
    g.M = n; g.N = kHeadCols;
    g.m_tiles = (n + 127) / 128; g.n_tiles = 1; g.k_splits = 1;
    g.kb_total = (hd.in + 63) / 64; g.kb_per_split = g.kb_total;
    loss_args(g);
    ProfScope ps(c, s, "head_loss", 2.0 * n * hd.in * hd.out,
                 2.0 * n * hd.in + 2.0 * n * kHeadCols + (16.0 + 4.0 * g.n_heads) * n);
    if (srl_status st = gemm(64, false, false, EPI_LOSS, 1, ta, tb, to, to, g, sms, s, &grid_loss)) return st;
    colsum_parts[HI] = grid_loss;
  }
  // a6 through NVLink peer memory: finalise and extras write this rank's bucket into its
  // exposed buffer (parity of the step's epoch) and the allreduce kernel sums all ranks' into
  // c->grads.  Otherwise they write c->grads directly (NCCL allreduce in place, or world 1).
  const bool p2p = apply && c->world > 1 && c->p2p && !ar_overlap();
  const unsigned long long epoch = p2p ? c->epoch + 1 : 0;
  const int64_t xoff = (int64_t)(epoch & 1ull) * c->xstride();
  float* bk = p2p ? c->xbuf + xoff : c->grads;
  // ---------------- a5: backward.  dW via split-K partials, dX with fused dtanh + db sums
  // dW of layer index i (c->lay): D[dM][dN] = A^T B over the n samples (MN-major operands)
  auto dW = [&](int i, const __half* Amat, int lda, const __half* Bmat, int ldb) -> srl_status {
    const Lay& y = c->lay[i];
    const bool is_head = i == HI;
    const int dM = is_head ? y.in : y.out;
    const int dN = is_head ? kHeadCols : y.in;
    CUtensorMap ta, tb;
    TMC(ta, Amat, dM, n, (uint64_t)lda * 2, 64, 64);
    TMC(tb, Bmat, dN, n, (uint64_t)ldb * 2, 64, 64);
    GemmArgs g{};
    g.M = dM; g.N = dN;
    g.m_tiles = y.dw_m_tiles; g.n_tiles = y.dw_n_tiles;
    g.kb_total = (n + 63) / 64;
    int S = std::min(y.splits_max, g.kb_total);
    g.kb_per_split = (g.kb_total + S - 1) / S;
    S = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
    g.k_splits = S;
    g.part = y.part; g.ld_part = y.ld_part; g.part_split_stride = y.part_rows * y.ld_part;
    splits[i] = S;
    if (!is_head && dw_fixup_enabled() && dN % 4 == 0) {
      // the split-K sum inside the launch, straight into the bucket the exchange / Adam read
      g.red_out = bk + y.w_off; g.red_scale = inv_n; g.red_bar = c->gbar + 4;
      g.red_discard = dw_discard_enabled();
      g.counters = c->counters;
      reduced[i] = 1;
    }
    const int realN = is_head ? y.out : dN;
    ProfScope ps(c, s, is_head ? "dW_head" : (y.l == 0 ? "dW_l1" : "dW_hidden"),
                 2.0 * n * dM * realN, 2.0 * n * (dM + dN) + 4.0 * S * dM * y.ld_part);
    return gemm(y.bn_dw, true, true, EPI_PART, y.cg_dw, ta, tb, ta, ta, g, sms, s);
  };
  // dX of layer index i: dZ_in = (dZ_out W) * (1 - Y_in^2) with the input's column sums;
  // operands as (pointer, row stride) so a trunk works on its column half
  auto dX = [&](int i, const __half* dz_in, int k_width, int ld_in, __half* dz_out,
                const __half* yprev, int ld_out, float* colsum, int colsum_ld) -> srl_status {
    const Lay& y = c->lay[i];
    const bool is_head = i == HI;
    CUtensorMap ta, tb;
    TMC(ta, dz_in, k_width, n, (uint64_t)ld_in * 2, 64, 128);
    TMC(tb, y.w16, y.in, y.w16_rows, (uint64_t)y.w16_ld * 2, 64, 64);
    CUtensorMap to, ty;
    TMC(to, dz_out, y.in, n, (uint64_t)ld_out * 2, 32, 32, 64);
    TMC(ty, yprev, y.in, n, (uint64_t)ld_out * 2, 32, 32, 64);
    GemmArgs g{};
    g.M = n; g.N = y.in;
    g.m_tiles = (n + 128 * y.cg_dx - 1) / (128 * y.cg_dx); g.n_tiles = y.in / y.bn_dx; g.k_splits = 1;
    g.kb_total = (k_width + 63) / 64; g.kb_per_split = g.kb_total;
    g.colsum = colsum; g.colsum_ld = colsum_ld;
    g.counters = c->counters;
    int grid = 0;
    const int realK = is_head ? y.out : k_width;
    ProfScope ps(c, s, is_head ? "dX_head" : "dX_hidden", 2.0 * n * realK * y.in,
                 2.0 * n * (k_width + 2.0 * y.in) + 2.0 * y.in * k_width);
    srl_status st = gemm(y.bn_dx, false, true, EPI_DTANH, y.cg_dx, ta, tb, to, ty, g, sms, s, &grid);
    if (is_head) dz_parts = grid;
    else colsum_parts[c->hidx(y.t, y.l - 1)] = grid;
    return st;
  };
  // finalise (1/N-scaled split/column-sum reduction into the bucket) layers [lo, hi] (T = 1)
  auto finalize_layers = [&](int lo, int hi) -> srl_status {
    SegTable all = make_segs(c, splits, colsum_parts, dz_parts, reduced), t{};
    double rd = 0;
    for (int l = lo; l <= hi; ++l) {
      t.s[t.n++] = all.s[2 * l];
      t.s[t.n++] = all.s[2 * l + 1];
      rd += 4.0 * splits[l] * c->lay[l].out * c->lay[l].in + 4.0 * colsum_parts[l] * c->lay[l].colsum_ld;
    }
    ProfScope ps(c, s, "grad_finalize", 0.0, rd);
    CK(launch_finalize_grads(t, c->P, inv_n, bk, c->counters, s));
    return SRL_OK;
  };
  // a6 overlap: once dW of layer 1 is done, layers 1..L (a contiguous bucket tail) are final;
  // their allreduce runs on comm_stream during layer 0's dX/dW.
  // Opt-in (SRL_AR_OVERLAP=1, shared trunk only): measured slower on 2-4 B200 for the
  // Atari-shaped step, because NCCL's kernel takes SMs from the persistent GEMMs beside it.
  const bool overlap = apply && c->world > 1 && ar_overlap() && T == 1;
  const int64_t split_off = c->lay[std::min(1, L)].w_off;   // bucket [split_off, P) = layers 1..L
  auto early_reduce = [&]() -> srl_status {
    if (srl_status st = finalize_layers(1, L)) return st;
    CK(cudaEventRecord(c->ev_early, s));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_early, 0));
    ProfScope ps(c, c->comm_stream, "allreduce", 0.0, 4.0 * (c->P - split_off));
    CKN(ncclAllReduce(c->grads + split_off, c->grads + split_off, (size_t)(c->P - split_off),
                      ncclFloat, ncclSum, c->comm, c->comm_stream));
    return SRL_OK;
  };
  if (!fused) {
    if (srl_status st = dW(HI, c->Y[L - 1], hd.in, c->G16, kHeadCols)) return st;
  }
  if (overlap && L == 1) if (srl_status st = early_reduce()) return st;
  if (!fused) {
    if (srl_status st = dX(HI, c->G16, kHeadCols, kHeadCols, c->dZ[cur], c->Y[L - 1], hd.in,
                           hd.dz_colsum, hd.in)) return st;
  }
  for (int l = L - 1; l >= 0; --l) {
    for (int tr = 0; tr < T; ++tr) {
      const Lay& y = c->hid(tr, l);
      const __half* Xl = l == 0 ? X0 : c->Y[l - 1] + (size_t)tr * y.in;
      const int ldx = l == 0 ? ld_obs : T * y.in;
      if (srl_status st = dW(c->hidx(tr, l), c->dZ[cur] + (size_t)tr * y.out, T * y.out, Xl, ldx)) return st;
    }
    if (overlap && l == 1) if (srl_status st = early_reduce()) return st;
    if (l > 0) {
      for (int tr = 0; tr < T; ++tr) {
        const Lay& y = c->hid(tr, l);
        const Lay& yp = c->hid(tr, l - 1);
        if (srl_status st = dX(c->hidx(tr, l), c->dZ[cur] + (size_t)tr * y.out, y.out, T * y.out,
                               c->dZ[cur ^ 1] + (size_t)tr * y.in, c->Y[l - 1] + (size_t)tr * y.in,
                               T * y.in, yp.colsum, yp.colsum_ld)) return st;
      }
      cur ^= 1;
    }
  }
  SegTable segs = make_segs(c, splits, colsum_parts, dz_parts, reduced);
  const bool gclip = apply && c->cfg.max_grad_norm > 0.f;
  double part_bytes = 4.0 * dz_parts * hd.in;
  for (int i = 0; i <= HI; ++i)
    part_bytes += 4.0 * splits[i] * c->lay[i].out * c->lay[i].in + 4.0 * colsum_parts[i] * c->lay[i].colsum_ld;
  // the fused finalise -> [grad norm] -> Adam launch (update_kernel)
  auto update = [&](bool finalize, bool adam, float* bucket, bool stats) -> srl_status {
    UpdateArgs u{};
    u.stats = stats; u.apply = apply; u.mean_std = adv_mean_std; u.n_global = n_global;
    u.cv = c->cfg.value_coef; u.ce = c->cfg.entropy_coef; u.out = stats_out;
    u.t = segs; u.P = c->P; u.inv_n = inv_n; u.bucket = bucket; u.counters = c->counters;
    u.stats_part = c->stats_part; u.nstats = grid_loss;
    u.finalize = finalize; u.adam = adam;
    u.g = c->grads; u.p = c->params; u.m = c->m; u.v = c->v; u.t_dev = c->t_dev;
    u.lr = c->cfg.lr; u.b1 = c->cfg.beta1; u.b2 = c->cfg.beta2; u.eps = c->cfg.adam_eps;
    u.max_norm = gclip ? c->cfg.max_grad_norm : 0.f;
    u.gn_part = c->gn; u.gn_norm = c->gn_norm(); u.gn_coef = c->gn_coef();
    u.comm_err = c->world > 1 ? c->cc.err_dev : nullptr;
    u.bar = c->gbar;
    ProfScope ps(c, s, finalize ? (adam ? "grad_update" : "grad_finalize") : "adam",
                 0.0, (finalize ? part_bytes : 0.0) + (adam ? 30.0 * c->P : 0.0));
    CK(launch_update(u, s));
    return SRL_OK;
  };
  if (!overlap && p2p && xfused_enabled()) {
    // world > 1 over peer memory: ONE launch -- finalise into the exposed bucket, the two-shot
    // exchange into c->grads, [norm], Adam, statistics (misc.cu update_kernel, `xchg`)
    UpdateArgs u{};
    u.t = segs; u.P = c->P; u.inv_n = inv_n; u.bucket = bk; u.counters = c->counters;
    u.stats_part = c->stats_part; u.nstats = grid_loss;
    u.finalize = 1; u.adam = 1; u.stats = 1; u.apply = apply;
    u.g = c->grads; u.p = c->params; u.m = c->m; u.v = c->v; u.t_dev = c->t_dev;
    u.lr = c->cfg.lr; u.b1 = c->cfg.beta1; u.b2 = c->cfg.beta2; u.eps = c->cfg.adam_eps;
    u.max_norm = gclip ? c->cfg.max_grad_norm : 0.f;
    u.gn_part = c->gn; u.gn_norm = c->gn_norm(); u.gn_coef = c->gn_coef();
    u.comm_err = c->cc.err_dev;
    u.bar = c->gbar;
    u.mean_std = adv_mean_std; u.n_global = n_global;
    u.cv = c->cfg.value_coef; u.ce = c->cfg.entropy_coef; u.out = stats_out;
    u.xchg = 1; u.world = c->world; u.rank = c->rank; u.pe = c->peers; u.cc = c->cc;
    u.xoff = xoff; u.epoch = epoch; u.xout = c->grads;
    c->epoch = epoch;
    ProfScope ps(c, s, "grad_update_x", 0.0,
                 part_bytes + 4.0 * (c->P + 8) * 2.0 * (c->world - 1) / c->world + 30.0 * c->P);
    CK(launch_update(u, s));
  } else if (!overlap) {
    // world 1: ONE launch from the partials to the updated parameters; world > 1: finalise
    // into the bucket the exchange reads, exchange, then the norm + Adam launch
    // the last launch also writes the step's statistics (its last block)
    const bool one = apply && c->world == 1;
    if (srl_status st = update(true, one, bk, !apply || c->world == 1)) return st;
    if (apply && c->world > 1) {
      if (p2p) {
        ProfScope ps(c, s, "allreduce", 0.0, 4.0 * (c->P + 8) * 2.0 * (c->world - 1) / c->world);
        c->epoch = epoch;
        CK(launch_p2p_allreduce(c->peers, c->world, c->rank, xoff, c->P + 8, epoch, 1.f, c->grads,
                                c->cc, 3, s));
      } else {
        ProfScope ps(c, s, "allreduce", 0.0, 4.0 * (c->P + 8));
        CKN(ncclAllReduce(c->grads, c->grads, (size_t)(c->P + 8), ncclFloat, ncclSum, c->comm, s));
      }
      if (srl_status st = update(false, true, c->grads, true)) return st;
    }
  } else {
    // opt-in NCCL overlap path (SRL_AR_OVERLAP=1): layers 1..L were finalised and their
    // allreduce started during the backward; layer 0 + the statistics now
    if (srl_status st = finalize_layers(0, 0)) return st;
    CK(launch_extras(c->P, inv_n, c->stats_part, grid_loss, c->counters, bk, s));
    CK(cudaEventRecord(c->ev_late, s));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_late, 0));
    {
      ProfScope ps(c, c->comm_stream, "allreduce", 0.0, 4.0 * (split_off + 8));
      CKN(ncclGroupStart());
      CKN(ncclAllReduce(c->grads, c->grads, (size_t)split_off, ncclFloat, ncclSum, c->comm, c->comm_stream));
      CKN(ncclAllReduce(c->grads + c->P, c->grads + c->P, 8, ncclFloat, ncclSum, c->comm, c->comm_stream));
      CKN(ncclGroupEnd());
    }
    CK(cudaEventRecord(c->ev_comm, c->comm_stream));
    CK(cudaStreamWaitEvent(s, c->ev_comm, 0));
    if (gclip) {
      ProfScope ps(c, s, "grad_norm", 0.0, 4.0 * c->P);
      CK(launch_gradnorm(c->grads, c->P, c->gn, c->gn_counter, c->cfg.max_grad_norm,
                         c->gn_norm(), c->gn_coef(), s));
    }
    ProfScope ps(c, s, "adam", 0.0, 30.0 * c->P);
    CK(launch_adam(segs, c->P, c->params, c->m, c->v, c->grads, c->t_dev, c->cfg.lr,
                   c->cfg.beta1, c->cfg.beta2, c->cfg.adam_eps, s, gclip ? c->gn_coef() : nullptr,
                   c->cc.err_dev));
    ProfScope ps_stats(c, s, "stats", 0.0, 0.0);
    CK(launch_stats(c->grads, c->P, adv_mean_std, n_global, c->cfg.value_coef, c->cfg.entropy_coef,
                    c->t_dev, apply, stats_out, s, c->counters,
                    gclip ? c->gn_norm() : nullptr, c->world > 1 ? c->cc.err_dev : nullptr));
  }
  return SRL_OK;
}

// ------------------------------------------------------------------ a1..a7 in one call
extern "C" srl_status srl_ppo_train_step(srl_ctx* c, int T, int B, int64_t n_global,
                                         const float* rewards, const float* values,
                                         const uint8_t* dones, const float* trunc_values,
                                         const uint8_t* valid, const uint16_t* obs,
                                         const int32_t* actions, const float* logp_old,
                                         srl_ppo_stats* stats_out, srl_stream_t stream) {
  if (!c) FAIL(SRL_EINVAL, "srl_ppo_train_step: null ctx");
  if (srl_status st = comm_check(c, "srl_ppo_train_step")) return st;
  if (T < 1 || B < 1 || (int64_t)T * B > c->max_n || n_global < (valid ? 1 : (int64_t)T * B))
    FAIL(SRL_EINVAL, "srl_ppo_train_step: need 1 <= T*B <= max_local_n, T*B <= n_global "
                     "(n_global >= 1 with a valid mask)");
  if (!rewards || !values || !dones) FAIL(SRL_EINVAL, "srl_ppo_train_step: null trajectory input");
  const int nb = gae_num_blocks(B);
  if (nb > c->gae_part_cap) FAIL(SRL_EINVAL, "srl_ppo_train_step: B too large");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = (int64_t)T * B;
  {
    // a1 + a2 (local): the scan's last block merges the moments (world 1: straight to mean/std)
    ProfScope ps(c, s, "gae_scan", 0.0, 17.0 * n);
    CK(launch_gae(T, B, B, rewards, values, dones, trunc_values, valid, c->cfg.gamma,
                  c->cfg.gae_lambda, c->adv,
                  c->ret, c->gae_part, s, c->gae_counter, c->gae_stats,
                  c->world == 1 ? c->mean_std : nullptr, c->cfg.adv_unbiased));
  }
  if (c->world > 1) {
    // a2 (global): all-gather the ranks' {n, mean, M2} and merge them in rank order
    if (c->p2p && !ar_overlap()) {
      // on comm_stream, beside the forward GEMMs (which do not read mean/std): the exchange's
      // wait for the slowest rank overlaps a3; srl_ppo_step's loss launch waits for ev_ms.
      // One 256-thread block that co-resides with a GEMM CTA; it spins only on OTHER ranks.
      CK(cudaEventRecord(c->ev_gae, s));
      CK(cudaStreamWaitEvent(c->comm_stream, c->ev_gae, 0));
      {
        ProfScope ps(c, c->comm_stream, "adv_norm", 0.0, 24.0 * c->world);
        CK(launch_p2p_moments(c->peers, c->world, c->rank, ++c->mepoch, c->gae_stats, c->mean_std,
                              c->cfg.adv_unbiased, c->cc, 3, c->comm_stream));
      }
      CK(cudaEventRecord(c->ev_ms, c->comm_stream));
      c->ms_pending = true;
    } else {
      ProfScope ps(c, s, "adv_norm", 0.0, 24.0 * c->world);
      double* gathered = c->norm_scratch;
      CKN(ncclAllGather(c->gae_stats, gathered, 3, ncclDouble, c->comm, s));
      CK(launch_merge_moments(gathered, c->world, nullptr, c->mean_std, c->cfg.adv_unbiased, s));
    }
  }
  // a3..a7 once per minibatch per epoch (NEXT-3, reading R-M); E = M = 1 is one update
  const int E = c->cfg.epochs, M = c->cfg.minibatches;
  const float* v_old = c->cfg.value_clip > 0.f ? values : nullptr;   // rows 0..T-1 = V_old
  if (E == 1 && M == 1)
    return srl_ppo_step(c, n, n_global, obs, actions, logp_old, c->adv, c->ret, v_old, valid,
                        c->mean_std, 1, stats_out, stream);
  if (M > 1 && n_global != (int64_t)c->world * n)
    FAIL(SRL_EINVAL, "srl_ppo_train_step: minibatches > 1 needs the same T*B on every rank");
  if (M > n) FAIL(SRL_EINVAL, "srl_ppo_train_step: minibatches > T*B");
  if (M > 1 && valid)   // N_k would be the valid count of each global minibatch: not on the host
    FAIL(SRL_EUNSUPPORTED, "srl_ppo_train_step: minibatches > 1 with a valid mask");
  const int H = (int)c->heads.size();
  const int64_t ld = c->cfg.ld_obs;
  for (int e = 0; e < E; ++e)
    for (int k = 0; k < M; ++k) {
      const int64_t lo = k * n / M, hi = (k + 1) * n / M;
      const int64_t nk = hi - lo;
      if (srl_status st = srl_ppo_step(c, nk, M == 1 ? n_global : (int64_t)c->world * nk, obs + lo * ld,
                                       actions + lo * H, logp_old + lo, c->adv + lo, c->ret + lo,
                                       v_old ? v_old + lo : nullptr, valid ? valid + lo : nullptr,
                                       c->mean_std, 1, stats_out, stream))
        return st;
    }
  return SRL_OK;
}

// ------------------------------------------------------------------ NEXT-2 policy inference
extern "C" srl_status srl_policy_rollout(srl_ctx* c, int64_t n, const uint16_t* obs,
                                         const uint64_t* keys, uint64_t seed, int deterministic,
                                         int32_t* actions_out, float* logp_out, float* value_out,
                                         srl_stream_t stream) {
  if (!c) FAIL(SRL_EINVAL, "srl_policy_rollout: null ctx");
  if (n < 1 || n > c->max_n) FAIL(SRL_EINVAL, "srl_policy_rollout: need 1 <= n <= max_local_n");
  if (!obs || !actions_out || !logp_out || !value_out) FAIL(SRL_EINVAL, "srl_policy_rollout: null pointer");
  if ((reinterpret_cast<uintptr_t>(obs) & 15) != 0) FAIL(SRL_EINVAL, "srl_policy_rollout: obs must be 16-byte aligned");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nn = (int)n;
  if (srl_status st = forward_hidden(c, nn, reinterpret_cast<const __half*>(obs), s)) return st;
  const Lay& hd = c->head();
  CUtensorMap ta, tb;
  TMC(ta, c->Y[c->L - 1], hd.in, nn, (uint64_t)hd.in * 2, 64, 128);
  TMC(tb, hd.w16, hd.in, kHeadCols, (uint64_t)hd.w16_ld * 2, 64, 64);
  GemmArgs g{};
  g.M = nn; g.N = kHeadCols;
  g.m_tiles = (nn + 127) / 128; g.n_tiles = 1; g.k_splits = 1;
  g.kb_total = (hd.in + 63) / 64; g.kb_per_split = g.kb_total;
  g.bias = c->T == 1 ? c->params + hd.b_off : c->hbias;
  g.n_heads = (int)c->heads.size(); g.A = c->A;
  for (int h = 0; h < g.n_heads; ++h) g.head_size[h] = c->heads[h];
  g.seed = seed; g.keys = reinterpret_cast<const unsigned long long*>(keys);
  g.deterministic = deterministic;
  g.act_out = actions_out; g.logp_out = logp_out; g.value_out = value_out;
  ProfScope ps(c, s, "head_sample", 2.0 * nn * hd.in * hd.out,
               2.0 * nn * hd.in + (8.0 + 4.0 * g.n_heads) * nn);
  return gemm(64, false, false, EPI_SAMPLE, 1, ta, tb, ta, ta, g, c->sms, s);
}

// ------------------------------------------------------------------ NEXT-1 pre-fetching
extern "C" srl_status srl_batch_upload(srl_ctx* c, int slot, int T, int B, const float* rewards,
                                       const float* values, const uint8_t* dones,
                                       const uint16_t* obs, const int32_t* actions,
                                       const float* logp_old, const float* trunc_values,
                                       const uint8_t* valid) {
  if (!c || slot < 0 || slot > 1) FAIL(SRL_EINVAL, "srl_batch_upload: bad ctx/slot");
  if (T < 1 || B < 1 || (int64_t)T * B > c->max_n) FAIL(SRL_EINVAL, "srl_batch_upload: need 1 <= T*B <= max_local_n");
  if (!rewards || !values || !dones || !obs || !actions || !logp_old)
    FAIL(SRL_EINVAL, "srl_batch_upload: null pointer");
  CK(cudaSetDevice(c->device));
  auto& sl = c->slot[slot];
  const int64_t n = c->max_n;
  if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!sl.obs) {
    srl_status st;
    if ((st = dalloc(c, &sl.rewards, sizeof(float) * n))) return st;
    if ((st = dalloc(c, &sl.values, sizeof(float) * 2 * n))) return st;   // (T+1)B <= 2TB
    if ((st = dalloc(c, &sl.dones, n))) return st;
    if ((st = dalloc(c, &sl.obs, sizeof(__half) * n * c->cfg.ld_obs))) return st;
    if ((st = dalloc(c, &sl.actions, sizeof(int32_t) * n * c->heads.size()))) return st;
    if ((st = dalloc(c, &sl.logp_old, sizeof(float) * n))) return st;
    CK(cudaEventCreateWithFlags(&sl.uploaded, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl.released, cudaEventDisableTiming));
    CK(cudaDeviceSynchronize());                   // the zeroing memsets (see below)
    CK(cudaEventRecord(sl.released, c->copy_stream));
  }
  bool fresh = false;
  if (trunc_values && !sl.trunc_values) {
    if (srl_status st = dalloc(c, &sl.trunc_values, sizeof(float) * n)) return st;
    fresh = true;
  }
  if (valid && !sl.valid) {
    if (srl_status st = dalloc(c, &sl.valid, n)) return st;
    fresh = true;
  }
  // dalloc zeroes new buffers with cudaMemset on the legacy stream, which the non-blocking copy
  // stream does not wait for: finish the zeroing before the first upload into them
  if (fresh) CK(cudaDeviceSynchronize());
  const int64_t m = (int64_t)T * B;
  cudaStream_t cs = c->copy_stream;
  CK(cudaStreamWaitEvent(cs, sl.released, 0));      // the last step on this slot is done with it
  CK(cudaMemcpyAsync(sl.rewards, rewards, sizeof(float) * m, cudaMemcpyHostToDevice, cs));
  CK(cudaMemcpyAsync(sl.values, values, sizeof(float) * (m + B), cudaMemcpyHostToDevice, cs));
  CK(cudaMemcpyAsync(sl.dones, dones, m, cudaMemcpyHostToDevice, cs));
  CK(cudaMemcpyAsync(sl.obs, obs, sizeof(__half) * m * c->cfg.ld_obs, cudaMemcpyHostToDevice, cs));
  CK(cudaMemcpyAsync(sl.actions, actions, sizeof(int32_t) * m * c->heads.size(), cudaMemcpyHostToDevice, cs));
  CK(cudaMemcpyAsync(sl.logp_old, logp_old, sizeof(float) * m, cudaMemcpyHostToDevice, cs));
  if (trunc_values)
    CK(cudaMemcpyAsync(sl.trunc_values, trunc_values, sizeof(float) * m, cudaMemcpyHostToDevice, cs));
  if (valid) CK(cudaMemcpyAsync(sl.valid, valid, m, cudaMemcpyHostToDevice, cs));
  sl.has_tv = trunc_values != nullptr;
  sl.has_valid = valid != nullptr;
  CK(cudaEventRecord(sl.uploaded, cs));
  sl.T = T;
  sl.B = B;
  sl.ready = true;
  return SRL_OK;
}

extern "C" srl_status srl_ppo_train_step_slot(srl_ctx* c, int slot, int64_t n_global,
                                              srl_ppo_stats* stats_out, srl_stream_t stream) {
  if (!c || slot < 0 || slot > 1) FAIL(SRL_EINVAL, "srl_ppo_train_step_slot: bad ctx/slot");
  auto& sl = c->slot[slot];
  if (!sl.ready) FAIL(SRL_ESTATE, "srl_ppo_train_step_slot: slot has no uploaded batch");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaStreamWaitEvent(s, sl.uploaded, 0));
  srl_status st = srl_ppo_train_step(c, sl.T, sl.B, n_global, sl.rewards, sl.values, sl.dones,
                                     sl.has_tv ? sl.trunc_values : nullptr,
                                     sl.has_valid ? sl.valid : nullptr,
                                     reinterpret_cast<const uint16_t*>(sl.obs), sl.actions,
                                     sl.logp_old, stats_out, stream);
  CK(cudaEventRecord(sl.released, s));
  sl.ready = false;
  return st;
}

// ------------------------------------------------------------------ profiling
extern "C" srl_status srl_prof_enable(srl_ctx* c, int on) {
  if (!c) FAIL(SRL_EINVAL, "srl_prof_enable: null ctx");
  c->prof = on != 0;
  return SRL_OK;
}

extern "C" srl_status srl_prof_reset(srl_ctx* c) {
  if (!c) FAIL(SRL_EINVAL, "srl_prof_reset: null ctx");
  c->recs.clear();
  c->pool_used = 0;
  return SRL_OK;
}

extern "C" int srl_prof_count(srl_ctx* c) { return c ? (int)c->recs.size() : 0; }

extern "C" srl_status srl_prof_read(srl_ctx* c, int i, const char** name, float* ms,
                                    double* flops, double* bytes) {
  if (!c || i < 0 || i >= (int)c->recs.size()) FAIL(SRL_EINVAL, "srl_prof_read: index");
  const auto& r = c->recs[i];
  CK(cudaSetDevice(c->device));
  CK(cudaEventSynchronize(r.b));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, r.a, r.b));
  if (name) *name = r.name;
  if (ms) *ms = t;
  if (flops) *flops = r.flops;
  if (bytes) *bytes = r.bytes;
  return SRL_OK;
}

// ------------------------------------------------------------------ test hook
__global__ void sum_parts_kernel(const float* part, int S, int64_t split_stride, int M, int N,
                                 int64_t ld_part, float* D) {
  griddep_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)M * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / N), cc = (int)(i % N);
    float acc = 0.f;
    for (int k = 0; k < S; ++k) acc += part[k * split_stride + r * ld_part + cc];
    D[i] = acc;
  }
}

extern "C" srl_status srl_debug_gemm(int M, int N, int K, const uint16_t* A, int a_mn, int lda,
                                     const uint16_t* B, int b_mn, int ldb, int bn, int splits,
                                     int cg, float* D, srl_stream_t stream) {
  if (M < 1 || N < 1 || K < 1 || !A || !B || !D || lda % 8 || ldb % 8 || splits < 1)
    FAIL(SRL_EINVAL, "srl_debug_gemm: bad args");
  if (bn != 64 && bn != 128 && bn != 256 && bn != 512) FAIL(SRL_EINVAL, "srl_debug_gemm: bn");
  if (bn == 512 && (cg != 2 || !a_mn || !b_mn))
    FAIL(SRL_EINVAL, "srl_debug_gemm: bn = 512 is the CTA-pair MN-major x MN-major (dW) tile");
  if (cg != 1 && cg != 2) FAIL(SRL_EINVAL, "srl_debug_gemm: cg");
  if (cg == 2 && bn == 64) FAIL(SRL_EINVAL, "srl_debug_gemm: cg = 2 needs bn >= 128");
  if (srl_status st = require_device()) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CUtensorMap ta, tb;
  if (!a_mn) TM(ta, A, K, M, (uint64_t)lda * 2, 64, 128);
  else TM(ta, A, M, K, (uint64_t)lda * 2, 64, 64);
  if (!b_mn) TM(tb, B, K, N, (uint64_t)ldb * 2, 64, bn / cg);
  else TM(tb, B, N, K, (uint64_t)ldb * 2, 64, 64);
  GemmArgs g{};
  g.M = M; g.N = N;
  g.m_tiles = (M + 128 * cg - 1) / (128 * cg); g.n_tiles = (N + bn - 1) / bn;
  g.kb_total = (K + 63) / 64;
  int S = std::min(splits, g.kb_total);
  g.kb_per_split = (g.kb_total + S - 1) / S;
  S = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  g.k_splits = S;
  g.ld_part = (int64_t)g.n_tiles * bn;
  g.part_split_stride = (int64_t)M * g.ld_part;
  float* part = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(float) * S * g.part_split_stride, s));
  g.part = part;
  if (srl_status st = gemm(bn, a_mn != 0, b_mn != 0, EPI_PART, cg, ta, tb, ta, ta, g, num_sms(), s)) return st;
  CK(launch_k(sum_parts_kernel, dim3(256), dim3(256), 0, s, 1, (const float*)part, S,
              (int64_t)g.part_split_stride, M, N, (int64_t)g.ld_part, D));
  CK(cudaGetLastError());
  CK(cudaFreeAsync(part, s));
  return SRL_OK;
}

// ------------------------------------------------------------------ test hook: a2/a6 exchange
// The production exchange kernels (p2p_allreduce_kernel, p2p_moments_kernel) run for `world`
// VIRTUAL ranks on this one GPU: rank r's exposed bucket is x + r*ld and its sync block a local
// allocation.  No launch ever waits on another (B200_PROFILING.md: ranks that spin on each
// other must not be separate launches on one GPU): every flag a rank would wait for is
// pre-published, and the phases run in order -- phase 1 (publish + reduce my chunk) of every
// rank, then phase 2 (gather the other chunks) of every rank -- which is the order the real
// flags enforce.
static __global__ void fill_u64_kernel(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

extern "C" srl_status srl_debug_exchange(int world, int64_t count, int64_t ld, float* x, float* out,
                                         float scale, const double* tri, double* mean_std,
                                         int unbiased, srl_stream_t stream) {
  if (world < 1 || world > kMaxPeers || count < 1 || ld < count || ld % 4 || !x || !out)
    FAIL(SRL_EINVAL, "srl_debug_exchange: need 1 <= world <= 8, 1 <= count <= ld, ld % 4 == 0");
  if ((tri == nullptr) != (mean_std == nullptr)) FAIL(SRL_EINVAL, "srl_debug_exchange: tri and mean_std go together");
  if (srl_status st = require_device()) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long* sync = nullptr;
  int* err = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&sync), kSyncBytes * world, s));
  CK(cudaMallocAsync(reinterpret_cast<void**>(&err), sizeof(int) * 2, s));
  CK(cudaMemsetAsync(sync, 0, kSyncBytes * world, s));
  CK(cudaMemsetAsync(err, 0, sizeof(int) * 2, s));
  const unsigned long long epoch = 1;
  P2PPeers pe{};
  for (int r = 0; r < world; ++r) {
    pe.x[r] = x + (int64_t)r * ld;
    pe.flag[r] = sync + (int64_t)r * kSyncWords;
    // pre-publish every flag a rank waits for: phase-1 slots and the reduced-chunk slots
    CK(launch_k(fill_u64_kernel, dim3(4), dim3(256), 0, s, 1, pe.flag[r], (int64_t)(2 * kMaxPeers), epoch));
    CK(launch_k(fill_u64_kernel, dim3(4), dim3(256), 0, s, 1, p2p_rflags(pe.flag[r]),
                (int64_t)kMaxPeers * kXBlocks, epoch));
  }
  CommCtl cc{err, err + 1, 1000000000ull};
  for (int ph = 1; ph <= 2; ++ph)
    for (int r = 0; r < world; ++r) {
      CK(launch_p2p_allreduce(pe, world, r, 0, count, epoch, scale, out + (int64_t)r * ld, cc, ph, s));
      if (tri) CK(launch_p2p_moments(pe, world, r, epoch, tri + 3 * r, mean_std + 2 * r, unbiased, cc, ph, s));
    }
  CK(cudaGetLastError());
  int herr[2] = {0, 0};
  CK(cudaMemcpyAsync(herr, err, sizeof(herr), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaFreeAsync(sync, s));
  CK(cudaFreeAsync(err, s));
  if (herr[0] || herr[1]) FAIL(SRL_ENCCL, "srl_debug_exchange: a pre-published wait timed out");
  return SRL_OK;
}
