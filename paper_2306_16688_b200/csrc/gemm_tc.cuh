// gemm_tc.cuh -- warp-specialised TMA + tcgen05 GEMM for sm_100a with the trainer's fused
// epilogues.  D[M][N] = sum_k A(m,k) * B(n,k), fp16 operands, fp32 accumulation in TMEM.
//
//   A(m,k): K-major = row-major [M][K] (A_MN=false)  |  MN-major = row-major [K][M] (A_MN=true)
//   B(n,k): K-major = row-major [N][K] (B_MN=false)  |  MN-major = row-major [K][N] (B_MN=true)
//
// Tile 128 x BN x 64, SWIZZLE_128B smem operands fed by TMA through an mbarrier ring of
// args.stages slots; one elected thread issues tcgen05.mma (kind::f16, M=128) into 512/BN
// TMEM accumulators, so the MMA runs up to 512/BN - 1 tiles ahead of the epilogue.
// Persistent CTAs walk the work units (m tile, n tile, k split) with a static stride, so every
// per-CTA partial is deterministic.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w3 idle,
// w4..w11 epilogue in two warpgroups g = 0, 1 that take alternate tiles (tile i uses TMEM
// stage i % ACC_STAGES, drained by group i % 2); warp w reads TMEM lanes 32(w%4)..+31.
// Epilogue output goes through per-warp 32x32 fp16 staging tiles (64-byte swizzle, conflict
// free) and leaves by TMA bulk-tensor stores; y_prev tiles arrive by TMA loads.
//
// Epilogues (rows a3-a5):
//   EPI_TANH  : out16 = tanh(acc + bias)                          (forward hidden layer, a3)
//   EPI_DTANH : dz16 = acc * (1 - y^2), + per-CTA column sums     (backward dX, a5; db)
//   EPI_PART  : part32[ks] = acc                                  (backward dW split-K, a5)
//   EPI_LOSS  : head logits -> PPO loss, per-sample dlogits, stats (a4)
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "ptx.cuh"

namespace srl {

enum { EPI_TANH = 0, EPI_DTANH = 1, EPI_PART = 2, EPI_LOSS = 3, EPI_TANH_ACC = 4, EPI_SAMPLE = 5 };

constexpr int kMaxHeads = 8;
constexpr int kHeadCols = 64;   // padded head width G (logits + value + zero pad)

struct GemmArgs {
  int M, N;                       // valid rows / cols of D
  int m_tiles, n_tiles, k_splits;
  int kb_total, kb_per_split;     // 64-wide k blocks
  int stages;                     // operand ring slots (<= 8), from gemm_stages()
  // outputs / epilogue inputs (TANH/DTANH/LOSS write through the output tensor map)
  float* part; int64_t ld_part; int64_t part_split_stride;   // PART
  // PART with red_out: after a grid barrier the kernel itself sums the k_splits partials (in
  // split order, L2-hot) into red_out[M][N] scaled by red_scale (the 1/N-scaled gradient)
  float* red_out; float red_scale; unsigned* red_bar; int red_discard;
  const float* bias;                              // TANH, LOSS
  float* colsum; int colsum_ld;                   // DTANH, LOSS: [grid][colsum_ld]
  unsigned long long* counters;                   // [0] nonfinite, [1] fp16 saturations
  // loss (a4)
  const int32_t* actions; const float* logp_old; const float* adv; const float* ret;
  const double* mean_std; double* stats;          // stats: [grid][8]
  int n_heads, A;
  int head_size[kMaxHeads];
  float clip_eps, value_coef, entropy_coef, adv_eps;
  const float* v_old; float value_clip;           // NEXT-3 value clipping (v_old null: off)
  const uint8_t* valid;                           // NEXT-3 padding mask [M] (null: all valid)
  // NEXT-2 policy inference (EPI_SAMPLE): counter-RNG sampling or argmax per head
  unsigned long long seed; const unsigned long long* keys; int deterministic;
  int32_t* act_out; float* logp_out; float* value_out;
};

// Shared-memory layout (identical on host and device):
//   [operand ring][out staging 32 KB][y staging 32 KB (DTANH)][colsum 8 x ld][bias 4 KB][bars]
struct SmemLayout {
  uint32_t ring, ostage, ystage, colsum, bias, zbuf, bars, total;
};
constexpr int kZPitch = 33;                       // loss row buffer [64 cols][33] per warp
constexpr int kStageTile = 32 * 32 * 2;           // one 32x32 fp16 staging tile
#ifndef SRL_Y_SLOTS
#define SRL_Y_SLOTS 2
#endif
#ifndef SRL_OUT_SLOTS
#define SRL_OUT_SLOTS 2
#endif
constexpr int kYSlots = SRL_Y_SLOTS;              // y_prev ring per warp (1 chunk in flight)
constexpr int kOutSlots = SRL_OUT_SLOTS;          // output staging tiles per warp
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kBarBytes = 640;                    // 64 mbarriers + TMEM slot
constexpr uint32_t kSmemLimit = 232448;           // 227 KB per CTA

// zcols: columns of the per-warp row buffer of the loss / sample epilogues (A + 1 + H)
__host__ __device__ inline SmemLayout smem_layout(int bn, int epi, int stages, int colsum_ld,
                                                  int cg = 1, int zcols = 64 + 8) {
  SmemLayout L;
  const uint32_t stage_bytes = (uint32_t)(128 + bn / cg) * 64 * 2;
  L.ring = 0;
  L.ostage = stages * stage_bytes;
  const uint32_t ost = (epi == EPI_PART || epi == EPI_SAMPLE) ? 0 : kEpiWarps * kOutSlots * kStageTile;
  L.ystage = L.ostage + ost;
  const uint32_t yst = (epi == EPI_DTANH) ? kEpiWarps * kYSlots * kStageTile : 0;
  L.colsum = L.ystage + yst;
  const uint32_t cs = (epi == EPI_DTANH || epi == EPI_LOSS) ? kEpiWarps * colsum_ld * 4 : 0;
  L.bias = L.colsum + cs;
  const uint32_t bs = (epi == EPI_TANH || epi == EPI_LOSS || epi == EPI_SAMPLE) ? 4096 : 0;
  L.zbuf = L.bias + bs;
  const uint32_t zs = (epi == EPI_LOSS || epi == EPI_SAMPLE) ? kEpiWarps * zcols * kZPitch * 4 : 0;
  L.bars = L.zbuf + zs;
  L.total = L.bars + kBarBytes;
  return L;
}

// largest ring (<= 8 slots) that fits next to the epilogue buffers; 1 KB alignment slack and
// 512 B for the kernel's static shared memory
inline int gemm_stages(int bn, int epi, int colsum_ld, int cg = 1, int zcols = 64 + 8) {
  const uint32_t stage_bytes = (uint32_t)(128 + bn / cg) * 64 * 2;
  const SmemLayout z = smem_layout(bn, epi, 0, colsum_ld, cg, zcols);
  const int64_t avail = (int64_t)kSmemLimit - 1024 - 512 - z.total;
  const int st = (int)(avail / stage_bytes);
  return st > 8 ? 8 : st;
}

// CG = 1: one CTA computes a 128 x BN tile.  CG = 2: a CTA pair (cluster of 2) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2 issued by the leader: each CTA holds its 128
// rows of A and half of B (BN/2 columns) in smem, and its 128 rows of D in its own TMEM.
template <int BN, int CG = 1>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TX_BYTES = CG * STAGE_BYTES;   // bytes the leader's full barrier expects
  static constexpr int ACC_STAGES = 512 / BN;     // TMEM accumulators: 1 / 2 / 4 / 8
  // BN = 512 (dW only): two N = 256 MMAs per K step share the A tile (A read once per tile)
  static constexpr int MMA_N = BN > 256 ? 256 : BN;
  static constexpr int N_HALVES = BN / MMA_N;
  static constexpr int BOXES_PER_HALF = MMA_N / CG / 64;   // 64-col MN-major B boxes per CTA
  static constexpr int TMEM_COLS = 512;
};

__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t parity) {
  // the thread sleeps in try_wait (suspend-time hint) instead of spinning and stealing issue
  // slots from working warps; bounded: a lost arrival (a kernel bug, never another rank)
  // traps after ~17 s so the error reaches the host instead of a hang
  if (mbar_try_wait_sleep(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait_sleep(bar, parity))
    if (clock64() - t0 > (1ll << 35)) __trap();
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// lane j ends with sum over the 32 lanes of v[j] (31 shuffles, fixed order)
__device__ __forceinline__ float transpose_reduce32(float (&v)[32]) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      float send = up ? v[i] : v[i + w];
      float keep = up ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return v[0];
}

__device__ __forceinline__ float sat_f16(float x, uint32_t& nsat) {
  if (fabsf(x) > 65504.f) { ++nsat; x = copysignf(65504.f, x); }
  return x;
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// row `r` (0..31) of a 32x32 fp16 staging tile in the TMA 64-byte swizzle: the 16-byte chunk
// q of a row lives at chunk q ^ ((r >> 1) & 3).  Eight consecutive rows then hit 8 distinct
// 16-byte bank groups: the row-per-thread writes/reads are conflict free.
__device__ __forceinline__ uint32_t stile_off(int r, int q) {
  return (uint32_t)(r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
}

__device__ __forceinline__ void stile_write_row(uint8_t* tile, int r, const float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_half2(v[8 * q + 0], v[8 * q + 1]);
    u.y = pack_half2(v[8 * q + 2], v[8 * q + 3]);
    u.z = pack_half2(v[8 * q + 4], v[8 * q + 5]);
    u.w = pack_half2(v[8 * q + 6], v[8 * q + 7]);
    *reinterpret_cast<uint4*>(tile + stile_off(r, q)) = u;
  }
}

__device__ __forceinline__ void stile_read_row(const uint8_t* tile, int r, float (&y)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = *reinterpret_cast<const uint4*>(tile + stile_off(r, q));
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      y[8 * q + 2 * e] = f.x;
      y[8 * q + 2 * e + 1] = f.y;
    }
  }
}

__device__ __forceinline__ void count_warp(unsigned long long* ctr, uint32_t n) {
  // warp-aggregated integer atomic (deterministic total)
  uint32_t tot = __reduce_add_sync(0xffffffffu, n);
  if (lane_id() == 0 && tot) atomicAdd(ctr, (unsigned long long)tot);
}

// ---------------------------------------------------------------------------------------
// a4: PPO loss for the warp's 32 rows.  zb[j * kZPitch + lane] holds logit j (bias added) of
// row `lane`; on return it holds dloss_i/dz_j (j <= A), the per-sample logit gradient.
// Compact runtime loops over the A+1 real columns only (no 64-wide unrolling).
// Formulas: DESIGN.md §3.1 (SURVEY C-4).
__device__ __forceinline__ void ppo_rows_smem(const GemmArgs& a, float* zb, const int32_t* arow,
                                              float Ahat, float lp_old, float R, float vo,
                                              bool rvalid, double (&st)[5], uint32_t& nonfinite) {
  const uint32_t lane = lane_id();
  float* z = zb + lane;                       // z[j * kZPitch]: this row's column j
  float logpi = 0.f, ent = 0.f;
  float* Hh = z + (a.A + 1) * kZPitch;        // per-head entropies, columns A+1 .. A+H
  int off = 0;
#pragma unroll 1
  for (int h = 0; h < a.n_heads; ++h) {
    const int sz = a.head_size[h];
    float mx = -INFINITY;
#pragma unroll 4
    for (int j = off; j < off + sz; ++j) mx = fmaxf(mx, z[j * kZPitch]);
    float se = 0.f;
#pragma unroll 4
    for (int j = off; j < off + sz; ++j) se += __expf(z[j * kZPitch] - mx);
    const float lse = mx + __logf(se);
    float hh = 0.f;
#pragma unroll 4
    for (int j = off; j < off + sz; ++j) {
      const float l = z[j * kZPitch] - lse;    // log-softmax, kept in place
      z[j * kZPitch] = l;
      hh -= __expf(l) * l;
    }
    Hh[h * kZPitch] = hh;
    ent += hh;
    logpi += z[(off + (arow ? __ldg(arow + h) : 0)) * kZPitch];
    off += sz;
  }
  const float rho = expf(logpi - lp_old);
  const float lo = 1.f - a.clip_eps, hi = 1.f + a.clip_eps;
  const float rc = fminf(fmaxf(rho, lo), hi);
  const float lpg = -fminf(rho * Ahat, rc * Ahat);
  const float V = z[a.A * kZPitch];
  const float dv = V - R;
  float lv = dv * dv;
  float gv = 2.f * dv;                       // d lv / dV
  if (a.v_old) {                             // NEXT-3 value clipping (reading R-V)
    const float d = V - vo;
    const float dc = vo + fminf(fmaxf(d, -a.value_clip), a.value_clip) - R;
    if (dc * dc > lv) {
      lv = dc * dc;
      gv = fabsf(d) <= a.value_clip ? 2.f * dc : 0.f;
    }
  }
  const float mask = (Ahat >= 0.f) ? (rho <= hi ? 1.f : 0.f) : (rho >= lo ? 1.f : 0.f);
  const float pol = -mask * Ahat * rho;      // coefficient of (onehot - p)
  const float li = lpg + a.value_coef * lv - a.entropy_coef * ent;
  const bool ok = rvalid && isfinite(li);
  off = 0;
#pragma unroll 1
  for (int h = 0; h < a.n_heads; ++h) {
    const int sz = a.head_size[h];
    const int ah = off + (arow ? __ldg(arow + h) : 0);
    const float H = Hh[h * kZPitch];
#pragma unroll 4
    for (int j = off; j < off + sz; ++j) {
      const float l = z[j * kZPitch];
      const float p = __expf(l);
      const float g = pol * ((j == ah ? 1.f : 0.f) - p) + a.entropy_coef * p * (l + H);
      z[j * kZPitch] = ok ? g : 0.f;
    }
    off += sz;
  }
  z[a.A * kZPitch] = ok ? a.value_coef * gv : 0.f;
  if (!rvalid) return;
  if (!ok) {
    ++nonfinite;
    return;
  }
  st[0] += lpg;
  st[1] += lv;
  st[2] += ent;
  st[3] += fabsf(rho - 1.f) > a.clip_eps ? 1.0 : 0.0;
  st[4] += lp_old - logpi;
}

// a4 for ONE categorical head (A actions, value at column A; A + 1 <= 32) with the row in
// registers: z[j] = logit j (bias added) of this lane's row on entry, dloss_i/dz_j on return
// (0 past A).  The same formulas and per-row operations as ppo_rows_smem (
// SPEC.md S:L603-611), in the same order (bit-identical g).  act = the row's action (any
// value if !rvalid).
__device__ __forceinline__ void ppo_row_regs(const GemmArgs& a, float (&z)[32], int act,
                                             float Ahat, float lp_old, float R, float vo,
                                             bool rvalid, double (&st)[5], uint32_t& nonfinite) {
  const int A = a.A;
  // the columns in 8-wide chunks; chunks past the value column are skipped by a warp-uniform
  // branch (A + 1 = 19 for Atari: 3 of 4 chunks), the same operations in the same order
  const int nch = (A + 1 + 7) >> 3;
  float V = 0.f, mx = -INFINITY;
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8)
    if (c8 < nch) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 8 * c8 + i;
        if (j < A) mx = fmaxf(mx, z[j]);
        if (j == A) V = z[j];                    // the value column (not a logit)
      }
    }
  float se = 0.f;
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8)
    if (c8 < nch) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 8 * c8 + i;
        if (j < A) se += __expf(z[j] - mx);
      }
    }
  const float lse = mx + __logf(se);
  float ent = 0.f, logpi = 0.f;
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8)
    if (c8 < nch) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 8 * c8 + i;
        const float l = z[j] - lse;              // log-softmax
        if (j < A) ent -= __expf(l) * l;         // entropy
        z[j] = l;
        if (j == act) logpi = l;
      }
    }
  const float rho = expf(logpi - lp_old);
  const float lo = 1.f - a.clip_eps, hi = 1.f + a.clip_eps;
  const float rc = fminf(fmaxf(rho, lo), hi);
  const float lpg = -fminf(rho * Ahat, rc * Ahat);
  const float dv = V - R;
  float lv = dv * dv;
  float gv = 2.f * dv;
  if (a.v_old) {                                 // NEXT-3 value clipping (reading R-V)
    const float d = V - vo;
    const float dc = vo + fminf(fmaxf(d, -a.value_clip), a.value_clip) - R;
    if (dc * dc > lv) {
      lv = dc * dc;
      gv = fabsf(d) <= a.value_clip ? 2.f * dc : 0.f;
    }
  }
  const float mask = (Ahat >= 0.f) ? (rho <= hi ? 1.f : 0.f) : (rho >= lo ? 1.f : 0.f);
  const float pol = -mask * Ahat * rho;
  const float li = lpg + a.value_coef * lv - a.entropy_coef * ent;
  const bool ok = rvalid && isfinite(li);
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8) {
    if (c8 < nch) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 8 * c8 + i;
        const float l = z[j];
        const float p = __expf(l);
        const float g = pol * ((j == act ? 1.f : 0.f) - p) + a.entropy_coef * p * (l + ent);
        z[j] = (ok && j < A) ? g : 0.f;
        if (j == A) z[j] = ok ? a.value_coef * gv : 0.f;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) z[8 * c8 + i] = 0.f;
    }
  }
  if (!rvalid) return;
  if (!ok) {
    ++nonfinite;
    return;
  }
  st[0] += lpg;
  st[1] += lv;
  st[2] += ent;
  st[3] += fabsf(rho - 1.f) > a.clip_eps ? 1.0 : 0.0;
  st[4] += lp_old - logpi;
}

// NEXT-2 (DESIGN.md §3.6 reading R-S): SplitMix64 finaliser of x + golden gamma; the uniform
// of (seed, key, head) is the top 24 bits of sm64(sm64(seed ^ key) + head), exact in fp32.
__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One row of head outputs (lane = row, column j at zb[j * kZPitch + lane]): per head
// log-softmax, then inverse-CDF sampling with the counter RNG (or argmax), logp and value.
__device__ __forceinline__ void sample_row(const GemmArgs& a, const float* zb, int row) {
  const float* z = zb + lane_id();
  const unsigned long long base = sm64(a.seed ^ (a.keys ? __ldg(a.keys + row) : (unsigned long long)row));
  float lp = 0.f;
  int off = 0;
#pragma unroll 1
  for (int h = 0; h < a.n_heads; ++h) {
    const int sz = a.head_size[h];
    float mx = -INFINITY;
    int am = 0;
    for (int j = 0; j < sz; ++j) {
      const float v = z[(off + j) * kZPitch];
      if (v > mx) { mx = v; am = j; }          // first maximum
    }
    float se = 0.f;
    for (int j = 0; j < sz; ++j) se += __expf(z[(off + j) * kZPitch] - mx);
    const float lse = mx + __logf(se);
    int act = am;
    if (!a.deterministic) {
      const float u = (float)(sm64(base + (unsigned long long)h) >> 40) * (1.f / 16777216.f);
      float cdf = 0.f;
      act = sz - 1;
      for (int j = 0; j < sz; ++j) {
        cdf += __expf(z[(off + j) * kZPitch] - lse);
        if (u < cdf) { act = j; break; }
      }
    }
    lp += z[(off + act) * kZPitch] - lse;
    a.act_out[(int64_t)row * a.n_heads + h] = act;
    off += sz;
  }
  a.logp_out[row] = lp;
  a.value_out[row] = z[a.A * kZPitch];
}

// Per-warp output staging: kOutSlots 32x32 tiles, a tile is reused once the TMA store issued
// kOutSlots tiles ago has read it (the TMA unit also serves the operand loads, so stores can
// queue for a while).
struct OutStage {
  uint8_t* buf;       // kOutSlots x kStageTile, 1024-aligned
  int k;              // tiles issued so far
  __device__ __forceinline__ uint8_t* acquire() {
    uint8_t* t = buf + (k % kOutSlots) * kStageTile;
    if (k >= kOutSlots && lane_id() == 0) bulk_wait_read<kOutSlots - 1>();
    __syncwarp();
    return t;
  }
  __device__ __forceinline__ void release(uint8_t* t, const CUtensorMap* map, int col, int row) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane_id() == 0) {
      tma_store_2d(map, t, col, row);
      bulk_commit();
    }
    ++k;
  }
};

// one staging tile per warp: reused once the previous TMA store has read it
struct OutStage1 {
  uint8_t* buf;
  int k;
  uint64_t policy;   // 0: no L2 hint; else a createpolicy value for the stores
  __device__ __forceinline__ uint8_t* acquire() {
    if (k > 0 && lane_id() == 0) bulk_wait_read<0>();
    __syncwarp();
    return buf;
  }
  __device__ __forceinline__ void release(uint8_t* t, const CUtensorMap* map, int col, int row) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane_id() == 0) {
      if (policy) tma_store_2d_hint(map, t, col, row, policy);
      else tma_store_2d(map, t, col, row);
      bulk_commit();
    }
    ++k;
  }
};

// ---------------------------------------------------------------------------------------
// Grid-wide barrier of a persistent launch (grid <= #SMs, one CTA per SM, all co-resident):
// arrival count + generation word.  bar[0..1], zero-initialised, reusable across launches.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// a5 split-K reduction inside the dW launch (EPI_PART with red_out): every CTA has written its
// partial, so after the barrier the [M][N] gradient is summed over the k_splits partials in
// split order -- deterministic -- while they are still in L2, scaled by 1/N and stored into
// the bucket; the partial lines are then discarded from L2 (never written back to HBM).
// Warp-strided over float4 quads (N % 4 == 0), 8 split loads in flight per lane.
__device__ __forceinline__ void part_fixup(const GemmArgs& a) {
  grid_barrier(a.red_bar);
  const uint32_t lane = lane_id();
  const int S = a.k_splits;
  const int qpr = a.N >> 2;
  const int64_t nq = (int64_t)a.M * qpr;
  const int64_t st4 = a.part_split_stride >> 2;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec_out = (reinterpret_cast<uintptr_t>(a.red_out) & 15) == 0;
  const bool discard = a.red_discard && (qpr & 7) == 0 && (a.ld_part & 31) == 0;
  uint32_t bad = 0;
  for (int64_t qb = gw * 32; qb < nq; qb += nw * 32) {
    const int64_t q = qb + lane;
    const bool valid = q < nq;
    const int r = valid ? (int)(q / qpr) : 0, c = valid ? 4 * (int)(q % qpr) : 0;
    const float4* src = reinterpret_cast<const float4*>(a.part + (int64_t)r * a.ld_part + c);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      for (int k0 = 0; k0 < S; k0 += 8) {
        float4 x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (k0 + j < S) x[j] = __ldcg(src + (int64_t)(k0 + j) * st4);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (k0 + j < S) { acc.x += x[j].x; acc.y += x[j].y; acc.z += x[j].z; acc.w += x[j].w; }
      }
      acc.x *= a.red_scale; acc.y *= a.red_scale; acc.z *= a.red_scale; acc.w *= a.red_scale;
      bad += !isfinite(acc.x) + !isfinite(acc.y) + !isfinite(acc.z) + !isfinite(acc.w);
      float* dst = a.red_out + (int64_t)r * a.N + c;
      if (vec_out) {
        *reinterpret_cast<float4*>(dst) = acc;
      } else {
        dst[0] = acc.x; dst[1] = acc.y; dst[2] = acc.z; dst[3] = acc.w;
      }
    }
    __syncwarp();
    // the 8 lanes of a 128-byte partial line have read it: drop it from L2 unwritten (only when
    // rows hold whole lines, so a line's 8 quads are lanes 8j..8j+7 of this iteration)
    if (discard && valid && (c & 31) == 0)
      for (int k = 0; k < S; ++k)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(src + (int64_t)k * st4) : "memory");
  }
  const uint32_t tot = __reduce_add_sync(0xffffffffu, bad);
  if (lane == 0 && tot && a.counters) atomicAdd(a.counters, (unsigned long long)tot);
}

// ---------------------------------------------------------------------------------------
template <int BN, bool A_MN, bool B_MN, int EPI_KIND, int CG>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmY,
               const GemmArgs args) {
  // EPI_TANH_ACC: the TANH epilogue with the accurate rational tanh (SRL_TANH=accurate)
  constexpr int EPI = EPI_KIND == EPI_TANH_ACC ? EPI_TANH : EPI_KIND;
  constexpr bool ACC_TANH = EPI_KIND == EPI_TANH_ACC;
  // SPLIT: both epilogue warpgroups drain every tile, each half of its 32-column chunks, which
  // halves the per-tile epilogue latency the MMA waits on (only 512/BN accumulators exist).
  // The loss epilogue needs whole rows: its groups take alternate tiles instead.
  constexpr bool ROWEPI = EPI == EPI_LOSS || EPI == EPI_SAMPLE;   // whole head rows per lane
  constexpr bool SPLIT = !ROWEPI && BN >= 64;
  constexpr int NCH_ALL = BN / 32;
  constexpr int NCH = SPLIT ? NCH_ALL / 2 : NCH_ALL;     // chunks per warp per tile
  using Cfg = GemmCfg<BN, CG>;
  static_assert(!ROWEPI || BN == kHeadCols, "loss/sample epilogues work on the 64-col head");
  static_assert(CG == 1 || (BN / CG) % 64 == 0 || !B_MN, "MN-major B halves must be 64-wide");
  static_assert(BN <= 256 || (B_MN && EPI == EPI_PART), "BN = 512 is the dW (MN-major B, partials) tile");
  const int STAGES = args.stages;
  const int zcols = args.A + 1 + args.n_heads;    // row buffer columns (loss / sample only)
  const SmemLayout SL = smem_layout(BN, EPI, STAGES, args.colsum_ld, CG, zcols);
  const int rank = (CG == 2) ? (int)cluster_ctarank() : 0;   // CTA rank in the pair
  const bool leader = rank == 0;
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;      // pair (cluster) index / count
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SL.bars);
  uint64_t* empty = full + 8;
  uint64_t* tfull = empty + 8;
  uint64_t* tempty = tfull + 8;
  uint64_t* ybar = tempty + 8;                    // [8 warps][kYSlots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ybar + kEpiWarps * kYSlots);
  float* colsum_s = reinterpret_cast<float*>(smem + SL.colsum);
  float* bias_s = reinterpret_cast<float*>(smem + SL.bias);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const int units = args.m_tiles * args.n_tiles * args.k_splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < Cfg::ACC_STAGES; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], (SPLIT ? 8 : 4) * CG);   // every epilogue warp on the tile, both CTAs
    }
    for (int s = 0; s < kEpiWarps * kYSlots; ++s) mbar_init(&ybar[s], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_cg<CG>(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();   // peer barriers initialised before remote use
  tc_fence_after();
  // PDL: everything above overlapped the previous kernel's tail; its outputs are read below
  griddep_wait();
  griddep_launch();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      auto load = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
        if constexpr (CG == 1) tma_load_2d(dst, m, bar, c0, c1);
        else tma_load_2d_cg2(dst, m, bar, c0, c1);   // bytes counted on the leader's barrier
      };
      for (int u = cid; u < units; u += ncl) {
        const int nt = u % args.n_tiles;
        const int mt = (u / args.n_tiles) % args.m_tiles;
        const int ks = u / (args.n_tiles * args.m_tiles);
        const int kb0 = ks * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int m0 = mt * 128 * CG + rank * 128;           // this CTA's A rows
        const int n0 = nt * BN + rank * (BN / CG);           // this CTA's B columns
        for (int kb = kb0; kb < kb1; ++kb) {
          wait_bounded(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], Cfg::TX_BYTES);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          const int k0 = kb * 64;
          if (!A_MN) {
            load(sa, &tmA, &full[stage], k0, m0);
          } else {
            load(sa, &tmA, &full[stage], m0, k0);
            load(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          }
          if (!B_MN) {
            load(sb, &tmB, &full[stage], k0, n0);
          } else {
            // box j of this CTA: MMA half h = j / BOXES_PER_HALF; within it this CTA's
            // MMA_N / CG columns (the pair splits every N = 256 MMA's columns)
#pragma unroll
            for (int j = 0; j < BN / CG / 64; ++j) {
              const int h = j / Cfg::BOXES_PER_HALF, jj = j % Cfg::BOXES_PER_HALF;
              load(sb + j * 8192, &tmB, &full[stage],
                   nt * BN + h * Cfg::MMA_N + rank * (Cfg::MMA_N / CG) + 64 * jj, k0);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ============================ MMA issuer (the pair's leader CTA only)
    constexpr uint32_t IDESC = umma_idesc_f16(128 * CG, Cfg::MMA_N, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = cid; u < units; u += ncl, ++it) {
      const int ks = u / (args.n_tiles * args.m_tiles);
      const int kb0 = ks * args.kb_per_split;
      const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
      const int acc = it % Cfg::ACC_STAGES;
      const uint32_t acc_phase = (uint32_t)(it / Cfg::ACC_STAGES) & 1u;
      wait_bounded(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        wait_bounded(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_base = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t b_base = a_base + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a_base + k * 2048, 8192, 1024)
                                     : umma_desc_sw128(a_base + k * 32, 16, 1024);
#pragma unroll
            for (int h = 0; h < Cfg::N_HALVES; ++h) {
              const uint32_t bh = b_base + h * Cfg::BOXES_PER_HALF * 8192;
              const uint64_t bd = B_MN ? umma_desc_sw128(bh + k * 2048, 8192, 1024)
                                       : umma_desc_sw128(bh + k * 32, 16, 1024);
              tc_mma_f16_cg<CG>(d_tmem + h * Cfg::MMA_N, ad, bd, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          tc_commit_cg<CG>(&empty[stage]);      // frees the slot in both CTAs
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit_cg<CG>(&tfull[acc]);   // both CTAs' epilogues
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ============================ epilogue (two warpgroups, alternate tiles)
    const int ew = warp - 4;                 // 0..7
    const int grp = ew >> 2;                 // warpgroup
    const int quad = warp & 3;               // TMEM lane quadrant = 32-row slice of the tile
    float* my_colsum = colsum_s + ew * args.colsum_ld;
    OutStage ost{smem + SL.ostage + ew * kOutSlots * kStageTile, 0};
    uint8_t* ystage = smem + SL.ystage + ew * kYSlots * kStageTile;
    uint64_t* my_ybar = ybar + kYSlots * ew;
    uint32_t yph = 0;                        // phase bit per y slot
    int yslot = 0;                           // next slot to fill (ring over tiles)
    if (EPI == EPI_DTANH || EPI == EPI_LOSS) {
      for (int i = lane; i < args.colsum_ld; i += 32) my_colsum[i] = 0.f;
      __syncwarp();
    }
    if (EPI == EPI_TANH || ROWEPI) {
      const int nb = ROWEPI ? args.A + 1 : args.N;
      for (int i = ew * 32 + lane; i < 1024; i += 256) bias_s[i] = i < nb ? __ldg(args.bias + i) : 0.f;
      named_bar_sync(1, 256);
    }
    uint32_t nsat = 0, nonfinite = 0;
    double st[5] = {0, 0, 0, 0, 0};
    int it = 0;
    for (int u = cid; u < units; u += ncl, ++it) {
      if (!SPLIT && (it & 1) != grp) continue;
      const int acc = it % Cfg::ACC_STAGES;
      const uint32_t acc_phase = (uint32_t)(it / Cfg::ACC_STAGES) & 1u;
      const int nt = u % args.n_tiles;
      const int mt = (u / args.n_tiles) % args.m_tiles;
      const int ks = u / (args.n_tiles * args.m_tiles);
      const int row0 = mt * 128 * CG + rank * 128 + quad * 32;   // first row of this warp's slice
      const int row = row0 + (int)lane;
      const int n0 = nt * BN + (SPLIT ? grp * NCH * 32 : 0);   // this warp's first column
      const bool rvalid = row < args.M;
      int ybase = 0;
      if constexpr (EPI == EPI_DTANH) {
        // the first kYSlots-1 y_prev chunks of this tile, before waiting for the accumulator
        // (TMA; rows past M read as zero).  Slots were released by __syncwarp after their reads.
        ybase = yslot;
        if (lane == 0) {
          fence_proxy_async_smem();
#pragma unroll
          for (int c = 0; c < kYSlots - 1; ++c) {
            if (c < NCH) {
              const int sl = (ybase + c) % kYSlots;
              mbar_expect_tx(&my_ybar[sl], kStageTile);
              tma_load_2d(ystage + sl * kStageTile, &tmY, &my_ybar[sl], n0 + c * 32, row0);
            }
          }
        }
        yslot = (ybase + NCH) % kYSlots;
      }
      wait_bounded(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN +
                             (SPLIT ? grp * NCH * 32 : 0);

      if constexpr (EPI == EPI_TANH) {
        auto body = [&](int c, float (&v)[32]) {
          const int col0 = n0 + c * 32;
          const float4* b4 = reinterpret_cast<const float4*>(bias_s + col0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 bb = b4[q];
            if constexpr (ACC_TANH) {
              v[4 * q + 0] = tanh_fast_accurate(v[4 * q + 0] + bb.x);
              v[4 * q + 1] = tanh_fast_accurate(v[4 * q + 1] + bb.y);
              v[4 * q + 2] = tanh_fast_accurate(v[4 * q + 2] + bb.z);
              v[4 * q + 3] = tanh_fast_accurate(v[4 * q + 3] + bb.w);
            } else {
              v[4 * q + 0] = tanh_mufu(v[4 * q + 0] + bb.x);
              v[4 * q + 1] = tanh_mufu(v[4 * q + 1] + bb.y);
              v[4 * q + 2] = tanh_mufu(v[4 * q + 2] + bb.z);
              v[4 * q + 3] = tanh_mufu(v[4 * q + 3] + bb.w);
            }
          }
          uint8_t* t = ost.acquire();
          stile_write_row(t, (int)lane, v);
          ost.release(t, &tmO, col0, row0);      // rows >= M are clipped by TMA
        };
        // ping-pong register buffers (compile-time after unrolling): the next chunk's TMEM
        // read is in flight while this one is computed, without a register copy
        float b0[32], b1[32];
        tmem_ld32(taddr, b0);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          tc_wait_ld();
          if (c & 1) {
            if (c + 1 < NCH) tmem_ld32(taddr + (c + 1) * 32, b0);
            body(c, b1);
          } else {
            if (c + 1 < NCH) tmem_ld32(taddr + (c + 1) * 32, b1);
            body(c, b0);
          }
        }
      } else if constexpr (EPI == EPI_DTANH) {
        // dY chunks as 16x256b TMEM fragments (v[16 hf + 4k + 2h + e] = row 16hf + 8h + lane/4,
        // col 8k + 2(lane%4) + e of the warp's 32x32 block): packed fp32x2 math, and the db
        // column sums need 4 in-thread rows + a 3-level butterfly instead of a 32x32 transpose
        // (the head_fused.cu dtanh epilogue).  v := dY .* (Y^2 - 1) = -dZ; the
        // stores negate the fp16 pairs and the per-CTA sums are negated when written.
        uint32_t s_off[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) s_off[k] = stile_off((int)(lane >> 2), k) + 4 * (lane & 3);
        const int cs_col = 8 * (2 * (int)((lane >> 4) & 1) + (int)((lane >> 3) & 1)) +
                           2 * (int)(lane & 3) + (int)((lane >> 2) & 1);
        auto body = [&](int c, float (&v)[32]) {
          const int yb = (ybase + c) % kYSlots;
          if (c + kYSlots - 1 < NCH && lane == 0) {   // keep kYSlots-1 chunks in flight
            const int sl = (ybase + c + kYSlots - 1) % kYSlots;
            fence_proxy_async_smem();
            mbar_expect_tx(&my_ybar[sl], kStageTile);
            tma_load_2d(ystage + sl * kStageTile, &tmY, &my_ybar[sl], n0 + (c + kYSlots - 1) * 32, row0);
          }
          const int col0 = n0 + c * 32;
          wait_bounded(&my_ybar[yb], (yph >> yb) & 1u);
          yph ^= 1u << yb;
          const uint32_t ys = smem_u32(ystage + yb * kStageTile);
          float mx = 0.f;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int k = 0; k < 4; ++k) {       // rows >= M: acc = 0, y = 0 -> 0
                const uint32_t u = lds32(ys + s_off[k] + (uint32_t)(16 * hf + 8 * h) * 64);
                const float2 y = __half22float2(*reinterpret_cast<const __half2*>(&u));
                float& a0 = v[16 * hf + 4 * k + 2 * h];
                float& a1 = v[16 * hf + 4 * k + 2 * h + 1];
                mul_sqm1_x2(a0, a1, y.x, y.y);
                mx = fmaxf(mx, fmaxf(fabsf(a0), fabsf(a1)));
              }
          __syncwarp();                            // the y slot may be refilled
          if (mx > 65504.f) {                    // rare: clamp to the fp16 range and count
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = sat_f16(v[j], nsat);
          }
          uint8_t* t = ost.acquire();
          const uint32_t ts = smem_u32(t);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int i = 16 * hf + 4 * k + 2 * h;
                sts32(ts + s_off[k] + (uint32_t)(16 * hf + 8 * h) * 64,
                      pack_half2(v[i], v[i + 1]) ^ 0x80008000u);
              }
          ost.release(t, &tmO, col0, row0);
          // db column sums of the fp32 values (summing the fp16-rounded tile on the tensor
          // core was measured too imprecise for some bias tensors, and slower)
          float c8[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float x0 = v[4 * k], x1 = v[4 * k + 1], z0 = v[16 + 4 * k], z1 = v[16 + 4 * k + 1];
            add_x2(x0, x1, v[4 * k + 2], v[4 * k + 3]);
            add_x2(z0, z1, v[16 + 4 * k + 2], v[16 + 4 * k + 3]);
            add_x2(x0, x1, z0, z1);
            c8[2 * k] = x0;
            c8[2 * k + 1] = x1;
          }
#pragma unroll
          for (int w = 4; w >= 1; w >>= 1) {
            const bool up = (lane & (4u * w)) != 0;
#pragma unroll
            for (int i = 0; i < w; ++i) {
              const float send = up ? c8[i] : c8[i + w];
              const float keep = up ? c8[i + w] : c8[i];
              c8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4 * w);
            }
          }
          my_colsum[col0 + cs_col] += c8[0];
        };
        auto ld16 = [&](uint32_t ta, float* v) {
          tmem_ld16x256_x4(ta, v);
          tmem_ld16x256_x4(ta + (16u << 16), v + 16);
        };
        float b0[32], b1[32];
        ld16(taddr, b0);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          tc_wait_ld();
          if (c & 1) {
            if (c + 1 < NCH) ld16(taddr + (c + 1) * 32, b0);
            body(c, b1);
          } else {
            if (c + 1 < NCH) ld16(taddr + (c + 1) * 32, b1);
            body(c, b0);
          }
        }
      } else if constexpr (EPI == EPI_PART) {
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          tc_wait_ld();
          if (rvalid) {
            float4* dst = reinterpret_cast<float4*>(args.part + (int64_t)ks * args.part_split_stride +
                                                    (int64_t)row * args.ld_part + n0 + c * 32);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      } else if constexpr (EPI == EPI_SAMPLE) {
        float* zb = reinterpret_cast<float*>(smem + SL.zbuf) + ew * zcols * kZPitch;
        float z[64];
        tmem_ld32(taddr, z);
        tmem_ld32(taddr + 32, z + 32);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (j <= args.A) zb[j * kZPitch + lane] = z[j] + bias_s[j];
        if (rvalid) sample_row(args, zb, row);   // each lane reads only its own zb column
        __syncwarp();
      } else {  // EPI_LOSS
        const int32_t* arow = nullptr;
        float Ahat = 0.f, lp = 0.f, R = 0.f, vo = 0.f;
        // padding rows (valid == 0) take no part: zero dlogits, no statistics
        const bool lvalid = rvalid && (!args.valid || __ldg(args.valid + row) != 0);
        if (lvalid) {   // per-row inputs: coalesced across lanes, issued before the TMEM wait
          arow = args.actions + (int64_t)row * args.n_heads;
          Ahat = __ldg(args.adv + row);
          lp = __ldg(args.logp_old + row);
          R = __ldg(args.ret + row);
          if (args.v_old) vo = __ldg(args.v_old + row);
        }
        float* zb = reinterpret_cast<float*>(smem + SL.zbuf) + ew * zcols * kZPitch;
        {
          float z[64];
          tmem_ld32(taddr, z);
          tmem_ld32(taddr + 32, z + 32);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j <= args.A) zb[j * kZPitch + lane] = z[j] + bias_s[j];
        }
        if (args.mean_std) {
          const double mu = args.mean_std[0], sd = args.mean_std[1];
          Ahat = (float)(((double)Ahat - mu) / (sd + (double)args.adv_eps));
        }
        ppo_rows_smem(args, zb, arow, Ahat, lp, R, vo, lvalid, st, nonfinite);
        __syncwarp();
        // per-CTA bias-gradient partials: lane j sums column j over the warp's 32 rows
        for (int j = lane; j <= args.A; j += 32) {
          float cs = 0.f;
#pragma unroll 8
          for (int r = 0; r < 32; ++r) cs += zb[j * kZPitch + r];
          my_colsum[j] += cs;
        }
        // this row's 64 fp16 outputs (zero pad past A), saturated, through TMA stores
        float z0[32], z1[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          z0[j] = (j <= args.A) ? sat_f16(zb[j * kZPitch + lane], nsat) : 0.f;
          z1[j] = (j + 32 <= args.A) ? sat_f16(zb[(j + 32) * kZPitch + lane], nsat) : 0.f;
        }
        __syncwarp();
        uint8_t* t0 = ost.acquire();
        stile_write_row(t0, (int)lane, z0);
        ost.release(t0, &tmO, 0, row0);
        uint8_t* t1 = ost.acquire();
        stile_write_row(t1, (int)lane, z1);
        ost.release(t1, &tmO, 32, row0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
        else mbar_arrive_leader(&tempty[acc]);   // the leader's MMA waits on it
      }
    }
    if (EPI != EPI_PART && lane == 0) bulk_wait<0>();   // all TMA stores of this warp done
    __syncwarp();
    // ---- per-CTA partials (deterministic: fixed unit set per CTA, fixed reduction order)
    if (args.counters) {
      count_warp(args.counters + 1, nsat);
      count_warp(args.counters + 0, nonfinite);
    }
    if constexpr (EPI == EPI_LOSS) {
      __shared__ double red[8][5];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        double x = st[k];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[ew][k] = x;
      }
      named_bar_sync(1, 256);
      if (ew == 0 && lane < 5) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += red[w][lane];
        args.stats[(int64_t)blockIdx.x * 8 + lane] = x;
      }
    }
    if (EPI == EPI_DTANH || EPI == EPI_LOSS) {
      named_bar_sync(1, 256);
      float* dst = args.colsum + (int64_t)blockIdx.x * args.colsum_ld;
      for (int i = ew * 32 + lane; i < args.colsum_ld; i += 256) {
        float x = 0.f;
        for (int w = 0; w < 8; ++w) x += colsum_s[w * args.colsum_ld + i];
        dst[i] = EPI == EPI_DTANH ? -x : x;    // DTANH summed -dZ
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();   // no CTA leaves while its peer may still signal it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg<CG>(tmem_base, Cfg::TMEM_COLS);
  }
  if constexpr (EPI == EPI_PART) {
    if (args.red_out) part_fixup(args);   // a5: the split-K sum, in this launch
  }
}

}  // namespace srl
