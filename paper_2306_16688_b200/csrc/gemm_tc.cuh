// gemm_tc.cuh -- warp-specialised TMA + tcgen05 GEMM for sm_100a with the trainer's fused
// epilogues.  D[M][N] = sum_k A(m,k) * B(n,k), fp16 operands, fp32 accumulation in TMEM.
//
//   A(m,k): K-major = row-major [M][K] (A_MN=false)  |  MN-major = row-major [K][M] (A_MN=true)
//   B(n,k): K-major = row-major [N][K] (B_MN=false)  |  MN-major = row-major [K][N] (B_MN=true)
//
// Tile 128 x BN x 64, SWIZZLE_128B smem operands fed by TMA through an mbarrier ring,
// one elected thread issues tcgen05.mma (kind::f16, M=128), two TMEM accumulators so the
// epilogue of tile i overlaps the MMAs of tile i+1.  Persistent CTAs walk the work units
// (m tile, n tile, k split) with a static stride, so every per-CTA partial is deterministic.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w3 idle,
// w4..w11 epilogue in two warpgroups g = 0, 1 that take alternate tiles (group g owns TMEM
// accumulator stage g), so each group has two MMA periods to drain a tile; warp w reads TMEM
// lanes 32(w%4)..32(w%4)+31 = tile rows of that quadrant.
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

enum { EPI_TANH = 0, EPI_DTANH = 1, EPI_PART = 2, EPI_LOSS = 3 };

constexpr int kMaxHeads = 8;
constexpr int kHeadCols = 64;   // padded head width G (logits + value + zero pad)

struct GemmArgs {
  int M, N;                       // valid rows / cols of D
  int m_tiles, n_tiles, k_splits;
  int kb_total, kb_per_split;     // 64-wide k blocks
  // outputs / epilogue inputs
  __half* out; int64_t ld_out;                    // TANH, DTANH, LOSS
  float* part; int64_t ld_part; int64_t part_split_stride;   // PART
  const float* bias;                              // TANH, LOSS
  const __half* y_prev; int64_t ld_y;             // DTANH
  float* colsum; int colsum_ld;                   // DTANH, LOSS: [grid][colsum_ld]
  unsigned long long* counters;                   // [0] nonfinite, [1] fp16 saturations
  // loss (a4)
  const int32_t* actions; const float* logp_old; const float* adv; const float* ret;
  const double* mean_std; double* stats;          // stats: [grid][8]
  int n_heads, A;
  int head_size[kMaxHeads];
  float clip_eps, value_coef, entropy_coef, adv_eps;
};

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;        // 128 / 256 / 512: power of two
  static constexpr int BAR_BYTES = 256;
  static constexpr int EPI_WARPS = 8;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static size_t smem_bytes(int colsum_ld) {
    return 1024 + (size_t)STAGES * STAGE_BYTES + BAR_BYTES + (size_t)EPI_WARPS * colsum_ld * 4;
  }
};

__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t parity) {
  // bounded spin: a lost arrival traps (error surfaced to the host) instead of hanging
  uint32_t it = 0;
  long long t0 = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (((++it) & 1023) == 0) {
      long long now = clock64();
      if (t0 == 0) t0 = now;
      else if (now - t0 > (1ll << 35)) __trap();
    }
  }
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

__device__ __forceinline__ void store32_f16(__half* dst, const float (&v)[32]) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __half2 h0 = __floats2half2_rn(v[8 * q + 0], v[8 * q + 1]);
    __half2 h1 = __floats2half2_rn(v[8 * q + 2], v[8 * q + 3]);
    __half2 h2 = __floats2half2_rn(v[8 * q + 4], v[8 * q + 5]);
    __half2 h3 = __floats2half2_rn(v[8 * q + 6], v[8 * q + 7]);
    uint4 u;
    u.x = *reinterpret_cast<uint32_t*>(&h0);
    u.y = *reinterpret_cast<uint32_t*>(&h1);
    u.z = *reinterpret_cast<uint32_t*>(&h2);
    u.w = *reinterpret_cast<uint32_t*>(&h3);
    d4[q] = u;
  }
}

__device__ __forceinline__ void load32_f16(const __half* src, float (&y)[32]) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = __ldg(s4 + q);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __half22float2(h[e]);
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
// a4: PPO loss on one row held in registers (z: 64 logits incl. bias; g out: dloss_i/dz).
// Formulas: DESIGN.md §3.1 (SURVEY C-4).
__device__ __forceinline__ void ppo_row(const GemmArgs& a, float (&z)[64], const int* act,
                                        float Ahat, float lp_old, float R, double (&st)[5],
                                        uint32_t& nonfinite) {
  float logpi = 0.f, ent = 0.f;
  float Hh[kMaxHeads];
  int off = 0;
  for (int h = 0; h < a.n_heads; ++h) {
    const int sz = a.head_size[h];
    const int ah = off + act[h];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (j >= off && j < off + sz) mx = fmaxf(mx, z[j]);
    float se = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (j >= off && j < off + sz) se += __expf(z[j] - mx);
    const float lse = mx + __logf(se);
    float hh = 0.f, la = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      if (j >= off && j < off + sz) {
        const float l = z[j] - lse;        // log-softmax, kept in z
        z[j] = l;
        hh -= __expf(l) * l;
        if (j == ah) la = l;
      }
    }
    Hh[h] = hh;
    ent += hh;
    logpi += la;
    off += sz;
  }
  const float rho = expf(logpi - lp_old);
  const float lo = 1.f - a.clip_eps, hi = 1.f + a.clip_eps;
  const float rc = fminf(fmaxf(rho, lo), hi);
  const float lpg = -fminf(rho * Ahat, rc * Ahat);
  float V = 0.f;
#pragma unroll
  for (int j = 0; j < 64; ++j)
    if (j == a.A) V = z[j];   // unrolled select keeps z in registers
  const float dv = V - R;
  const float lv = dv * dv;
  const float mask = (Ahat >= 0.f) ? (rho <= hi ? 1.f : 0.f) : (rho >= lo ? 1.f : 0.f);
  const float pol = -mask * Ahat * rho;   // coefficient of (onehot - p)
  const float li = lpg + a.value_coef * lv - a.entropy_coef * ent;
  const bool ok = isfinite(li);
  off = 0;
  for (int h = 0; h < a.n_heads; ++h) {
    const int sz = a.head_size[h];
    const int ah = off + act[h];
    const float H = Hh[h];
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      if (j >= off && j < off + sz) {
        const float l = z[j];
        const float p = __expf(l);
        z[j] = pol * ((j == ah ? 1.f : 0.f) - p) + a.entropy_coef * p * (l + H);
      }
    }
    off += sz;
  }
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    if (j == a.A) z[j] = 2.f * a.value_coef * dv;
    else if (j > a.A || !ok) z[j] = 0.f;
  }
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

// ---------------------------------------------------------------------------------------
template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(GemmCfg<BN>::THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  static_assert(EPI != EPI_LOSS || BN == kHeadCols, "loss epilogue works on the 64-col head");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* colsum_s = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::BAR_BYTES);

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
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int nt = u % args.n_tiles;
        const int mt = (u / args.n_tiles) % args.m_tiles;
        const int ks = u / (args.n_tiles * args.m_tiles);
        const int kb0 = ks * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int m0 = mt * 128, n0 = nt * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          wait_bounded(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          const int k0 = kb * 64;
          if (!A_MN) {
            tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          } else {
            tma_load_2d(sa, &tmA, &full[stage], m0, k0);
            tma_load_2d(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    constexpr uint32_t IDESC = umma_idesc_f16(128, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int ks = u / (args.n_tiles * args.m_tiles);
      const int kb0 = ks * args.kb_per_split;
      const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
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
            const uint64_t bd = B_MN ? umma_desc_sw128(b_base + k * 2048, 8192, 1024)
                                     : umma_desc_sw128(b_base + k * 32, 16, 1024);
            tc_mma_f16(d_tmem, ad, bd, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ============================ epilogue (two warpgroups, alternate tiles)
    const int ew = warp - 4;                 // 0..7
    const int grp = ew >> 2;                 // warpgroup = TMEM accumulator stage it drains
    const int quad = warp & 3;               // TMEM lane quadrant
    const int trow = quad * 32 + (int)lane;
    float* my_colsum = colsum_s + ew * args.colsum_ld;
    if (EPI == EPI_DTANH || EPI == EPI_LOSS) {
      for (int i = lane; i < args.colsum_ld; i += 32) my_colsum[i] = 0.f;
      __syncwarp();
    }
    uint32_t nsat = 0, nonfinite = 0;
    double st[5] = {0, 0, 0, 0, 0};
    uint32_t acc_phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
      if ((it & 1) != grp) continue;
      const int nt = u % args.n_tiles;
      const int mt = (u / args.n_tiles) % args.m_tiles;
      const int ks = u / (args.n_tiles * args.m_tiles);
      const int row = mt * 128 + trow;
      const int n0 = nt * BN;
      const bool rvalid = row < args.M;
      wait_bounded(&tfull[grp], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + grp * BN;

      if constexpr (EPI == EPI_TANH) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          tc_wait_ld();
          const int col0 = n0 + c * 32;
          if (rvalid) {
            const float4* b4 = reinterpret_cast<const float4*>(args.bias + col0);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 bb = __ldg(b4 + q);
              v[4 * q + 0] = tanh_fast_accurate(v[4 * q + 0] + bb.x);
              v[4 * q + 1] = tanh_fast_accurate(v[4 * q + 1] + bb.y);
              v[4 * q + 2] = tanh_fast_accurate(v[4 * q + 2] + bb.z);
              v[4 * q + 3] = tanh_fast_accurate(v[4 * q + 3] + bb.w);
            }
            store32_f16(args.out + (int64_t)row * args.ld_out + col0, v);
          }
        }
      } else if constexpr (EPI == EPI_DTANH) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          tc_wait_ld();
          const int col0 = n0 + c * 32;
          if (rvalid) {
            float y[32];
            load32_f16(args.y_prev + (int64_t)row * args.ld_y + col0, y);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = sat_f16(v[j] * (1.f - y[j] * y[j]), nsat);
            store32_f16(args.out + (int64_t)row * args.ld_out + col0, v);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          const float s = transpose_reduce32(v);
          my_colsum[col0 + lane] += s;
        }
      } else if constexpr (EPI == EPI_PART) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
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
      } else {  // EPI_LOSS
        float z[64];
        tmem_ld32(taddr, z);
        tmem_ld32(taddr + 32, z + 32);
        tc_wait_ld();
        if (rvalid) {
#pragma unroll
          for (int j = 0; j < 64; ++j) z[j] += (j <= args.A) ? __ldg(args.bias + j) : 0.f;
          int act[kMaxHeads];
          for (int h = 0; h < args.n_heads; ++h) act[h] = __ldg(args.actions + (int64_t)row * args.n_heads + h);
          float Ahat = __ldg(args.adv + row);
          if (args.mean_std) {
            const double mu = args.mean_std[0], sd = args.mean_std[1];
            Ahat = (float)(((double)Ahat - mu) / (sd + (double)args.adv_eps));
          }
          ppo_row(args, z, act, Ahat, __ldg(args.logp_old + row), __ldg(args.ret + row), st,
                  nonfinite);
#pragma unroll
          for (int j = 0; j < 64; ++j) z[j] = sat_f16(z[j], nsat);
          store32_f16(args.out + (int64_t)row * args.ld_out, *reinterpret_cast<float(*)[32]>(z));
          store32_f16(args.out + (int64_t)row * args.ld_out + 32, *reinterpret_cast<float(*)[32]>(z + 32));
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j) z[j] = 0.f;
        }
        const float s0 = transpose_reduce32(*reinterpret_cast<float(*)[32]>(z));
        my_colsum[lane] += s0;
        const float s1 = transpose_reduce32(*reinterpret_cast<float(*)[32]>(z + 32));
        my_colsum[32 + lane] += s1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[grp]);
      acc_phase ^= 1;
    }
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
        dst[i] = x;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace srl
