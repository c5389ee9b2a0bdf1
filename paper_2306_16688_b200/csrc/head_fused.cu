// head_fused.cu -- rows a4 + a5(head) of the trainer step in ONE persistent tcgen05 kernel.
//
// For every 128-row tile of the last hidden activation Y_L [n][hL] (fp16):
//   a4  z = Y_L W_h^T + b_h (64 padded head columns), the PPO loss and the per-sample logit
//       gradient g, g kept in shared memory as fp16;
//   a5  dZ_L = (g W_h) .* (1 - Y_L^2)  -> HBM (fp16) with per-CTA column sums (db_L);
//       dW_h^T += Y_L^T g accumulated in TMEM over all of the CTA's tiles, flushed once.
// This replaces three launches (head GEMM + loss, dX of the head, split-K dW of the head)
// that streamed Y_L three times and round-tripped g through HBM (VERDICT r1 "fuse the head").
// HBM traffic: Y_L read once (the second pass over a tile, seconds microseconds later, hits
// L2), dZ_L written once.
//
// Per tile, two passes over the tile's hL/64 column blocks of Y_L, each through its own TMA
// ring (pass A: 3 slots, loaded by warp 0; pass B: 4 slots, loaded by warp 3), so pass A and the
// loss of tile j+1 run while the dtanh epilogue of tile j is still consuming pass B:
//   pass A: MMA1  logits[128][32]  += Y_kb . W_h[:, kb]^T          (A K-major, B K-major)
//   pass B: MMA2  dY_kb[128][64]    = g[:, 0:32] . W_h[0:32, kb]   (A K-major, B MN-major)
//           MMA3  dW^T[pair c]     += Y_{2c,2c+1}^T . g              (A MN-major over the two
//                                     ring slots of the pair, B MN-major)
// The head has A + 1 <= 32 real rows (the host checks), so W_h lives in smem as 32-row boxes.
// One smem copy of W_h ([32 head rows][hL], 64-column boxes) serves as the K-major B of
// MMA1 and the MN-major B of MMA2; the g tile serves as the K-major A of MMA2 and the
// MN-major B of MMA3; a Y ring slot serves as the K-major A of MMA1 and the MN-major A of MMA3.
//
// TMEM (512 columns): [0, hL/2) dW^T (hL/128 chunks of 64), [256, 320) two 32-column logits
// buffers (MMA1 of tile j+1 runs while the loss warps still read tile j's), [320, 512) three
// 64-column dY buffers.
//
// Warp roles (512 threads): w0 TMA producer (pass A), w1 MMA issuer of pass A, w2 TMEM
// allocator + MMA issuer of pass B, w3 TMA producer (pass B),
// w4..w7 loss epilogue (row quadrant w % 4), w8..w15 dtanh epilogue (two warpgroups: 32-column
// halves of each 64-column dY block, row quadrant w % 4).
#include <atomic>

#include "internal.h"

namespace srl {

#ifdef SRL_HF_TRACE
// tools/hf_trace.py: per-CTA cycle counters of the waits of each role (variant builds only)
__device__ unsigned long long g_hf_trace[256 * 16];
#define HF_WAIT(bar, par, k)                                   \
  do {                                                         \
    const long long _t0 = clock64();                           \
    wait_bounded(bar, par);                                    \
    trc[k] += (unsigned long long)(clock64() - _t0);           \
  } while (0)
#else
#define HF_WAIT(bar, par, k) wait_bounded(bar, par)
#endif

#if defined(SRL_HF_EXP_NOB) || defined(SRL_HF_EXP_NOA)
// timing experiment: complete the expected transaction bytes of a ring slot without a load
__device__ __forceinline__ void mbar_arrive_expect_noop(uint64_t* bar) {
  asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(16384) : "memory");
}
#endif

// build flag for A/B: -DSRL_HF_STORE_HINT=1 adds an evict-first hint to the dZ stores (measured
// neutral: 225 -> 215 MB of DRAM reads, same duration)
#ifndef SRL_HF_STORE_HINT
#define SRL_HF_STORE_HINT 0
#endif
__device__ __forceinline__ bool hf_store_hint() { return SRL_HF_STORE_HINT != 0; }

namespace hf {
// pass-A ring depth RA (template, 3..5): the deepest that fits next to everything else.
// Pass A streams Y_L from HBM and its TMA loads see ~3 us latency under the kernel's own
// load, so the bytes in flight per SM (RA x 16 KB) bound the tile rate (Little's law).
constexpr int kRingB = 4;                     // pass-B ring (even: an MMA3 pair is adjacent)
constexpr int kSlot = 128 * 64 * 2;           // one [128 rows][64 cols] fp16 block, 16 KB
constexpr int kWRows = 32;                    // head rows kept (A + 1 <= 32)
constexpr int kWBox = kWRows * 64 * 2;        // one [32 head rows][64 cols] W_h box, 4 KB
constexpr int kGBytes = 128 * 64 * 2;         // g tile [128][64] fp16
constexpr int kDy = 3;                        // dY buffers
constexpr int kThreads = 512;
constexpr int kLossWarps = 4, kDtWarps = 8;
constexpr uint32_t kColLogits = 256, kColDy = 320;

struct Layout {
  uint32_t ring, w, g, ostage, zbuf, cs_y, cs_h, bias, bars, total;
};
// zcols = 0: one categorical head, the loss runs in registers (no row buffer)
__host__ __device__ inline Layout layout(int hL, int zcols, int ra) {
  Layout L;
  L.ring = 0;                                     // [ra slots][kRingB slots]
  L.w = L.ring + (ra + kRingB) * kSlot;
  L.g = L.w + (hL / 64) * kWBox;
  L.ostage = L.g + 2 * kGBytes;
  L.zbuf = L.ostage + kDtWarps * kStageTile;
  L.cs_y = L.zbuf + kLossWarps * zcols * kZPitch * 4;
  L.cs_h = L.cs_y + kDtWarps * (hL / 2) * 4;       // per dtanh warp: its hL / 2 columns
  L.bias = L.cs_h + kLossWarps * 64 * 4;
  L.bars = L.bias + 64 * 4;
  L.total = L.bars + 512;
  return L;
}
// ring positions: pass A of tile j, block kb is position j*KB + kb of ring A; pass B likewise
// of ring B (KB even and kRingB even: the two blocks of an MMA3 pair sit in adjacent slots)
}  // namespace hf

static size_t smem_of(int hL, int zcols, int n_heads, int ra) {
  return 1024 + hf::layout(hL, n_heads == 1 ? 0 : zcols, ra).total;
}
size_t head_fused_smem(int hL, int zcols, int n_heads) { return smem_of(hL, zcols, n_heads, 3); }

template <int KB, int kRingA>
__global__ void __launch_bounds__(hf::kThreads, 1)
head_fused_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmO, const GemmArgs args,
                  float* __restrict__ colsum_y) {
  using namespace hf;
  constexpr int hL = KB * 64, NP = KB / 2;
  const int zcols = args.A + 1 + args.n_heads;
  const Layout SL = layout(hL, args.n_heads == 1 ? 0 : zcols, kRingA);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + SL.bars);
  uint64_t* emptyA = fullA + kRingA;
  uint64_t* fullB = emptyA + kRingA;
  uint64_t* emptyB = fullB + kRingB;
  uint64_t* dfull = emptyB + kRingB;
  uint64_t* dempty = dfull + kDy;
  uint64_t* m3done = dempty + kDy;            // [2]
  uint64_t* gfull = m3done + 2;               // [2] per g buffer
  uint64_t* gempty = gfull + 2;               // [2]
  uint64_t* wfull = gempty + 2;
  uint64_t* lfull = wfull + 1;                // [2] per logits buffer
  uint64_t* lempty = lfull + 2;               // [2]
  uint64_t* dwdone = lempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dwdone + 1);
  float* bias_s = reinterpret_cast<float*>(smem + SL.bias);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const int cid = blockIdx.x, ncl = gridDim.x;
  const int m = cid < args.m_tiles ? (args.m_tiles - 1 - cid) / ncl + 1 : 0;   // my tiles
  auto tile = [&](int j) { return cid + j * ncl; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmY);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < kRingA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < kRingB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    for (int b = 0; b < kDy; ++b) {
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], kDtWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&m3done[b], 1);
      mbar_init(&gfull[b], kLossWarps);
      mbar_init(&gempty[b], 1);
    }
    mbar_init(wfull, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&lfull[b], 1);
      mbar_init(&lempty[b], kLossWarps);
    }
    mbar_init(dwdone, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_cg<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();                    // Y_L and the parameters come from earlier kernels
  griddep_launch();
  const uint32_t tmem_base = *tmem_slot;
#ifdef SRL_HF_TRACE
  unsigned long long trc[16] = {};
  const long long t_start = clock64();
#endif

  if (warp == 0 || warp == 3) {
    // ============================ TMA producers: warp 0 W_h once + pass A, warp 3 pass B
    if (elect_one()) {
      const bool pa = warp == 0;
      if (pa) {
        mbar_expect_tx(wfull, KB * kWBox);
        for (int kb = 0; kb < KB; ++kb) tma_load_2d(smem + SL.w + kb * kWBox, &tmW, wfull, kb * 64, 0);
      }
      const int R = pa ? kRingA : kRingB;
      uint64_t* full = pa ? fullA : fullB;
      uint64_t* empty = pa ? emptyA : emptyB;
      uint8_t* ring = smem + SL.ring + (pa ? 0 : kRingA * kSlot);
      uint32_t w = 0;
      const uint64_t pol = pa ? l2_policy_evict_last() : l2_policy_evict_first();
      for (int j = 0; j < m; ++j)
        for (int kb = 0; kb < KB; ++kb, ++w) {
          const int s = w % R;
          HF_WAIT(&empty[s], ((w / R) & 1u) ^ 1u, pa ? 1 : 2);
          mbar_expect_tx(&full[s], kSlot);
#ifdef SRL_HF_EXP_NOB
          if (!pa) { mbar_arrive_expect_noop(&full[s]); continue; }   // timing experiment only
#endif
#ifdef SRL_HF_EXP_NOA
          if (pa) { mbar_arrive_expect_noop(&full[s]); continue; }    // timing experiment only
#endif
          // pass A marks the tile evict-last so pass B (one tile period later) hits L2; pass
          // B's read is the last use: evict-first
          tma_load_2d_hint(ring + s * kSlot, &tmY, &full[s], kb * 64, tile(j) * 128, pol);
        }
    }
  } else if (warp == 1 || warp == 2) {
    // ============================ MMA issuers: warp 1 pass A (MMA1), warp 2 pass B (MMA2 +
    // MMA3).  A tcgen05.mma costs its issuing warp ~100 cycles (operand moves to uniform
    // registers, elect), far more than the tensor core needs for these N = 32 / 64 shapes, so
    // one issuer for both passes was the kernel's critical path; each warp commits (and so
    // tracks) only its own MMAs, and the two touch disjoint TMEM columns.
    constexpr uint32_t ID1 = umma_idesc_f16(128, kWRows, false, false);
    constexpr uint32_t ID2 = umma_idesc_f16(128, 64, false, true);
    constexpr uint32_t ID3 = umma_idesc_f16(128, 64, true, true);
    const uint32_t ringA = smem_u32(smem + SL.ring), ringB = ringA + kRingA * kSlot;
    const uint32_t w0 = smem_u32(smem + SL.w);
    const uint32_t g00 = smem_u32(smem + SL.g);
    wait_bounded(wfull, 0);
    if (warp == 1) {
      // ---- pass A of tile j: logits into buffer j % 2 (free once tile j-2's were read)
      for (int j = 0; j < m; ++j) {
        HF_WAIT(&lempty[j & 1], ((j >> 1) & 1) ^ 1, 4);
        for (int kb = 0; kb < KB; ++kb) {
          const uint32_t w = (uint32_t)(j * KB + kb);
          const int sa = w % kRingA;
          HF_WAIT(&fullA[sa], (w / kRingA) & 1u, 6);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a = ringA + sa * kSlot, b = w0 + kb * kWBox;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16_cg<1>(tmem_base + kColLogits + 32 * (j & 1), umma_desc_sw128(a + k * 32, 16, 1024),
                               umma_desc_sw128(b + k * 32, 16, 1024), ID1, (kb > 0 || k > 0) ? 1u : 0u);
            tc_commit_cg<1>(&emptyA[sa]);
            if (kb == KB - 1) tc_commit_cg<1>(&lfull[j & 1]);
          }
          __syncwarp();
        }
      }
    } else {
      // ---- pass B of tile j: dY blocks and the dW^T pairs (needs its g)
      uint32_t dyc = 0, u3 = 0;
      for (int j = 0; j < m; ++j) {
        const int gb = j & 1;
        const uint32_t g0 = g00 + gb * kGBytes;
        HF_WAIT(&gfull[gb], (j >> 1) & 1, 5);
        for (int c = 0; c < NP; ++c, ++u3) {
          for (int h = 0; h < 2; ++h, ++dyc) {
            const int kb = 2 * c + h, bf = dyc % kDy;
            HF_WAIT(&dempty[bf], ((dyc / kDy) & 1u) ^ 1u, 7);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t wb = w0 + kb * kWBox;
#pragma unroll
              for (int k = 0; k < kWRows / 16; ++k)      // K = the 32 real head columns of g
                tc_mma_f16_cg<1>(tmem_base + kColDy + 64 * bf, umma_desc_sw128(g0 + k * 32, 16, 1024),
                                 umma_desc_sw128(wb + k * 2048, 8192, 1024), ID2, k > 0 ? 1u : 0u);
              tc_commit_cg<1>(&dfull[bf]);
            }
            __syncwarp();
          }
          const uint32_t w = (uint32_t)(j * KB + 2 * c);
          const int sb = w % kRingB;                 // the pair's slots sb, sb + 1 (sb even)
          HF_WAIT(&fullB[sb], (w / kRingB) & 1u, 7);
          HF_WAIT(&fullB[sb + 1], ((w + 1) / kRingB) & 1u, 7);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a = ringB + sb * kSlot;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              tc_mma_f16_cg<1>(tmem_base + 64 * c, umma_desc_sw128(a + k * 2048, kSlot, 1024),
                               umma_desc_sw128(g0 + k * 2048, 8192, 1024), ID3,
                               (j > 0 || k > 0) ? 1u : 0u);
            tc_commit_cg<1>(&m3done[u3 & 1]);
          }
          __syncwarp();
        }
        if (lane == 0) tc_commit_cg<1>(&gempty[gb]);   // g buffer gb free once these complete
        __syncwarp();
      }
      if (lane == 0) tc_commit_cg<1>(dwdone);
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    // ============================ loss epilogue: one row per lane, quadrant warp % 4
    const int lw = warp - 4, quad = warp & 3;
    float* zb = reinterpret_cast<float*>(smem + SL.zbuf) + lw * zcols * kZPitch;
    float* my_cs = reinterpret_cast<float*>(smem + SL.cs_h) + lw * 64;
    for (int i = lane; i < 64; i += 32) my_cs[i] = 0.f;
    for (int i = lw * 32 + lane; i < 64; i += 128) bias_s[i] = i <= args.A ? __ldg(args.bias + i) : 0.f;
    named_bar_sync(3, 128);
    uint32_t nsat = 0, nonfinite = 0;
    double st[5] = {0, 0, 0, 0, 0};
    const bool single = args.n_heads == 1;          // the register path (ppo_row_regs)
    for (int j = 0; j < m; ++j) {
      const int t = tile(j);
      const int r = quad * 32 + (int)lane;          // row in the tile
      const int row = t * 128 + r;
      const bool rvalid = row < args.M;
      const bool lvalid = rvalid && (!args.valid || __ldg(args.valid + row) != 0);
      const int32_t* arow = nullptr;
      float Ahat = 0.f, lp = 0.f, R = 0.f, vo = 0.f;
      if (lvalid) {
        arow = args.actions + (int64_t)row * args.n_heads;
        Ahat = __ldg(args.adv + row);
        lp = __ldg(args.logp_old + row);
        R = __ldg(args.ret + row);
        if (args.v_old) vo = __ldg(args.v_old + row);
      }
      const int act0 = (lvalid && single) ? __ldg(arow) : 0;
      HF_WAIT(&lfull[j & 1], (j >> 1) & 1, j == 0 ? 3 : 8);
      tc_fence_after();
      float z[32];                                   // the A + 1 <= 32 head outputs
      tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + kColLogits + 32 * (j & 1), z);
      tc_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lempty[j & 1]);   // MMA1 of tile j + 2 may overwrite
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) z[jj] += bias_s[jj];   // 0 past A
      if (args.mean_std) {
        const double mu = args.mean_std[0], sd = args.mean_std[1];
        Ahat = (float)(((double)Ahat - mu) / (sd + (double)args.adv_eps));
      }
      const int gb = j & 1;
      uint8_t* gtile = smem + SL.g + gb * kGBytes;
      if (single) {
        // one categorical head: the row stays in registers
        ppo_row_regs(args, z, act0, Ahat, lp, R, vo, lvalid, st, nonfinite);
        HF_WAIT(&gempty[gb], ((j >> 1) & 1) ^ 1, 9);   // tile j-2's MMA2 / MMA3 are done
#pragma unroll
        for (int j8 = 0; j8 < 8; ++j8) {
          uint4 u = make_uint4(0u, 0u, 0u, 0u);
          if (j8 < 4) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = sat_f16(z[8 * j8 + e], nsat);
            u.x = pack_half2(v[0], v[1]);
            u.y = pack_half2(v[2], v[3]);
            u.z = pack_half2(v[4], v[5]);
            u.w = pack_half2(v[6], v[7]);
          }
          *reinterpret_cast<uint4*>(gtile + r * 128 + ((j8 ^ (r & 7)) << 4)) = u;
        }
        fence_proxy_async_smem();                    // generic writes -> tcgen05 (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&gfull[gb]);
        my_cs[lane] += transpose_reduce32(z);        // db_h partials: column lane, 32 rows
        continue;
      }
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        if (jj <= args.A) zb[jj * kZPitch + lane] = z[jj];
      ppo_rows_smem(args, zb, arow, Ahat, lp, R, vo, lvalid, st, nonfinite);
      __syncwarp();
      for (int jj = lane; jj <= args.A; jj += 32) {  // db_h partials: column jj over 32 rows
        float cs = 0.f;
#pragma unroll 8
        for (int q = 0; q < 32; ++q) cs += zb[jj * kZPitch + q];
        my_cs[jj] += cs;
      }
      // g row -> fp16 g buffer j % 2 (128-byte rows, 16-byte chunks swizzled by row % 8)
      HF_WAIT(&gempty[gb], ((j >> 1) & 1) ^ 1, 9);   // tile j-2's MMA2 / MMA3 are done
#pragma unroll
      for (int j8 = 0; j8 < 8; ++j8) {
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int col = 8 * j8 + e;
          v[e] = col <= args.A ? sat_f16(zb[col * kZPitch + lane], nsat) : 0.f;
        }
        uint4 u;
        u.x = pack_half2(v[0], v[1]);
        u.y = pack_half2(v[2], v[3]);
        u.z = pack_half2(v[4], v[5]);
        u.w = pack_half2(v[6], v[7]);
        *reinterpret_cast<uint4*>(gtile + r * 128 + ((j8 ^ (r & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();                      // generic writes -> tcgen05 (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&gfull[gb]);
    }
#ifdef SRL_HF_TRACE
    trc[10] = (unsigned long long)(clock64() - t_start);
#endif
    if (args.counters) {
      count_warp(args.counters + 1, nsat);
      count_warp(args.counters + 0, nonfinite);
    }
    __shared__ double red[kLossWarps][5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      double x = st[k];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) red[lw][k] = x;
    }
    named_bar_sync(3, 128);
    if (lw == 0 && lane < 5) {
      double x = 0.0;
      for (int q = 0; q < kLossWarps; ++q) x += red[q][lane];
      args.stats[(int64_t)blockIdx.x * 8 + lane] = x;
    }
    const float* cs0 = reinterpret_cast<const float*>(smem + SL.cs_h);
    for (int i = lw * 32 + lane; i < 64; i += 128) {
      float x = 0.f;
      for (int q = 0; q < kLossWarps; ++q) x += cs0[q * 64 + i];
      args.colsum[(int64_t)blockIdx.x * args.colsum_ld + i] = x;
    }
  } else if (warp >= 8) {
    // ============================ dtanh epilogue: dZ_L = dY .* (1 - Y^2), db_L column sums
    const int dw = warp - 8, grp = dw >> 2, quad = warp & 3;
    float* my_cs = reinterpret_cast<float*>(smem + SL.cs_y) + dw * (hL / 2);   // col kb*32 + c
    for (int i = lane; i < hL / 2; i += 32) my_cs[i] = 0.f;
    __syncwarp();
    // dZ_L stores evict-first: they must not push pass B's Y blocks out of L2
    OutStage1 ost{smem + SL.ostage + dw * kStageTile, 0, hf_store_hint() ? l2_policy_evict_first() : 0ull};
    uint32_t nsat = 0;
    uint32_t dyc = 0, u3 = 0;
    // per-thread constant offsets of the 16x256b fragment: Y row (quad*32 + 16hf + 8h +
    // lane/4) % 8 == lane/4, so the 128B-swizzled chunk (4 grp + k) ^ (lane/4) is fixed per k;
    // the 64B-swizzled staging tile row 16hf + 8h + lane/4
    const uint32_t ring_b0 = smem_u32(smem + SL.ring) + kRingA * kSlot + (uint32_t)(quad * 32 + (lane >> 2)) * 128;
    // (stile_off(row, k) with row = 16hf + 8h + lane/4: its swizzle (row >> 1) & 3 = (lane >> 3)
    // & 3 for every hf, h, so row (16hf + 8h) only adds an immediate)
    uint32_t y_off[4], s_off[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      y_off[k] = (uint32_t)((((4 * grp + k) ^ (int)(lane >> 2)) << 4) + 4 * (lane & 3));
      s_off[k] = stile_off((int)(lane >> 2), k) + 4 * (lane & 3);
    }
    // the column this lane ends the butterfly with: value index 4 b4 + 2 b3 + b2 = 2k + e
    const int cs_col = 8 * (2 * (int)((lane >> 4) & 1) + (int)((lane >> 3) & 1)) + 2 * (int)(lane & 3) + (int)((lane >> 2) & 1);
    for (int j = 0; j < m; ++j) {
      const int t = tile(j);
      const uint32_t p0 = (uint32_t)(j * KB);
#pragma unroll 1                     // one copy of the body: the unrolled loop (8 copies
                                     // at hL = 512) missed in the instruction cache
      for (int c = 0; c < NP; ++c, ++u3) {
#pragma unroll 1
        for (int h = 0; h < 2; ++h, ++dyc) {
          const int kb = 2 * c + h, b = dyc % kDy;
          const uint32_t wk = p0 + kb;
          HF_WAIT(&dfull[b], (dyc / kDy) & 1u, 11);
          tc_fence_after();
          // dY block [32 rows of the quadrant][32 columns of the half] as 16x256b fragments:
          // v[16 hf + 4k + 2h + e] = (row 16hf + 8h + lane/4, col 8k + 2(lane%4) + e), so the
          // column sums need 4 in-thread rows + a 3-level butterfly instead of a 32x32 transpose
          float v[32];
          const uint32_t tq = tmem_base + ((uint32_t)(quad * 32) << 16) + kColDy + 64 * b + 32 * grp;
          tmem_ld16x256_x4(tq, v);
          tmem_ld16x256_x4(tq + (16u << 16), v + 16);
          tc_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[b]);
          const int s = wk % kRingB;
          HF_WAIT(&fullB[s], (wk / kRingB) & 1u, 12);
          // v := dY .* (Y^2 - 1) = -dZ (negated: the packed fma needs no operand negation; the
          // stores negate the fp16 pairs, the column sums are negated once at the end)
          const uint32_t ybase = ring_b0 + s * kSlot;
          float mx = 0.f;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t yr = ybase + (uint32_t)(16 * hf + 8 * h) * 128;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint32_t u = lds32(yr + y_off[k]);
                const float2 y = __half22float2(*reinterpret_cast<const __half2*>(&u));
                float& a0 = v[16 * hf + 4 * k + 2 * h];
                float& a1 = v[16 * hf + 4 * k + 2 * h + 1];
                mul_sqm1_x2(a0, a1, y.x, y.y);
                mx = fmaxf(mx, fmaxf(fabsf(a0), fabsf(a1)));
              }
            }
          if (mx > 65504.f) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) v[jj] = sat_f16(v[jj], nsat);
          }
#ifdef SRL_HF_TRACE
          const long long ta0 = clock64();
#endif
          uint8_t* tl = ost.acquire();
#ifdef SRL_HF_TRACE
          trc[14] += (unsigned long long)(clock64() - ta0);
#endif
          const uint32_t tls = smem_u32(tl);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int i = 16 * hf + 4 * k + 2 * h;
                sts32(tls + s_off[k] + (uint32_t)(16 * hf + 8 * h) * 64,
                      pack_half2(v[i], v[i + 1]) ^ 0x80008000u);
              }
#ifdef SRL_HF_EXP_NOSTORE
          ++ost.k;                                   // timing experiment only: no dZ store
#else
          ost.release(tl, &tmO, kb * 64 + 32 * grp, t * 128 + quad * 32);
#endif
          // column sums of -dZ: 4 rows in-thread, then lanes differing in bits 4, 3, 2
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
          my_cs[kb * 32 + cs_col] += c8[0];
        }
        // both blocks of the pair read by all 8 dtanh warps: once MMA3 of the pair is done too,
        // the two ring slots go back to the producer
#ifdef SRL_HF_TRACE
        const long long tb0 = clock64();
#endif
        named_bar_sync(2, 256);
#ifdef SRL_HF_TRACE
        trc[13] += (unsigned long long)(clock64() - tb0);
#endif
        if (dw == 0 && lane == 0) {
          wait_bounded(&m3done[u3 & 1], (u3 >> 1) & 1u);
          const int s = (p0 + 2 * c) % kRingB;
          mbar_arrive(&emptyB[s]);
          mbar_arrive(&emptyB[s + 1]);
        }
      }
    }
#ifdef SRL_HF_TRACE
    trc[15] = (unsigned long long)(clock64() - t_start);
#endif
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
    if (args.counters) count_warp(args.counters + 1, nsat);
    // per-CTA column sums: the four row quadrants of each half, in quadrant order
    named_bar_sync(2, 256);
    const float* cs0 = reinterpret_cast<const float*>(smem + SL.cs_y);
    for (int i = dw * 32 + lane; i < hL; i += 256) {
      const int kb = i / 64, g2 = (i % 64) / 32, c = i % 32;
      float x = 0.f;
      for (int q = 0; q < 4; ++q) x += cs0[(g2 * 4 + q) * (hL / 2) + kb * 32 + c];
      colsum_y[(int64_t)blockIdx.x * hL + i] = -x;      // the sums were of -dZ
    }
    // dW_h^T of this CTA -> partial [blockIdx][hL][64] (the transposed split-K layout of the
    // head segment; the finalise sums the CTAs in index order)
    wait_bounded(dwdone, 0);
    tc_fence_after();
    // only the quads of the A + 1 <= 32 real columns of g (the finalise reads no others; the
    // 64-column row is allocated)
    for (int c = grp; c < NP; c += 2) {
      float v[32];
      const int fr = 128 * c + quad * 32 + (int)lane;   // feature row of dW^T
      float* dst = args.part + (int64_t)blockIdx.x * args.part_split_stride + (int64_t)fr * args.ld_part;
      tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + 64 * c, v);
      tc_wait_ld();
      const int nq = (args.A + 1 + 3) >> 2;          // the quads the finalise reads
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nq)
          reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
#ifdef SRL_HF_TRACE
  // slot 0: kernel cycles (MMA warp); 10 / 15: loss / dtanh warp cycles to the end of its loop
  if (warp == 1) trc[0] = (unsigned long long)(clock64() - t_start);
  if (warp <= 4 || warp == 8)
    for (int k = 0; k < 16; ++k)
      if (trc[k] && (lane == 0 || warp == 0 || warp == 3))   // producers: the elected lane
        atomicAdd(&g_hf_trace[blockIdx.x * 16 + k], trc[k]);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg<1>(tmem_base, 512);
  }
}

template <int KB, int RA>
static cudaError_t launch_kb(const CUtensorMap& tmY, const CUtensorMap& tmW, const CUtensorMap& tmO,
                             const GemmArgs& args, float* colsum_y, int grid, size_t smem,
                             cudaStream_t s) {
  auto kern = head_fused_kernel<KB, RA>;
  static std::atomic<size_t> configured[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (smem > configured[dev].load(std::memory_order_relaxed)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev].store(smem, std::memory_order_relaxed);
  }
  cudaError_t e = launch_k(kern, dim3((unsigned)grid), dim3(hf::kThreads), smem, s, 1, tmY, tmW,
                           tmO, args, colsum_y);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int KB>
static cudaError_t launch_ra(const CUtensorMap& tmY, const CUtensorMap& tmW, const CUtensorMap& tmO,
                             const GemmArgs& args, float* colsum_y, int grid, int zcols, cudaStream_t s) {
  constexpr int hL = KB * 64;
  for (int ra = 5; ra >= 3; --ra) {
    const size_t smem = smem_of(hL, zcols, args.n_heads, ra);
    if (smem + 512 > kSmemLimit) continue;
    if (ra == 5) return launch_kb<KB, 5>(tmY, tmW, tmO, args, colsum_y, grid, smem, s);
    if (ra == 4) return launch_kb<KB, 4>(tmY, tmW, tmO, args, colsum_y, grid, smem, s);
    return launch_kb<KB, 3>(tmY, tmW, tmO, args, colsum_y, grid, smem, s);
  }
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_head_fused(const CUtensorMap& tmY, const CUtensorMap& tmW, const CUtensorMap& tmO,
                              const GemmArgs& args, int hL, float* colsum_y, int grid,
                              cudaStream_t s) {
  if (args.A + 1 > hf::kWRows) return cudaErrorInvalidValue;
  const int zcols = args.A + 1 + args.n_heads;
  switch (hL) {
    case 128: return launch_ra<2>(tmY, tmW, tmO, args, colsum_y, grid, zcols, s);
    case 256: return launch_ra<4>(tmY, tmW, tmO, args, colsum_y, grid, zcols, s);
    case 512: return launch_ra<8>(tmY, tmW, tmO, args, colsum_y, grid, zcols, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srl

#ifdef SRL_HF_TRACE
// tools/hf_trace.py: copy out and clear the per-CTA counters [256][16]
extern "C" int srl_debug_hf_trace(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, srl::g_hf_trace, sizeof(srl::g_hf_trace)) != cudaSuccess) return 1;
  static unsigned long long zero[256 * 16];
  return cudaMemcpyToSymbol(srl::g_hf_trace, zero, sizeof(zero)) != cudaSuccess;
}
#endif
