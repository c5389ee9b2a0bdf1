// gae.cu -- a1 (GAE reverse scan) and a2 (batch moments, merge, normalisation) kernels.
//
// GAE (BASELINE.json north_star):
//   m_t = 1 - d_t;  delta_t = r_t + gamma v_{t+1} m_t - v_t;  A_t = delta_t + gamma lambda m_t A_{t+1}
// as a chunked affine scan over T (gae_kernel below): each warp loads a 16-row chunk of 32
// columns once into registers, the chunks' (a, P) summaries are folded into carries, and the
// exact recursion then runs from the carry (integer data with gamma = lambda = 1 stays
// bit-exact, C-B1..C-B5; floating data differs from the sequential order by rounding only).
// The scan is HBM-bound: 17 B per sample (r, v, d in; adv, ret out).
// NEXT-3: a flag byte with (flag & 3) == 2 (bit 1 set, bit 0 clear) is a time-limit truncation
// (reading R-T): with trunc values the cut step bootstraps from them; a valid mask (reading R-P)
// leaves padding entries out of the moments (adv/ret are still written for every entry).
// Moments per block are {n, mean, M2} in double, merged in a fixed order (deterministic),
// shifted sums inside a thread.
#include <math.h>

#include <algorithm>

#include "internal.h"

namespace srl {

__device__ __forceinline__ void chan_merge(double& n, double& mean, double& m2, double nb,
                                           double mb, double m2b) {
  if (nb == 0.0) return;
  if (n == 0.0) { n = nb; mean = mb; m2 = m2b; return; }
  const double tot = n + nb;
  const double delta = mb - mean;
  mean = mean + delta * (nb / tot);
  m2 = m2 + m2b + delta * delta * (n * nb / tot);
  n = tot;
}

// warp merge (fixed butterfly order), result valid in every lane
__device__ __forceinline__ void warp_merge(double& n, double& mean, double& m2) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double nb = __shfl_xor_sync(0xffffffffu, n, o);
    double mb = __shfl_xor_sync(0xffffffffu, mean, o);
    double qb = __shfl_xor_sync(0xffffffffu, m2, o);
    // lower lane index first so both partners compute the same combination
    if (threadIdx.x & o) {
      double n0 = nb, m0 = mb, q0 = qb;
      chan_merge(n0, m0, q0, n, mean, m2);
      n = n0; mean = m0; m2 = q0;
    } else {
      chan_merge(n, mean, m2, nb, mb, qb);
    }
  }
}

// warp 0 merges `count` partial triples in index order: lane l folds a contiguous range, then a
// fixed butterfly; writes {n, mean, M2} and optionally {mean, sigma}
__device__ void warp0_merge_parts(const double* part, int count, double* out, double* ms,
                                  int unbiased) {
  const int lane = threadIdx.x & 31;
  double n = 0, mean = 0, m2 = 0;
  const int lo = (int)((int64_t)count * lane / 32), hi = (int)((int64_t)count * (lane + 1) / 32);
  for (int k = lo; k < hi; ++k) chan_merge(n, mean, m2, part[3 * k], part[3 * k + 1], part[3 * k + 2]);
  warp_merge(n, mean, m2);
  if (lane == 0) {
    if (out) { out[0] = n; out[1] = mean; out[2] = m2; }
    if (ms) {
      const double denom = unbiased ? n - 1.0 : n;
      ms[0] = mean;
      ms[1] = denom > 0 ? sqrt(m2 / denom) : 0.0;
    }
  }
}

// Chunked reverse scan with register-resident chunks.  A block owns 32 consecutive env columns
// (one per lane) and W warps; warp w owns the 16-row chunk [16 w, 16 w + 16) of every
// super-chunk of 16 W rows (T > 16 W loops over super-chunks, carrying A between them).  The
// recurrence A_t = delta_t + c_t A_{t+1} (c_t = gamma lambda m_t) is affine, so
//   load:   every warp loads its 16 rows once (r, v, d and v of the row after) -> delta, c;
//   pass 1: chunk summary with A = 0 after it: (a, P = prod c), published in shared memory;
//   carry:  A entering chunk w = fold of the later chunks' (a, P);
//   pass 2: the exact recursion from the carry, from registers: adv / ret / moments.
// Integer data with gamma = lambda = 1 stays bit-exact (C-B1).  All loads of a chunk are in
// flight together (row-wise, 128-byte segments across the warp); nothing is read twice.
constexpr int kTC = 16;                 // rows per chunk (per warp)

struct GaeMoments {          // shifted sums of this thread's advantages (no divisions)
  double sh = 0.0, s1 = 0.0, s2 = 0.0;
  int n = 0;
};

// warps per block (-DSRL_GAE_MAX_WARPS for the A/B): ncu per launch, atari / smac / hns /
// gfootball, 32 warps 10.2 / 61.0 / 32.4 / 12.2 us (64 registers: spills), 16 warps 6.9 / 53.5
// / 37.4 / 8.5, 8 warps 6.8 / 42.4 / 32.1 / 9.4 (no spills, two blocks per SM)
#ifndef SRL_GAE_MAX_WARPS
#define SRL_GAE_MAX_WARPS 8
#endif
template <bool TV, bool VM>
__global__ void __launch_bounds__(32 * SRL_GAE_MAX_WARPS)
gae_kernel(int T, int B, int ld, const float* __restrict__ r, const float* __restrict__ v,
           const uint8_t* __restrict__ d, const float* __restrict__ tv,
           const uint8_t* __restrict__ vmask, float gamma, float gl, float* __restrict__ adv,
           float* __restrict__ ret, double* __restrict__ part, unsigned int* counter,
           double* stats_out, double* mean_std_out, int unbiased) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int b = blockIdx.x * 32 + lane;
  const bool ok = b < B;
  const int col = ok ? b : 0;
  __shared__ float s_a[32][33], s_p[32][33];
  __shared__ float s_carry[32];
  GaeMoments mo;
  const int SC = W * kTC;
  const int nsc = (T + SC - 1) / SC;
  float carry = 0.f;                                   // A after the super-chunk (A_T = 0)
  for (int sc = nsc - 1; sc >= 0; --sc) {
    const int t0 = sc * SC + w * kTC;
    float delta[kTC], vt[kTC];
    uint32_t cut = 0, pad = 0, use = 0;                // bit i: c_i = 0 / row past T / in moments
    {
      float rr[kTC], vv[kTC + 1], tq[TV ? kTC : 1];
      uint32_t ff[kTC], mm[VM ? kTC : 1];
#pragma unroll
      for (int i = 0; i <= kTC; ++i) {                 // all loads first: one round trip
        const int64_t e = (int64_t)min(t0 + i, T) * ld + col;   // row T = bootstrap (v only)
        vv[i] = __ldg(v + e);
        if (i < kTC) {
          const int64_t e2 = (int64_t)min(t0 + i, T - 1) * ld + col;
          rr[i] = __ldg(r + e2);
          ff[i] = __ldg(d + e2);
          if constexpr (TV) tq[i] = __ldg(tv + e2);
          if constexpr (VM) mm[i] = __ldg(vmask + e2);
        }
      }
#pragma unroll
      for (int i = 0; i < kTC; ++i) {
        const bool in = t0 + i < T;
        const uint32_t f = ff[i];
        float boot = vv[i + 1];                        // v_{t+1}
        if constexpr (TV) { if (f) boot = (f & 3u) == 2u ? tq[i] : 0.f; }
        else { if (f) boot = 0.f; }
        delta[i] = in ? rr[i] + gamma * boot - vv[i] : 0.f;   // rows past T: identity step
        vt[i] = vv[i];
        if (f) cut |= 1u << i;
        if (!in) pad |= 1u << i;
        if (in && (!VM || mm[VM ? i : 0])) use |= 1u << i;
      }
    }
    auto cf = [&](int i) { return ((pad >> i) & 1u) ? 1.f : (((cut >> i) & 1u) ? 0.f : gl); };
    float a = 0.f, P = 1.f;                            // pass 1: chunk summary
#pragma unroll
    for (int i = kTC - 1; i >= 0; --i) {
      const float ci = cf(i);
      a = delta[i] + ci * a;
      P *= ci;
    }
    s_a[w][lane] = a;
    s_p[w][lane] = P;
    __syncthreads();
    float Ain = carry;
    for (int k = W - 1; k > w; --k) Ain = s_a[k][lane] + s_p[k][lane] * Ain;
    a = Ain;                                           // pass 2: the exact recursion
#pragma unroll
    for (int i = kTC - 1; i >= 0; --i) {
      a = delta[i] + cf(i) * a;
      if (ok && t0 + i < T) {
        const int64_t e = (int64_t)(t0 + i) * ld + b;
        adv[e] = a;
        if (ret) ret[e] = a + vt[i];
        if ((use >> i) & 1u) {
          if (mo.n == 0) mo.sh = a;
          const double x = (double)a - mo.sh;
          mo.s1 += x;
          mo.s2 += x * x;
          ++mo.n;
        }
      }
    }
    if (nsc > 1) {                                     // hand the carry to the earlier rows
      if (w == 0) s_carry[lane] = a;
      __syncthreads();
      carry = s_carry[lane];
      __syncthreads();
    }
  }
  if (!part) return;
  // moments: shifted sums (n, shift c, S1 = sum(a - c), S2 = sum(a - c)^2) re-centred to a
  // common shift and added -- no divisions until the block's final (mean, M2)
  auto recenter = [](double n, double c_from, double& s1, double& s2, double c_to) {
    const double dd = c_from - c_to;
    s2 += 2.0 * dd * s1 + n * dd * dd;
    s1 += n * dd;
  };
  double n = (double)mo.n, s1 = mo.s1, s2 = mo.s2;
  const unsigned valid = __ballot_sync(0xffffffffu, mo.n > 0);
  const double cw = __shfl_sync(0xffffffffu, mo.sh, valid ? __ffs(valid) - 1 : 0);
  recenter(n, mo.sh, s1, s2, cw);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {     // butterfly: both partners form the same sums
    n += __shfl_xor_sync(0xffffffffu, n, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  __shared__ double s_sum[32][4];
  if (lane == 0) { s_sum[w][0] = n; s_sum[w][1] = cw; s_sum[w][2] = s1; s_sum[w][3] = s2; }
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    double N = 0, C = 0, S1 = 0, S2 = 0;
    bool have = false;
    for (int k = 0; k < W; ++k) {          // warp order
      if (s_sum[k][0] == 0.0) continue;
      double a1 = s_sum[k][2], a2 = s_sum[k][3];
      if (!have) { C = s_sum[k][1]; have = true; }
      recenter(s_sum[k][0], s_sum[k][1], a1, a2, C);
      N += s_sum[k][0];
      S1 += a1;
      S2 += a2;
    }
    part[blockIdx.x * 3 + 0] = N;
    part[blockIdx.x * 3 + 1] = N > 0 ? C + S1 / N : 0.0;
    part[blockIdx.x * 3 + 2] = N > 0 ? fmax(S2 - S1 * S1 / N, 0.0) : 0.0;
    if (counter) {   // the last block to finish merges every block's triple (fixed order)
      __threadfence();
      s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  if (!counter) return;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) warp0_merge_parts(part, gridDim.x, stats_out, mean_std_out, unbiased);
  if (threadIdx.x == 0) *counter = 0;   // ready for the next launch
}

// one block per 32 columns; one warp per 16-row chunk (at most SRL_GAE_MAX_WARPS warps; longer
// T loops over super-chunks)
int gae_num_blocks(int B) { return (B + 31) / 32; }
static int gae_segments(int T, int B) {
  (void)B;
  // at most SRL_GAE_MAX_WARPS warps: the register-resident chunks need ~115 registers per
  // thread, which a 1024-thread bound (64 registers) spilled; longer T loops over super-chunks
  return std::max(1, std::min(SRL_GAE_MAX_WARPS, (T + kTC - 1) / kTC));
}

cudaError_t launch_gae(int T, int B, int ld, const float* r, const float* v, const uint8_t* d,
                       const float* tv, const uint8_t* vm, float gamma, float lambda, float* adv, float* ret, double* part,
                       cudaStream_t s, unsigned int* counter, double* stats_out,
                       double* mean_std_out, int unbiased) {
  const float gl = gamma * lambda;
  const dim3 grid(gae_num_blocks(B)), block(32 * gae_segments(T, B));
#define SRL_GAE(TVF, VMF)                                                                        \
  return launch_k(gae_kernel<TVF, VMF>, grid, block, 0, s, 1, T, B, ld, r, v, d, tv, vm, gamma, \
                  gl, adv, ret, part, counter, stats_out, mean_std_out, unbiased)
  if (tv && vm) SRL_GAE(true, true);
  if (tv) SRL_GAE(true, false);
  if (vm) SRL_GAE(false, true);
  SRL_GAE(false, false);
#undef SRL_GAE
}

// ---------------------------------------------------------------- a2: moments of a vector
__global__ void __launch_bounds__(256) moments_kernel(const float* __restrict__ x, int64_t n,
                                                      double* __restrict__ part) {
  griddep_wait();
  griddep_launch();
  __shared__ double s_mom[8][3];
  // block k owns the contiguous range [k*n/G, (k+1)*n/G); threads stride inside it
  const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
  double sh = 0.0, s1 = 0.0, s2 = 0.0;
  int64_t cnt = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double a = (double)__ldg(x + i);
    if (cnt == 0) sh = a;
    const double e = a - sh;
    s1 += e;
    s2 += e * e;
    ++cnt;
  }
  double N = (double)cnt;
  double mean = cnt ? sh + s1 / N : 0.0;
  double m2 = cnt ? fmax(s2 - s1 * s1 / N, 0.0) : 0.0;
  warp_merge(N, mean, m2);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_mom[w][0] = N; s_mom[w][1] = mean; s_mom[w][2] = m2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) chan_merge(a, b, c, s_mom[k][0], s_mom[k][1], s_mom[k][2]);
    part[blockIdx.x * 3 + 0] = a;
    part[blockIdx.x * 3 + 1] = b;
    part[blockIdx.x * 3 + 2] = c;
  }
}

cudaError_t launch_moments(const float* x, int64_t n, double* part, cudaStream_t s) {
  return launch_k(moments_kernel, dim3(kMomentBlocks), dim3(256), 0, s, 1, x, n, part);
}

// merge partial triples in index order (contiguous ranges per thread, then a fixed tree);
// 256 threads
__device__ void merge_parts_block(const double* part, int count, double* out, double* mean_std,
                                  int unbiased) {
  __shared__ double sn[256], sm[256], sq[256];
  const int t = threadIdx.x;
  const int lo = (int)((int64_t)count * t / 256), hi = (int)((int64_t)count * (t + 1) / 256);
  double n = 0, mean = 0, m2 = 0;
  for (int k = lo; k < hi; ++k) chan_merge(n, mean, m2, part[3 * k], part[3 * k + 1], part[3 * k + 2]);
  sn[t] = n; sm[t] = mean; sq[t] = m2;
  __syncthreads();
  for (int o = 128; o >= 1; o >>= 1) {
    if (t < o) {
      double a = sn[t], b = sm[t], c = sq[t];
      chan_merge(a, b, c, sn[t + o], sm[t + o], sq[t + o]);
      sn[t] = a; sm[t] = b; sq[t] = c;
    }
    __syncthreads();
  }
  if (t == 0) {
    if (out) { out[0] = sn[0]; out[1] = sm[0]; out[2] = sq[0]; }
    if (mean_std) {
      const double denom = unbiased ? sn[0] - 1.0 : sn[0];
      mean_std[0] = sm[0];
      mean_std[1] = denom > 0 ? sqrt(sq[0] / denom) : 0.0;
    }
  }
}

__global__ void __launch_bounds__(256) merge_moments_kernel(const double* __restrict__ part,
                                                            int count, double* out,
                                                            double* mean_std, int unbiased) {
  griddep_wait();
  griddep_launch();
  merge_parts_block(part, count, out, mean_std, unbiased);
}

// a2 across ranks over NVLink peer memory (the NCCL all-gather's replacement when the peer
// buckets are mapped): thread r stores this rank's {n, mean, M2} into rank r's slot for this
// rank (parity of the epoch), fences, release-stores the epoch into rank r's flag; then waits
// for every rank's flag here and merges the world triples in rank order with the same
// merge_parts_block as the NCCL path (identical result on every rank and on both paths).
// phases bit 0: publish this rank's triple; bit 1: wait for every rank's and merge.  A wait
// past the timeout raises the CommCtl error words and leaves mean_std as it was.
__global__ void __launch_bounds__(256) p2p_moments_kernel(const __grid_constant__ P2PPeers pe, int world, int rank,
                                                          unsigned long long epoch,
                                                          const double* __restrict__ local,
                                                          double* mean_std, int unbiased,
                                                          const CommCtl cc, int phases) {
  griddep_wait();
  griddep_launch();
  __shared__ double tri[kMaxPeers * 3];
  __shared__ int s_ok;
  const int t = threadIdx.x;
  const int par = (int)(epoch & 1ull);
  if (t == 0) s_ok = 1;
  __syncthreads();
  if ((phases & 1) && t < world) {
    double* dst = p2p_slots(pe.flag[t]) + (par * kMaxPeers + rank) * 4;
    dst[0] = local[0]; dst[1] = local[1]; dst[2] = local[2];
    __threadfence_system();
    st_release_sys(p2p_mflags(pe.flag[t]) + rank, epoch);
  }
  if (!(phases & 2)) return;
  if (t < world) {
    if (wait_epoch(p2p_mflags(pe.flag[rank]) + t, epoch, cc)) {
      const volatile double* src = p2p_slots(pe.flag[rank]) + (par * kMaxPeers + t) * 4;
      tri[3 * t] = src[0]; tri[3 * t + 1] = src[1]; tri[3 * t + 2] = src[2];
    } else {
      s_ok = 0;
    }
  }
  __syncthreads();
  if (!s_ok) return;
  merge_parts_block(tri, world, nullptr, mean_std, unbiased);
}

cudaError_t launch_p2p_moments(const P2PPeers& pe, int world, int rank, unsigned long long epoch,
                               const double* local, double* mean_std, int unbiased,
                               const CommCtl& cc, int phases, cudaStream_t s) {
  return launch_k(p2p_moments_kernel, dim3(1), dim3(256), 0, s, 1, pe, world, rank, epoch, local,
                  mean_std, unbiased, cc, phases);
}

cudaError_t launch_merge_moments(const double* part, int count, double* out, double* mean_std,
                                 int unbiased, cudaStream_t s) {
  return launch_k(merge_moments_kernel, dim3(1), dim3(256), 0, s, 1, part, count, out, mean_std,
                  unbiased);
}

__global__ void normalize_kernel(float* __restrict__ x, int64_t n, const double* __restrict__ ms,
                                 float eps) {
  griddep_wait();
  griddep_launch();
  const double mu = ms[0], sd = ms[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (float)(((double)x[i] - mu) / (sd + (double)eps));
}

cudaError_t launch_normalize(float* x, int64_t n, const double* mean_std, float eps,
                             cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * 148) blocks = 4 * 148;
  if (blocks < 1) blocks = 1;
  return launch_k(normalize_kernel, dim3((unsigned)blocks), dim3(256), 0, s, 1, x, n, mean_std, eps);
}

}  // namespace srl
