// misc.cu -- gradient-bucket finalisation (a5 tail), Adam (a7), fp16 weight shadow, stats.
//
// Bucket layout (srl.h): grads[0..P) in the flat parameter layout (C-A10),
// then 8 floats: {sum l_pg, sum l_v, sum H, sum clip, sum kl} / N_global, nonfinite count,
// fp16 saturation count, 0.  Everything is pre-scaled by 1/N_global so that the NCCL sum
// over ranks (a6) yields global means (C-A14).
#include <math.h>

#include <algorithm>

#include "internal.h"
#include "srl.h"

namespace srl {

__device__ __forceinline__ int find_seg(const SegTable& t, int64_t p) {
  int k = 0;
  for (int i = 0; i < t.n; ++i)
    if (p >= t.s[i].off) k = i;
  return k;
}

// weight gradients: dW = (1/N) * sum over the split-K partials, in split order.  Work item =
// 4 consecutive entries along the partial buffer's contiguous dimension (float4 loads of every
// split, coalesced across threads): W[r][c..c+3] for hidden layers; for the head, whose
// partial holds dW^T[in][64], entries [i][j..j+3] written to W[j..j+3][i].
__device__ __forceinline__ uint32_t finalize_w_body(const SegTable& t, int64_t items, float inv_n,
                                                    float* __restrict__ bucket, int64_t q0,
                                                    int64_t qstride) {
  uint32_t bad = 0;
  for (int64_t q = q0; q < items; q += qstride) {
    int k = 0;
    for (int i = 0; i < t.n; ++i)
      if (!t.s[i].is_bias && !t.s[i].done && !t.s[i].warp && q >= t.s[i].item0) k = i;
    const Segment& s = t.s[k];
    // contiguous extent of a partial row; a transposed (head) partial holds dW^T [in][64] of
    // which this segment's `rows` columns are used
    const int prow_len = s.transposed ? min((int)s.ld_part, s.rows) : s.cols;
    const int per_row = (prow_len + 3) / 4;                        // work items per row
    const int64_t qi = q - s.item0;
    const int pr = (int)(qi / per_row), pc = 4 * (int)(qi % per_row);
    const float* src = s.part + (int64_t)pr * s.ld_part + pc;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    // 4-wide loads also for a row's last, partial quad (the entries past prow_len are read
    // from the allocation and dropped below)
    if ((s.ld_part & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && pc + 4 <= s.prow_cap) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      const int64_t st4 = s.split_stride / 4;
      for (int k0 = 0; k0 < s.splits; k0 += 20) {   // 20 loads in flight, summed in split order
        float4 x[20];
#pragma unroll
        for (int j = 0; j < 20; ++j)
          if (k0 + j < s.splits) x[j] = __ldcs(s4 + (int64_t)(k0 + j) * st4);
#pragma unroll
        for (int j = 0; j < 20; ++j)
          if (k0 + j < s.splits) { a[0] += x[j].x; a[1] += x[j].y; a[2] += x[j].z; a[3] += x[j].w; }
      }
    } else {
      const int cnt = min(4, prow_len - pc);
      for (int sp = 0; sp < s.splits; ++sp)
        for (int e = 0; e < cnt; ++e) a[e] += __ldg(src + (int64_t)sp * s.split_stride + e);
    }
    for (int e = 0; e < 4; ++e) {
      const int c = pc + e;
      if (c >= prow_len) break;
      int64_t p;
      if (s.transposed) {                    // partial [i = pr][j = c] -> W[j][i]
        if (c >= s.rows) break;
        p = s.off + (int64_t)c * s.cols + pr;
      } else {
        p = s.off + (int64_t)pr * s.cols + c;
      }
      const float g = a[e] * inv_n;
      if (!isfinite(g)) ++bad;
      bucket[p] = g;
    }
  }
  return bad;
}

// the same for segments with many partials (the fused head kernel's one per CTA): one warp per
// item, lane l sums splits l, l+32, ... in order, then a fixed butterfly (deterministic)
__device__ __forceinline__ uint32_t finalize_w_warp_body(const SegTable& t, int64_t witems,
                                                         float inv_n, float* __restrict__ bucket,
                                                         int64_t w0, int64_t wstride) {
  const int lane = threadIdx.x & 31;
  uint32_t bad = 0;
  for (int64_t q = w0; q < witems; q += wstride) {
    int k = -1;
    for (int i = 0; i < t.n; ++i)
      if (!t.s[i].is_bias && !t.s[i].done && t.s[i].warp && q >= t.s[i].item0) k = i;
    if (k < 0) continue;
    const Segment& s = t.s[k];
    const int prow_len = s.transposed ? min((int)s.ld_part, s.rows) : s.cols;
    const int per_row = (prow_len + 3) / 4;
    const int64_t qi = q - s.item0;
    const int pr = (int)(qi / per_row), pc = 4 * (int)(qi % per_row);
    const float* src = s.part + (int64_t)pr * s.ld_part + pc;
    const int cnt = min(4, prow_len - pc);
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    if ((s.ld_part & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && pc + 4 <= s.prow_cap) {
      for (int sp0 = lane; sp0 < s.splits; sp0 += 256) {     // 8 loads in flight per lane
        float4 x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int sp = sp0 + 32 * j;
          x[j] = sp < s.splits ? __ldcs(reinterpret_cast<const float4*>(src + (int64_t)sp * s.split_stride))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) { a[0] += x[j].x; a[1] += x[j].y; a[2] += x[j].z; a[3] += x[j].w; }
      }
    } else {
      for (int sp0 = lane; sp0 < s.splits; sp0 += 256) {     // 8 splits in flight per lane
        float x[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            x[j][e] = (sp0 + 32 * j < s.splits && e < cnt) ? __ldg(src + (int64_t)(sp0 + 32 * j) * s.split_stride + e) : 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) a[e] += x[j][e];
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) a[e] += __shfl_xor_sync(0xffffffffu, a[e], o);
    if (lane == 0)
      for (int e = 0; e < cnt; ++e) {
        const int c = pc + e;
        if (s.transposed && c >= s.rows) break;
        const int64_t p = s.transposed ? s.off + (int64_t)c * s.cols + pr : s.off + (int64_t)pr * s.cols + c;
        const float g = a[e] * inv_n;
        if (!isfinite(g)) ++bad;
        bucket[p] = g;
      }
  }
  return bad;
}

// bias element e of the bias segments (warp-wide): (1/N) * sum of the per-CTA column sums,
// lane-strided partials then a fixed butterfly (deterministic)
__device__ __forceinline__ uint32_t finalize_b_one(const SegTable& t, int e, float inv_n,
                                                   float* __restrict__ bucket) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < t.n; ++i) {
    const Segment& s = t.s[i];
    if (!s.is_bias) continue;
    if (e >= s.cols) { e -= s.cols; continue; }
    float acc = 0.f;
    for (int k0 = lane; k0 < s.nparts; k0 += 256) {           // 8 loads in flight per lane
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + 32 * j;
        x[j] = k < s.nparts ? __ldg(s.colsum + (int64_t)k * s.colsum_ld + e) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += x[j];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const float g = acc * inv_n;
    if (lane == 0) bucket[s.off + e] = g;
    return isfinite(g) ? 0u : 1u;
  }
  return 0u;
}

__global__ void __launch_bounds__(256) finalize_w_kernel(const SegTable t, int64_t items,
                                                         float inv_n, float* __restrict__ bucket,
                                                         unsigned long long* counters) {
  griddep_wait();
  griddep_launch();
  const uint32_t bad = finalize_w_body(t, items, inv_n, bucket,
                                       blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                                       (int64_t)gridDim.x * blockDim.x);
  const uint32_t tot = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(counters, (unsigned long long)tot);
}

// bias gradients: db = (1/N) * sum over the per-CTA column sums; one warp per element,
// lane-strided partial sums then a fixed butterfly (deterministic)
__global__ void __launch_bounds__(256) finalize_b_kernel(const SegTable t, float inv_n,
                                                         float* __restrict__ bucket,
                                                         unsigned long long* counters) {
  griddep_wait();
  griddep_launch();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (finalize_b_one(t, warp, inv_n, bucket) && (threadIdx.x & 31) == 0) atomicAdd(counters, 1ull);
}

// work items of the weight segments (4 partial-buffer entries each); sets item0.  witems
// non-null: segments with more than 32 splits get warp items (their own index space)
static int64_t finalize_items(SegTable& t, int* nbias, int64_t* witems = nullptr) {
  int64_t items = 0, wit = 0;
  int nb = 0;
  for (int i = 0; i < t.n; ++i) {
    Segment& g = t.s[i];
    if (g.is_bias) { nb += g.cols; continue; }
    if (g.done) continue;
    const int64_t prow = g.transposed ? std::min<int64_t>(g.ld_part, g.rows) : g.cols;
    const int64_t nrow = g.transposed ? g.cols : g.rows;      // head partial: [in][64]
    const int64_t cnt = nrow * ((prow + 3) / 4);
    // a warp per item (lanes stride the splits) only for FEW items with many splits (the head's
    // per-CTA partials): with many items one thread per item and 20 splits in flight keeps
    // every thread busy, while a warp walking 20+ items one after another is latency-bound
    // (gFootball's 74-split hidden layers: 42 us -> see DESIGN.md §5)
    g.warp = (witems && g.splits > 32 && cnt <= 8192) ? 1 : 0;
    if (g.warp) { g.item0 = wit; wit += cnt; }
    else { g.item0 = items; items += cnt; }
  }
  if (nbias) *nbias = nb;
  if (witems) *witems = wit;
  return items;
}

cudaError_t launch_finalize_grads(const SegTable& t0, int64_t P, float inv_n, float* bucket,
                                  unsigned long long* counters, cudaStream_t s) {
  (void)P;
  SegTable t = t0;
  int nb = 0;
  const int64_t items = finalize_items(t, &nb);
  int64_t blocks = (items + 255) / 256;
  if (blocks > 16 * num_sms()) blocks = 16 * num_sms();
  if (blocks < 1) blocks = 1;
  cudaError_t e = launch_k(finalize_w_kernel, dim3((unsigned)blocks), dim3(256), 0, s, 1, t, items,
                           inv_n, bucket, counters);
  if (e != cudaSuccess) return e;
  return launch_k(finalize_b_kernel, dim3((nb + 7) / 8), dim3(256), 0, s, 1, t, inv_n, bucket,
                  counters);
}

__global__ void extras_kernel(int64_t P, float inv_n, const double* __restrict__ stats_part,
                              int nstats, const unsigned long long* counters, float* bucket) {
  griddep_wait();
  griddep_launch();
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k < 5) {
    double s = 0.0;
    for (int g = lane; g < nstats; g += 32) s += stats_part[(int64_t)g * 8 + k];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) bucket[P + k] = (float)(s * (double)inv_n);
  } else if (k == 5 && lane == 0) {
    bucket[P + 5] = (float)counters[0];
    bucket[P + 6] = (float)counters[1];
    bucket[P + 7] = 0.f;
  }
}

cudaError_t launch_extras(int64_t P, float inv_n, const double* stats_part, int nstats,
                          const unsigned long long* counters, float* bucket, cudaStream_t s) {
  return launch_k(extras_kernel, dim3(1), dim3(192), 0, s, 1, P, inv_n, stats_part, nstats,
                  counters, bucket);
}

// a7: Adam, PyTorch semantics (C-A13); skipped entirely if any rank saw a
// non-finite loss or gradient (bucket[P+5] > 0 after the allreduce).  4 parameters per
// thread (float4 p, m, v, g); segment offsets are multiples of 4 (hidden widths % 64 == 0).
__device__ __forceinline__ float adam_one(float& p, float& m, float& v, float g, float b1, float b2,
                                          float step_size, float bc2_sqrt, float eps) {
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  p = p - step_size * (m / (sqrtf(v) / bc2_sqrt + eps));
  return p;
}

// PyTorch's bias corrections for step = t + 1: {lr / (1 - b1^step), sqrt(1 - b2^step)}, in
// double like torch.optim.Adam; computed once per block (two pow() calls)
__device__ __forceinline__ float2 adam_bias_corr(float lr, float b1, float b2, double step) {
  const float bc1 = (float)(1.0 - pow((double)b1, step));
  const float bc2_sqrt = (float)sqrt(1.0 - pow((double)b2, step));
  return make_float2(lr / bc1, bc2_sqrt);
}

// Adam over segment s for quads q = q0, q0 + qstride, ... with the step's bias corrections
// Adam for quad q (entries 4q .. 4q+3) of segment s
__device__ __forceinline__ void adam_quad(const Segment& s, int64_t q, float* __restrict__ p,
                                          float* __restrict__ m, float* __restrict__ v,
                                          const float* __restrict__ g, float step_size,
                                          float bc2_sqrt, float b1, float b2, float eps,
                                          float cf) {
  const int cnt = s.rows * s.cols;
  const bool vec_w16 = !s.is_bias && (s.cols & 3) == 0 && (s.w16_ld & 3) == 0;
  // float4 only where the segment starts 16-byte aligned (every segment of the shared layout;
  // the separate-trunk layout (R-AC) puts the critic after b_pi[A], A arbitrary)
  const bool vec = (s.off & 3) == 0;
  {
    const int e0 = 4 * (int)q;
    const int64_t i0 = s.off + e0;
    if (vec && e0 + 4 <= cnt) {
      float4 pp = *reinterpret_cast<const float4*>(p + i0);
      float4 mm = *reinterpret_cast<const float4*>(m + i0);
      float4 vv = *reinterpret_cast<const float4*>(v + i0);
      float4 gg = *reinterpret_cast<const float4*>(g + i0);
      gg.x *= cf; gg.y *= cf; gg.z *= cf; gg.w *= cf;
      adam_one(pp.x, mm.x, vv.x, gg.x, b1, b2, step_size, bc2_sqrt, eps);
      adam_one(pp.y, mm.y, vv.y, gg.y, b1, b2, step_size, bc2_sqrt, eps);
      adam_one(pp.z, mm.z, vv.z, gg.z, b1, b2, step_size, bc2_sqrt, eps);
      adam_one(pp.w, mm.w, vv.w, gg.w, b1, b2, step_size, bc2_sqrt, eps);
      *reinterpret_cast<float4*>(p + i0) = pp;
      *reinterpret_cast<float4*>(m + i0) = mm;
      *reinterpret_cast<float4*>(v + i0) = vv;
      if (s.b32) {
        s.b32[e0] = pp.x; s.b32[e0 + 1] = pp.y; s.b32[e0 + 2] = pp.z; s.b32[e0 + 3] = pp.w;
      }
      if (vec_w16) {                              // 4 entries of one row of the fp16 shadow
        const int r = e0 / s.cols, c = e0 - r * s.cols;
        __half2 h0 = __floats2half2_rn(pp.x, pp.y), h1 = __floats2half2_rn(pp.z, pp.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(s.w16 + (int64_t)r * s.w16_ld + c) = u;
      } else if (!s.is_bias) {
        const float pv[4] = {pp.x, pp.y, pp.z, pp.w};
        for (int e = 0; e < 4; ++e) {
          const int r = (e0 + e) / s.cols, c = (e0 + e) - r * s.cols;
          s.w16[(int64_t)r * s.w16_ld + c] = __float2half_rn(pv[e]);
        }
      }
    } else {
      for (int e = e0; e < min(e0 + 4, cnt); ++e) {
        const int64_t i = s.off + e;
        float pi = p[i], mi = m[i], vi = v[i];
        adam_one(pi, mi, vi, g[i] * cf, b1, b2, step_size, bc2_sqrt, eps);
        p[i] = pi; m[i] = mi; v[i] = vi;
        if (s.b32) s.b32[e] = pi;
        if (!s.is_bias) {
          const int r = e / s.cols, c = e - r * s.cols;
          s.w16[(int64_t)r * s.w16_ld + c] = __float2half_rn(pi);
        }
      }
    }
  }
}

__device__ __forceinline__ void adam_seg_body(const Segment& s, float* __restrict__ p,
                                              float* __restrict__ m, float* __restrict__ v,
                                              const float* __restrict__ g, float step_size,
                                              float bc2_sqrt, float b1, float b2, float eps,
                                              float cf, int64_t q0, int64_t qstride) {
  const int64_t nq = ((int64_t)s.rows * s.cols + 3) >> 2;
  for (int64_t q = q0; q < nq; q += qstride)
    adam_quad(s, q, p, m, v, g, step_size, bc2_sqrt, b1, b2, eps, cf);
}

__global__ void __launch_bounds__(256) adam_kernel(const SegTable t, int64_t P,
                                                   float* __restrict__ p, float* __restrict__ m,
                                                   float* __restrict__ v,
                                                   const float* __restrict__ g,
                                                   const int64_t* __restrict__ t_dev, float lr,
                                                   float b1, float b2, float eps,
                                                   const float* __restrict__ coef,
                                                   const int* __restrict__ comm_err) {
  griddep_wait();
  griddep_launch();
  if (g[P + 5] > 0.f || (comm_err && *comm_err)) return;
  const float cf = coef ? *coef : 1.f;           // NEXT-3 global-norm clip coefficient
  const float2 bc = adam_bias_corr(lr, b1, b2, (double)(t_dev[0] + 1));
  adam_seg_body(t.s[blockIdx.y], p, m, v, g, bc.x, bc.y, b1, b2, eps, cf,
                blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

cudaError_t launch_adam(const SegTable& t, int64_t P, float* p, float* m, float* v,
                        const float* bucket, const int64_t* t_dev, float lr, float b1, float b2,
                        float eps, cudaStream_t s, const float* coef, const int* comm_err) {
  int64_t maxq = 1;
  for (int i = 0; i < t.n; ++i) maxq = std::max<int64_t>(maxq, ((int64_t)t.s[i].rows * t.s[i].cols + 3) / 4);
  int64_t bx = (maxq + 255) / 256;
  if (bx > 4 * num_sms()) bx = 4 * num_sms();
  return launch_k(adam_kernel, dim3((unsigned)bx, (unsigned)t.n), dim3(256), 0, s, 1, t, P, p, m,
                  v, bucket, t_dev, lr, b1, b2, eps, coef, comm_err);
}

// ---------------------------------------------------------------------------------------
// a5 tail + a7 in ONE persistent launch (grid = #SMs, all blocks co-resident): finalise the
// split-K / per-CTA partials into the 1/N-scaled bucket, the loss statistics into its 8 extra
// slots, then (optionally) the global gradient norm (NEXT-3 R-G) and Adam with the fp16
// shadow refresh.  Grid-wide barriers separate the phases, so the skip-on-non-finite rule of
// a7 sees the whole bucket, exactly as the separate kernels did.
// The block partials of the norm are summed in block order: deterministic.
// The blocks call griddepcontrol.launch_dependents first, so the next grid (PDL) can only
// start once every block of this one is resident: the spin barrier cannot starve.
__device__ void write_stats(const float* ex, const double* mean_std, int64_t n_global, float cv,
                            float ce, int64_t* t_dev, int apply, srl_ppo_stats* out,
                            unsigned long long* counters, const double* gnorm, int cerr);
__device__ __forceinline__ bool p2p_exchange_body(const P2PPeers& pe, int world, int rank, int64_t off,
                                  int64_t count, unsigned long long epoch, float scale,
                                  float* __restrict__ out, const CommCtl& cc, int phases,
                                  bool publish);


__device__ __forceinline__ void update_adam(const UpdateArgs& u, float2& bc, double* red,
                                            int64_t tid, int64_t nthr, int warp, int lane) {
  const float* g = u.g;
  // the local non-finite count at world 1; the reduced bucket's (every rank's) otherwise
  const bool skip = ((u.finalize && !u.xchg) ? (*reinterpret_cast<volatile unsigned long long*>(u.counters) > 0)
                                             : (__ldcg(g + u.P + 5) > 0.f)) ||
                    (u.comm_err && *reinterpret_cast<volatile const int*>(u.comm_err));
  float cf = 1.f;
  if (u.max_norm > 0.f) {                          // NEXT-3: global norm of the (reduced) bucket
    double acc = 0.0;
    const int64_t nq = u.P >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (int64_t q = tid; q < nq; q += nthr) {
      const float4 x = g4[q];
      acc += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
    }
    if (blockIdx.x == 0)
      for (int64_t i = 4 * nq + threadIdx.x; i < u.P; i += blockDim.x) acc += (double)g[i] * g[i];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += red[w];
      u.gn_part[blockIdx.x] = b;
    }
    grid_barrier(u.bar);
    double x = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) x += __ldcg(u.gn_part + b);   // block order
    const double norm = sqrt(x);
    const double c = (double)u.max_norm / (norm + 1e-6);
    cf = c < 1.0 ? (float)c : 1.f;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *u.gn_norm = norm;
      *u.gn_coef = cf;
    }
  }
  __syncthreads();                                 // bc
  if (skip) return;
  const float2 b = bc;
  // one flat quad space over all segments (Segment::aq0 prefix offsets): each thread takes
  // its ~P/4/#threads quads whichever segments they fall in, instead of one pass per segment
  for (int64_t q = tid; q < u.aquads; q += nthr) {
    int k = 0;
    for (int i = 1; i < u.t.n; ++i)
      if (q >= u.t.s[i].aq0) k = i;
    adam_quad(u.t.s[k], q - u.t.s[k].aq0, u.p, u.m, u.v, g, b.x, b.y, u.b1, u.b2, u.eps, cf);
  }
}

#ifdef SRL_UPD_TRACE
// tools/upd_trace.py: per-block clock64 marks of update_kernel phases (variant builds only)
__device__ long long g_upd_trace[256 * 12];
#define UPD_MARK(k) do { __syncthreads(); if (threadIdx.x == 0) g_upd_trace[blockIdx.x * 12 + (k)] = (long long)globaltimer_ns(); } while (0)
#else
#define UPD_MARK(k) do { } while (0)
#endif

__global__ void __launch_bounds__(512) update_kernel(const UpdateArgs u) {
  griddep_launch();
  UPD_MARK(0);
  griddep_wait();
  UPD_MARK(1);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double red[16];
  __shared__ float2 bc;                            // Adam bias corrections of step t + 1
  if (u.adam && threadIdx.x == 0)                  // t read before the last block advances it
    bc = adam_bias_corr(u.lr, u.b1, u.b2, (double)(u.t_dev[0] + 1));
  if (u.finalize) {
    uint32_t bad = finalize_w_body(u.t, u.items, u.inv_n, u.bucket, tid, nthr);
    UPD_MARK(2);
    const int64_t gw = tid >> 5, nw = nthr >> 5;
    bad += finalize_w_warp_body(u.t, u.witems, u.inv_n, u.bucket, gw, nw) * (lane == 0);
    UPD_MARK(6);
    for (int64_t e = gw; e < u.nbias; e += nw) bad += finalize_b_one(u.t, (int)e, u.inv_n, u.bucket) && lane == 0;
    UPD_MARK(7);
    const uint32_t tot = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && tot) atomicAdd(u.counters, (unsigned long long)tot);
    if (blockIdx.x == 0 && warp < 5) {             // loss statistics / N
      double x = 0.0;
      for (int g = lane; g < u.nstats; g += 32) x += u.stats_part[(int64_t)g * 8 + warp];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) u.bucket[u.P + warp] = (float)(x * (double)u.inv_n);
    }
    UPD_MARK(3);
    // (no per-block fence.sys: the blocks' bucket writes reach the peers through the barrier's
    // gpu-scope release/acquire and block 0's fence.sys + release store of the publish flag --
    // causality composes; a fence.sys in all 148 blocks cost ~5 us at 4 ranks)
    grid_barrier(u.bar);
    UPD_MARK(4);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      u.bucket[u.P + 5] = (float)u.counters[0];
      u.bucket[u.P + 6] = (float)u.counters[1];
      u.bucket[u.P + 7] = 0.f;
    }
  }
  if (u.xchg) {
    // a6 in the same launch (world > 1, NVLink peer memory): block 0 publishes the bucket once
    // its extras are written (the other blocks wait on that flag like any rank's), then the
    // two-shot rank-order sum of p2p_allreduce_kernel over this grid; a barrier before Adam
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x < u.world) {
      __threadfence_system();
      st_release_sys(u.pe.flag[threadIdx.x] + u.rank, u.epoch);
    }
    p2p_exchange_body(u.pe, u.world, u.rank, u.xoff, u.P + 8, u.epoch, 1.f, u.xout, u.cc, 3, false);
    UPD_MARK(8);
    grid_barrier(u.bar);
    UPD_MARK(9);
  }
  if (u.adam) update_adam(u, bc, red, tid, nthr, warp, lane);
  UPD_MARK(5);
  if (u.stats) {
    // the step's statistics by the LAST block to get here: every block has read t and the
    // counters by then, and block 0's extras / norm writes precede its arrival
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(u.bar + 2, 1u) == gridDim.x - 1) {
        __threadfence();
        u.bar[2] = 0;
        write_stats(u.g + u.P, u.mean_std, u.n_global, u.cv, u.ce, u.t_dev, u.apply, u.out,
                    u.counters, u.max_norm > 0.f ? u.gn_norm : nullptr,
                    u.comm_err ? *(volatile const int*)u.comm_err : 0);
      }
    }
  }
}

cudaError_t launch_update(UpdateArgs u, cudaStream_t s) {
  int nb = 0;
  int64_t wit = 0;
  int64_t aq = 0;
  for (int i = 0; i < u.t.n; ++i) {
    u.t.s[i].aq0 = aq;
    aq += ((int64_t)u.t.s[i].rows * u.t.s[i].cols + 3) / 4;
  }
  u.aquads = aq;
  u.items = finalize_items(u.t, &nb, &wit);
  u.witems = wit;
  u.nbias = nb;
  return launch_k(update_kernel, dim3(num_sms()), dim3(512), 0, s, 1, u);
}

// NEXT-3 global gradient-norm clipping (reading R-G, PyTorch clip_grad_norm_ semantics):
// norm = ||g[0..P)||_2 of the (allreduced) bucket in double, coef = min(1, max_norm /
// (norm + 1e-6)); Adam scales g by coef.  Fixed grid and fixed reduction order: the last
// block to finish sums the block partials in index order (deterministic, like the GAE merge).
__global__ void __launch_bounds__(256) gradnorm_kernel(const float* __restrict__ g, int64_t P,
                                                       double* __restrict__ part,
                                                       unsigned int* counter, float max_norm,
                                                       double* norm_out, float* coef_out) {
  griddep_wait();
  griddep_launch();
  double acc = 0.0;
  const int64_t nq = P >> 2;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t q = blockIdx.x * 256 + threadIdx.x; q < nq; q += (int64_t)gridDim.x * 256) {
    const float4 x = g4[q];
    acc += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
  }
  if (blockIdx.x == 0)
    for (int64_t i = 4 * nq + threadIdx.x; i < P; i += 256) acc += (double)g[i] * g[i];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[8];
  __shared__ bool s_last;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < 8; ++w) b += red[w];
    part[blockIdx.x] = b;
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x >= 32) return;
  __threadfence();
  double x = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) x += __ldcg(part + b);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (threadIdx.x == 0) {
    const double norm = sqrt(x);
    const double cf = (double)max_norm / (norm + 1e-6);
    *norm_out = norm;
    *coef_out = cf < 1.0 ? (float)cf : 1.f;
    *counter = 0;                                 // ready for the next launch
  }
}

// a6 as a two-shot allreduce over NVLink peer memory (reduce-scatter, then all-gather; SPEC
// reduce_gradients S:L505-513, "gradient synchronisation").  The finalise /
// extras kernels of this step wrote this rank's 1/N-scaled bucket into its exposed buffer
// x[rank][parity].  The bucket is cut into `world` chunks (float4 aligned); chunk r belongs
// to rank r and is cut into gridDim.x sub-blocks, one per CTA.
//   phase 1: block 0 publishes the bucket (system fence, release store of the step's epoch
//     into every rank's phase-1 slot for this rank); every CTA waits for all ranks, then sums
//     ITS sub-block of MY chunk over the world buffers in rank order 0..world-1 (ld.global.cg
//     from the peers' HBM), writes the result to `out` and back into x[rank] in place (no
//     other rank reads that range of x[rank] in phase 1), and publishes a per-(rank, block)
//     flag to every rank.
//   phase 2: CTA g waits for the flag (j, g) of every other rank j and copies sub-block g of
//     chunk j from x[j] into `out`.
// Every element is summed once, by its owner, in rank order: bit-identical on all ranks.
// Traffic per rank 2 (world-1)/world x bytes over NVLink (the one-shot form read world-1 x).
// Double buffering by epoch parity is safe: rank A writes step k+2 into a buffer only after
// its step k+1 exchange saw B's step k+1 phase-1 publication, which B issues after finishing
// step k (including its phase-2 reads of A's buffer).
// Waits are bounded (CommCtl): on timeout the error words are raised and the kernel leaves.
__device__ __forceinline__ int64_t split4(int64_t len, int k, int parts) {
  return k >= parts ? len : ((len * k / parts) & ~int64_t(3));   // float4-aligned cut points
}

__device__ __forceinline__ void sum_range(const P2PPeers& pe, int world, int64_t off, int64_t lo,
                                          int64_t hi, float scale, float* out, float* own) {
  const int64_t q0 = (lo + 3) >> 2, q1 = hi >> 2;        // lo is a multiple of 4
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    float4 s = __ldcg(reinterpret_cast<const float4*>(pe.x[0] + off) + q);
    for (int r = 1; r < world; ++r) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(pe.x[r] + off) + q);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    s.x *= scale; s.y *= scale; s.z *= scale; s.w *= scale;
    reinterpret_cast<float4*>(out)[q] = s;
    reinterpret_cast<float4*>(own)[q] = s;
  }
  for (int64_t i = 4 * q1 + threadIdx.x; i < hi; i += blockDim.x) {   // ragged end of the bucket
    float s = __ldcg(pe.x[0] + off + i);
    for (int r = 1; r < world; ++r) s += __ldcg(pe.x[r] + off + i);
    s *= scale;
    out[i] = s;
    own[i] = s;
  }
}

// The two phases for block g of G; `publish` = block 0 also publishes this rank's bucket
// (the standalone kernel; the fused update launch publishes after its extras).  Returns false
// after a comm timeout (the error words are raised; the caller skips the rest, no early exit).
__device__ __forceinline__ bool p2p_exchange_body(const P2PPeers& pe, int world, int rank, int64_t off,
                                  int64_t count, unsigned long long epoch, float scale,
                                  float* __restrict__ out, const CommCtl& cc, int phases,
                                  bool publish) {
  __shared__ int s_ok;
  const int g = blockIdx.x, G = gridDim.x;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (phases & 1) {
    if (publish && g == 0 && threadIdx.x < world) {
      __threadfence_system();
      st_release_sys(pe.flag[threadIdx.x] + rank, epoch);
    }
    if (threadIdx.x < world && !wait_epoch(pe.flag[rank] + threadIdx.x, epoch, cc)) s_ok = 0;
    __syncthreads();
    if (!s_ok) return false;
    const int64_t c0 = split4(count, rank, world), c1 = split4(count, rank + 1, world);
    const int64_t lo = c0 + split4(c1 - c0, g, G), hi = c0 + split4(c1 - c0, g + 1, G);
    sum_range(pe, world, off, lo, hi, scale, out, pe.x[rank] + off);
    __syncthreads();
    if (threadIdx.x < world) {
      __threadfence_system();
      st_release_sys(p2p_rflags(pe.flag[threadIdx.x]) + rank * kXBlocks + g, epoch);
    }
  }
  if (phases & 2) {
    for (int j = 0; j < world; ++j) {
      if (j == rank) continue;
      if (threadIdx.x == 0 && !wait_epoch(p2p_rflags(pe.flag[rank]) + j * kXBlocks + g, epoch, cc))
        s_ok = 0;
      __syncthreads();
      if (!s_ok) return false;
      const int64_t c0 = split4(count, j, world), c1 = split4(count, j + 1, world);
      const int64_t lo = c0 + split4(c1 - c0, g, G), hi = c0 + split4(c1 - c0, g + 1, G);
      const float* src = pe.x[j] + off;
      for (int64_t q = (lo >> 2) + threadIdx.x; q < (hi >> 2); q += blockDim.x)
        reinterpret_cast<float4*>(out)[q] = __ldcg(reinterpret_cast<const float4*>(src) + q);
      for (int64_t i = (hi & ~int64_t(3)) + threadIdx.x; i < hi; i += blockDim.x)
        if (i >= lo) out[i] = __ldcg(src + i);
    }
  }
  return true;
}

__global__ void __launch_bounds__(512) p2p_allreduce_kernel(const __grid_constant__ P2PPeers pe, int world, int rank,
                                                            int64_t off, int64_t count,
                                                            unsigned long long epoch, float scale,
                                                            float* __restrict__ out,
                                                            const CommCtl cc, int phases) {
  griddep_wait();
  griddep_launch();
  p2p_exchange_body(pe, world, rank, off, count, epoch, scale, out, cc, phases, true);
}

cudaError_t launch_p2p_allreduce(const P2PPeers& pe, int world, int rank, int64_t off,
                                 int64_t count, unsigned long long epoch, float scale, float* out,
                                 const CommCtl& cc, int phases, cudaStream_t s) {
  // the same grid on every rank (the sub-block partition must agree): a function of count only
  int64_t G = count / (4 * 1024);
  if (G > kXBlocks) G = kXBlocks;
  if (G < 1) G = 1;
  return launch_k(p2p_allreduce_kernel, dim3((unsigned)G), dim3(512), 0, s, 1, pe, world, rank,
                  off, count, epoch, scale, out, cc, phases);
}

cudaError_t launch_gradnorm(const float* bucket, int64_t P, double* part, unsigned int* counter,
                            float max_norm, double* norm_out, float* coef_out, cudaStream_t s) {
  return launch_k(gradnorm_kernel, dim3(kGradNormBlocks), dim3(256), 0, s, 1, bucket, P, part,
                  counter, max_norm, norm_out, coef_out);
}

__global__ void shadow_kernel(const SegTable t, const float* __restrict__ p) {
  griddep_wait();
  griddep_launch();
  for (int k = 0; k < t.n; ++k) {
    const Segment& s = t.s[k];
    const int64_t cnt = (int64_t)s.rows * s.cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
      if (s.is_bias) {
        if (s.b32) s.b32[i] = p[s.off + i];
        continue;
      }
      const int r = (int)(i / s.cols), c = (int)(i % s.cols);
      s.w16[(int64_t)r * s.w16_ld + c] = __float2half_rn(p[s.off + i]);
    }
  }
}

cudaError_t launch_shadow(const SegTable& t, const float* p, cudaStream_t s) {
  return launch_k(shadow_kernel, dim3(2 * num_sms()), dim3(256), 0, s, 1, t, p);
}

// the step's srl_ppo_stats from the (reduced) bucket extras, the policy version advance
// (Code 1 inc_version) and the counter reset for the next step; ONE thread
__device__ void write_stats(const float* ex, const double* mean_std, int64_t n_global, float cv,
                            float ce, int64_t* t_dev, int apply, srl_ppo_stats* out,
                            unsigned long long* counters, const double* gnorm, int cerr) {
  const float e5 = __ldcg(ex + 5);
  if (counters) { counters[0] = 0; counters[1] = 0; }   // ready for the next step
  if (apply && e5 == 0.f && !cerr) t_dev[0] += 1;       // policy version (Code 1 inc_version)
  if (!out) return;
  const float e0 = __ldcg(ex), e1 = __ldcg(ex + 1), e2 = __ldcg(ex + 2);
  out->policy_loss = e0;
  out->value_loss = e1;
  out->entropy = e2;
  out->clip_fraction = __ldcg(ex + 3);
  out->approx_kl = __ldcg(ex + 4);
  out->loss = (double)e0 + (double)cv * e1 - (double)ce * e2;
  out->adv_mean = mean_std ? __ldcg(mean_std) : 0.0;
  out->adv_std = mean_std ? __ldcg(mean_std + 1) : 1.0;
  out->n_global = n_global;
  out->nonfinite = (int64_t)e5;
  out->fp16_saturated = (int64_t)__ldcg(ex + 6);
  out->step = t_dev[0];
  out->grad_norm = gnorm ? __ldcg(gnorm) : 0.0;
  out->comm_error = cerr;
}

__global__ void stats_kernel(const float* __restrict__ bucket, int64_t P,
                             const double* __restrict__ mean_std, int64_t n_global, float cv,
                             float ce, int64_t* t_dev, int apply, srl_ppo_stats* out,
                             unsigned long long* counters, const double* gnorm,
                             const int* comm_err) {
  griddep_wait();
  griddep_launch();
  write_stats(bucket + P, mean_std, n_global, cv, ce, t_dev, apply, out, counters, gnorm,
              comm_err ? *comm_err : 0);
}

cudaError_t launch_stats(const float* bucket, int64_t P, const double* mean_std,
                         int64_t n_global, float value_coef, float entropy_coef, int64_t* t_dev,
                         int apply, void* stats_out, cudaStream_t s, unsigned long long* counters,
                         const double* gnorm, const int* comm_err) {
  return launch_k(stats_kernel, dim3(1), dim3(1), 0, s, 1, bucket, P, mean_std, n_global,
                  value_coef, entropy_coef, t_dev, apply, static_cast<srl_ppo_stats*>(stats_out),
                  counters, gnorm, comm_err);
}

}  // namespace srl

#ifdef SRL_UPD_TRACE
extern "C" int srl_debug_upd_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, srl::g_upd_trace, sizeof(srl::g_upd_trace)) != cudaSuccess;
}
#endif
