// misc.cu -- gradient-bucket finalisation (a5 tail), Adam (a7), fp16 weight shadow, stats.
//
// Bucket layout (srl.h): grads[0..P) in the flat parameter layout (C-A10),
// then 8 floats: {sum l_pg, sum l_v, sum H, sum clip, sum kl} / N_global, nonfinite count,
// fp16 saturation count, 0.  Everything is pre-scaled by 1/N_global so that the NCCL sum
// over ranks (a6) yields global means (C-A14).
#include <math.h>

#include "internal.h"
#include "srl.h"

namespace srl {

__device__ __forceinline__ int find_seg(const SegTable& t, int64_t p) {
  int k = 0;
  for (int i = 0; i < t.n; ++i)
    if (p >= t.s[i].off) k = i;
  return k;
}

// weight gradients: dW = (1/N) * sum over the split-K partials, in split order
__global__ void __launch_bounds__(256) finalize_w_kernel(const SegTable t, int64_t P, float inv_n,
                                                         float* __restrict__ bucket,
                                                         unsigned long long* counters) {
  uint32_t bad = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const Segment& s = t.s[find_seg(t, p)];
    if (s.is_bias) continue;
    const int64_t idx = p - s.off;
    const int r = (int)(idx / s.cols), cc = (int)(idx % s.cols);
    const float* src = s.transposed ? s.part + (int64_t)cc * s.ld_part + r
                                    : s.part + (int64_t)r * s.ld_part + cc;
    float acc = 0.f;
#pragma unroll 4
    for (int k = 0; k < s.splits; ++k) acc += __ldg(src + (int64_t)k * s.split_stride);
    const float g = acc * inv_n;
    if (!isfinite(g)) ++bad;
    bucket[p] = g;
  }
  const uint32_t tot = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(counters, (unsigned long long)tot);
}

// bias gradients: db = (1/N) * sum over the per-CTA column sums; one warp per element,
// lane-strided partial sums then a fixed butterfly (deterministic)
__global__ void __launch_bounds__(256) finalize_b_kernel(const SegTable t, float inv_n,
                                                         float* __restrict__ bucket,
                                                         unsigned long long* counters) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int e = warp;
  for (int i = 0; i < t.n; ++i) {
    const Segment& s = t.s[i];
    if (!s.is_bias) continue;
    if (e >= s.cols) { e -= s.cols; continue; }
    float acc = 0.f;
    for (int k = lane; k < s.nparts; k += 32) acc += __ldg(s.colsum + (int64_t)k * s.colsum_ld + e);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float g = acc * inv_n;
      bucket[s.off + e] = g;
      if (!isfinite(g)) atomicAdd(counters, 1ull);
    }
    return;
  }
}

cudaError_t launch_finalize_grads(const SegTable& t, int64_t P, float inv_n, float* bucket,
                                  unsigned long long* counters, cudaStream_t s) {
  int64_t blocks = (P + 255) / 256;
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  finalize_w_kernel<<<(int)blocks, 256, 0, s>>>(t, P, inv_n, bucket, counters);
  int nb = 0;
  for (int i = 0; i < t.n; ++i)
    if (t.s[i].is_bias) nb += t.s[i].cols;
  finalize_b_kernel<<<(nb + 7) / 8, 256, 0, s>>>(t, inv_n, bucket, counters);
  return cudaGetLastError();
}

__global__ void extras_kernel(int64_t P, float inv_n, const double* __restrict__ stats_part,
                              int nstats, const unsigned long long* counters, float* bucket) {
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
  extras_kernel<<<1, 192, 0, s>>>(P, inv_n, stats_part, nstats, counters, bucket);
  return cudaGetLastError();
}

// a7: Adam, PyTorch semantics (C-A13); skipped entirely if any rank saw a
// non-finite loss or gradient (bucket[P+5] > 0 after the allreduce).
__global__ void __launch_bounds__(256) adam_kernel(const SegTable t, int64_t P,
                                                   float* __restrict__ p, float* __restrict__ m,
                                                   float* __restrict__ v,
                                                   const float* __restrict__ g,
                                                   const int64_t* __restrict__ t_dev, float lr,
                                                   float b1, float b2, float eps) {
  if (g[P + 5] > 0.f) return;
  const double step = (double)(t_dev[0] + 1);
  const float bc1 = (float)(1.0 - pow((double)b1, step));
  const float bc2_sqrt = (float)sqrt(1.0 - pow((double)b2, step));
  const float step_size = lr / bc1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float denom = sqrtf(vi) / bc2_sqrt + eps;
    const float pi = p[i] - step_size * (mi / denom);
    p[i] = pi;
    const Segment& s = t.s[find_seg(t, i)];
    if (!s.is_bias) {
      const int64_t idx = i - s.off;
      const int r = (int)(idx / s.cols), c = (int)(idx % s.cols);
      s.w16[(int64_t)r * s.w16_ld + c] = __float2half_rn(pi);
    }
  }
}

cudaError_t launch_adam(const SegTable& t, int64_t P, float* p, float* m, float* v,
                        const float* bucket, const int64_t* t_dev, float lr, float b1, float b2,
                        float eps, cudaStream_t s) {
  int64_t blocks = (P + 255) / 256;
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  adam_kernel<<<(int)blocks, 256, 0, s>>>(t, P, p, m, v, bucket, t_dev, lr, b1, b2, eps);
  return cudaGetLastError();
}

__global__ void shadow_kernel(const SegTable t, const float* __restrict__ p) {
  for (int k = 0; k < t.n; ++k) {
    const Segment& s = t.s[k];
    if (s.is_bias) continue;
    const int64_t cnt = (int64_t)s.rows * s.cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int r = (int)(i / s.cols), c = (int)(i % s.cols);
      s.w16[(int64_t)r * s.w16_ld + c] = __float2half_rn(p[s.off + i]);
    }
  }
}

cudaError_t launch_shadow(const SegTable& t, const float* p, cudaStream_t s) {
  shadow_kernel<<<2 * num_sms(), 256, 0, s>>>(t, p);
  return cudaGetLastError();
}

__global__ void stats_kernel(const float* __restrict__ bucket, int64_t P,
                             const double* __restrict__ mean_std, int64_t n_global, float cv,
                             float ce, int64_t* t_dev, int apply, srl_ppo_stats* out) {
  const float* ex = bucket + P;
  if (apply && ex[5] == 0.f) t_dev[0] += 1;   // policy version (Code 1 inc_version)
  if (!out) return;
  out->policy_loss = ex[0];
  out->value_loss = ex[1];
  out->entropy = ex[2];
  out->clip_fraction = ex[3];
  out->approx_kl = ex[4];
  out->loss = (double)ex[0] + (double)cv * ex[1] - (double)ce * ex[2];
  out->adv_mean = mean_std ? mean_std[0] : 0.0;
  out->adv_std = mean_std ? mean_std[1] : 1.0;
  out->n_global = n_global;
  out->nonfinite = (int64_t)ex[5];
  out->fp16_saturated = (int64_t)ex[6];
  out->step = t_dev[0];
}

cudaError_t launch_stats(const float* bucket, int64_t P, const double* mean_std,
                         int64_t n_global, float value_coef, float entropy_coef, int64_t* t_dev,
                         int apply, void* stats_out, cudaStream_t s) {
  stats_kernel<<<1, 1, 0, s>>>(bucket, P, mean_std, n_global, value_coef, entropy_coef, t_dev,
                               apply, static_cast<srl_ppo_stats*>(stats_out));
  return cudaGetLastError();
}

}  // namespace srl
