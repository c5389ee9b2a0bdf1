// internal.h -- declarations shared by the libsrl translation units (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "gemm_tc.cuh"
#include "srl.h"

namespace srl {

// ---- error plumbing (thread-local message behind srl_last_error)
void set_error(const std::string& msg);

// ---- device info
int num_sms();

// ---- launches: every kernel goes out with programmatic stream serialisation (PDL) so its
// prologue overlaps the previous kernel's tail; kernels call griddep_wait() before reading
// what the previous kernel wrote.  SRL_PDL=0 in the environment turns it off.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster_x > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster_x;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- a1 / a2 kernels (gae.cu)
// Moments triple {n, mean, M2} as 3 doubles.
// counter != null: the last block merges the partials into stats_out {n, mean, M2} and
// mean_std_out {mean, sigma} (either may be null) and resets *counter to 0.
cudaError_t launch_gae(int T, int B, int ld, const float* r, const float* v, const uint8_t* d,
                       const float* tv /* nullable */, const uint8_t* vm /* nullable */,
                       float gamma, float lambda, float* adv, float* ret,
                       double* part /* [gae_num_blocks(B)][3] or null */, cudaStream_t s,
                       unsigned int* counter = nullptr, double* stats_out = nullptr,
                       double* mean_std_out = nullptr, int unbiased = 0);
int gae_num_blocks(int B);
constexpr int kMomentBlocks = 256;
cudaError_t launch_moments(const float* x, int64_t n, double* part /*[kMomentBlocks][3]*/,
                           cudaStream_t s);
// merge `count` partial triples in index order -> out[3]; if mean_std != null also writes
// {mean, sigma} with sigma = sqrt(M2 / (unbiased ? n-1 : n)).
cudaError_t launch_merge_moments(const double* part, int count, double* out, double* mean_std,
                                 int unbiased, cudaStream_t s);
cudaError_t launch_normalize(float* x, int64_t n, const double* mean_std, float eps,
                             cudaStream_t s);

// ---- GEMM (mlp.cu)
bool tmap_init();
bool make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                  uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle = 128);
// D = A * B^T over the given shape; picks the instantiation (bn, a_mn, b_mn, epi).
// to: epilogue output map (fp16, box 32x32, 64-byte swizzle); ty: y_prev map (DTANH).
// cg = 2: CTA pairs (cluster 2x1) with tcgen05 cta_group::2, 256-row tiles; grid even.
cudaError_t launch_gemm(int bn, bool a_mn, bool b_mn, int epi, int cg, const CUtensorMap& ta,
                        const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& ty,
                        const GemmArgs& args, int grid, cudaStream_t s);

// ---- a4 + head part of a5 in one kernel (head_fused.cu): loss, dZ_L (+ db_L column sums into
// colsum_y [grid][hL]) and dW_h^T partials [grid][hL][64] (args.part); hL % 128 == 0, <= 512
size_t head_fused_smem(int hL, int zcols, int n_heads);
cudaError_t launch_head_fused(const CUtensorMap& tmY, const CUtensorMap& tmW, const CUtensorMap& tmO,
                              const GemmArgs& args, int hL, float* colsum_y, int grid,
                              cudaStream_t s);

// ---- parameter segments (misc.cu): one weight matrix or bias vector of the flat layout
struct Segment {
  int64_t off;          // offset in the flat parameter / gradient vector
  int rows, cols;       // weight: [rows=out][cols=in]; bias: rows = 1, cols = out
  int is_bias;
  // gradient source
  const float* part;    // weight: dW partials [splits][part_rows][ld_part] (transposed if head)
  int splits;
  int64_t ld_part, split_stride;
  int transposed;       // head: partial holds dW^T ([in][G])
  int prow_cap;         // floats readable from a partial row's first used entry (<= ld_part):
                        // a 4-wide load at any used column stays inside the allocation
  const float* colsum;  // bias: [nparts][colsum_ld]
  int nparts, colsum_ld;
  // fp16 shadow (weights only)
  __half* w16;
  int w16_ld;
  float* b32;           // bias only, nullable: fp32 mirror the GEMM epilogue reads (R-AC head)
  int done;             // weight already reduced into the bucket by its dW launch (part_fixup)
  int64_t item0;        // finalize: first work item (4 partial-buffer entries) of this segment
  int64_t aq0;          // Adam (update_kernel): first quad of this segment in the flat space
  int warp;             // finalize: 1 = many splits, one WARP per item (lanes stride the splits)
};
constexpr int kMaxSegs = 20;
struct SegTable {
  int n;
  Segment s[kMaxSegs];
};
cudaError_t launch_finalize_grads(const SegTable& t, int64_t P, float inv_n, float* bucket,
                                  unsigned long long* counters, cudaStream_t s);
cudaError_t launch_extras(int64_t P, float inv_n, const double* stats_part, int nstats,
                          const unsigned long long* counters, float* bucket, cudaStream_t s);
cudaError_t launch_adam(const SegTable& t, int64_t P, float* p, float* m, float* v,
                        const float* bucket, const int64_t* t_dev, float lr, float b1,
                        float b2, float eps, cudaStream_t s, const float* coef = nullptr,
                        const int* comm_err = nullptr);
constexpr int kGradNormBlocks = 296;   // 2 x 148 SMs
// a6 over NVLink peer memory (world <= 8 on one node): every rank's exposed bucket (double
// buffered by step parity) and flag array, mapped into this process with CUDA IPC
constexpr int kMaxPeers = 8;
constexpr int kXBlocks = 148;             // CTAs of the two-shot exchange = sub-blocks per chunk
struct P2PPeers {
  float* x[kMaxPeers];                    // rank r's exposed buckets [2][count]
  unsigned long long* flag[kMaxPeers];    // rank r's sync block (layout below)
};
// layout of every rank's IPC-mapped sync block (flag[r] points at rank r's), in u64 words:
//   [0, 8)    bucket-published flags, slot src = src's epoch            (exchange phase 1)
//   [8, 16)   moments flags, slot src = src's moments epoch             (a2)
//   [16, 80)  doubles [2 parity][kMaxPeers][4] moment slots             (a2)
//   [80, 80 + kMaxPeers * kXBlocks) reduced-chunk flags [src][block]    (exchange phase 2)
__host__ __device__ inline unsigned long long* p2p_mflags(unsigned long long* base) { return base + kMaxPeers; }
__host__ __device__ inline double* p2p_slots(unsigned long long* base) {
  return reinterpret_cast<double*>(base + 2 * kMaxPeers);
}
__host__ __device__ inline unsigned long long* p2p_rflags(unsigned long long* base) {
  return base + 2 * kMaxPeers + 2 * kMaxPeers * 4;
}
constexpr size_t kSyncWords = 2 * kMaxPeers + 2 * kMaxPeers * 4 + kMaxPeers * kXBlocks;
constexpr size_t kSyncBytes = sizeof(unsigned long long) * kSyncWords;
// bounded waits of the exchange kernels (SPEC.md S:L532 ReduceTimeout): a wait that exceeds
// timeout_ns sets *err_dev and *err_host (host-mapped) to 1 and the kernel leaves without
// trapping; Adam then skips (err_dev) and the next srl_* call on the context returns SRL_ENCCL.
struct CommCtl {
  int* err_dev;                 // device word, read by adam_kernel / stats_kernel
  int* err_host;                // device alias of pinned host memory, read by the host
  unsigned long long timeout_ns;
};

// a5 tail + a7 in one persistent launch (misc.cu update_kernel): finalise (if `finalize`) the
// partials into `bucket` with the loss statistics, then (if `adam`) the optional global-norm
// clip and Adam + fp16 shadow reading `g` (== bucket at world 1, the reduced bucket otherwise),
// then (if `stats`) the step's statistics
struct UpdateArgs {
  SegTable t;
  int64_t P, items, witems, nbias, aquads;
  float inv_n;
  float* bucket;
  unsigned long long* counters;
  const double* stats_part;
  int nstats;
  int finalize, adam;
  const float* g;
  float *p, *m, *v;
  int64_t* t_dev;
  float lr, b1, b2, eps, max_norm;
  double* gn_part;          // [>= #SMs]
  double* gn_norm;
  float* gn_coef;
  const int* comm_err;
  unsigned* bar;            // grid barrier words [3], zero-initialised ([2]: blocks done)
  // the step's last launch (`stats`): its last block writes srl_ppo_stats from g[P..P+8),
  // advances t if Adam ran, re-zeroes the counters (what stats_kernel does standalone)
  int stats, apply;
  const double* mean_std;
  int64_t n_global;
  float cv, ce;
  srl_ppo_stats* out;
  // xchg: world > 1 over NVLink peer memory -- the a6 exchange between finalise and Adam in
  // this launch (grid = #SMs on every rank: the same sub-block partition everywhere)
  int xchg, world, rank;
  P2PPeers pe;
  CommCtl cc;
  int64_t xoff;
  unsigned long long epoch;
  float* xout;
};
cudaError_t launch_update(UpdateArgs u, cudaStream_t s);
// phases: bit 0 = publish / reduce my chunk, bit 1 = gather the other chunks (3 = both; the
// single-GPU virtual-rank test runs bit 0 for every rank, then bit 1 for every rank).
cudaError_t launch_p2p_moments(const P2PPeers& pe, int world, int rank, unsigned long long epoch,
                               const double* local, double* mean_std, int unbiased,
                               const CommCtl& cc, int phases, cudaStream_t s);
cudaError_t launch_p2p_allreduce(const P2PPeers& pe, int world, int rank, int64_t off,
                                 int64_t count, unsigned long long epoch, float scale, float* out,
                                 const CommCtl& cc, int phases, cudaStream_t s);
cudaError_t launch_gradnorm(const float* bucket, int64_t P, double* part, unsigned int* counter,
                            float max_norm, double* norm_out, float* coef_out, cudaStream_t s);
cudaError_t launch_shadow(const SegTable& t, const float* p, cudaStream_t s);
cudaError_t launch_stats(const float* bucket, int64_t P, const double* mean_std,
                         int64_t n_global, float value_coef, float entropy_coef,
                         int64_t* t_dev, int apply, void* stats_out, cudaStream_t s,
                         unsigned long long* counters = nullptr, const double* gnorm = nullptr,
                         const int* comm_err = nullptr);
// spin helpers shared by the exchange kernels (misc.cu, gae.cu)
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void comm_fail(const CommCtl& cc) {
  *reinterpret_cast<volatile int*>(cc.err_dev) = 1;
  *reinterpret_cast<volatile int*>(cc.err_host) = 1;
  __threadfence_system();
}
// wait until *f >= epoch; false (and the error raised) after cc.timeout_ns or once another
// wait of this step has failed
__device__ __forceinline__ bool wait_epoch(const unsigned long long* f, unsigned long long epoch,
                                           const CommCtl& cc) {
  if (ld_acquire_sys(f) >= epoch) return true;
  const unsigned long long t0 = globaltimer_ns();
  uint32_t it = 0;
  while (ld_acquire_sys(f) < epoch) {
    if ((++it & 255u) == 0) {
      if (*reinterpret_cast<volatile int*>(cc.err_dev)) return false;
      if (globaltimer_ns() - t0 > cc.timeout_ns) {
        comm_fail(cc);
        return false;
      }
    }
  }
  return true;
}

}  // namespace srl
