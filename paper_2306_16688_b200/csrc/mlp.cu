// mlp.cu -- TMA descriptor encoding and the GEMM instantiations used by the trainer step.
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>

#include "internal.h"

namespace srl {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool tmap_init() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// fp16 row-major matrix with `outer` rows of `inner` elements, row pitch row_bytes;
// box {box_inner, box_outer}, 128-byte (operands) or 64-byte (epilogue 32x32 tiles) swizzle;
// out-of-bounds elements read as zero and are clipped on store.
bool make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                  uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle) {
  if (!tmap_init()) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool AM, bool BM, int EPI, int CG>
static cudaError_t launch_one(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to,
                              const CUtensorMap& ty, GemmArgs a, int grid, cudaStream_t s) {
  auto kern = gemm_tc_kernel<BN, AM, BM, EPI, CG>;
  constexpr int E = EPI == EPI_TANH_ACC ? EPI_TANH : EPI;   // same smem layout
  const int zcols = a.A + 1 + a.n_heads;
  if (a.stages <= 0) a.stages = gemm_stages(BN, E, a.colsum_ld, CG, zcols);
  if (a.stages < 2) return cudaErrorInvalidConfiguration;
  const size_t smem = 1024 + smem_layout(BN, E, a.stages, a.colsum_ld, CG, zcols).total;
  if (smem + 512 > kSmemLimit) return cudaErrorInvalidConfiguration;
  // the attribute is per device: cache the configured size per device id (atomic: contexts on
  // several devices may launch from several threads)
  static std::atomic<size_t> configured[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (smem > configured[dev].load(std::memory_order_relaxed)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev].store(smem, std::memory_order_relaxed);
  }
  cudaError_t e = launch_k(kern, dim3((unsigned)grid), dim3(kThreads), smem, s, CG, ta, tb, to, ty, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

#define SRL_DISPATCH_BN(AM, BM, EPI, CG)                                                 \
  switch (bn) {                                                                          \
    case 64: return launch_one<64, AM, BM, EPI, 1>(ta, tb, to, ty, args, grid, s);       \
    case 128: return CG == 2 ? launch_one<128, AM, BM, EPI, 2>(ta, tb, to, ty, args, grid, s) \
                             : launch_one<128, AM, BM, EPI, 1>(ta, tb, to, ty, args, grid, s); \
    case 256: return CG == 2 ? launch_one<256, AM, BM, EPI, 2>(ta, tb, to, ty, args, grid, s) \
                             : launch_one<256, AM, BM, EPI, 1>(ta, tb, to, ty, args, grid, s); \
    default: return cudaErrorInvalidValue;                                               \
  }

cudaError_t launch_gemm(int bn, bool a_mn, bool b_mn, int epi, int cg, const CUtensorMap& ta,
                        const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& ty,
                        const GemmArgs& args, int grid, cudaStream_t s) {
  if (grid < 1) grid = 1;
  if (cg != 1 && cg != 2) return cudaErrorInvalidValue;
  if (cg == 2 && (grid & 1)) return cudaErrorInvalidConfiguration;
  switch (epi) {
    case EPI_TANH:
      if (!a_mn && !b_mn) { SRL_DISPATCH_BN(false, false, EPI_TANH, cg) }
      break;
    case EPI_TANH_ACC:
      if (!a_mn && !b_mn) { SRL_DISPATCH_BN(false, false, EPI_TANH_ACC, cg) }
      break;
    case EPI_DTANH:
      if (!a_mn && b_mn) { SRL_DISPATCH_BN(false, true, EPI_DTANH, cg) }
      break;
    case EPI_LOSS:
      if (!a_mn && !b_mn && bn == 64 && cg == 1)
        return launch_one<64, false, false, EPI_LOSS, 1>(ta, tb, to, ty, args, grid, s);
      break;
    case EPI_SAMPLE:
      if (!a_mn && !b_mn && bn == 64 && cg == 1)
        return launch_one<64, false, false, EPI_SAMPLE, 1>(ta, tb, to, ty, args, grid, s);
      break;
    case EPI_PART:
      if (a_mn && b_mn && bn == 512 && cg == 2)
        return launch_one<512, true, true, EPI_PART, 2>(ta, tb, to, ty, args, grid, s);
      if (!a_mn && !b_mn) { SRL_DISPATCH_BN(false, false, EPI_PART, cg) }
      if (!a_mn && b_mn) { SRL_DISPATCH_BN(false, true, EPI_PART, cg) }
      if (a_mn && !b_mn) { SRL_DISPATCH_BN(true, false, EPI_PART, cg) }
      if (a_mn && b_mn) { SRL_DISPATCH_BN(true, true, EPI_PART, cg) }
      break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace srl
