// Small-state resident executor: the SM-resident program kernel
// (kernels.cuh resident_kernel) compiled for one-warp CTAs. For n <= 10 a
// shot's state is at most 16 KiB, so a 256-thread CTA per shot spends most of
// its time in CTA-wide barriers around short ops and in the single-thread
// sequential steps (pick_outcome / terminal scan); with one warp per CTA, a
// dozen shots run per SM and every barrier is a warp barrier. Same device
// code, same arithmetic — only the block size differs. The headers are
// compiled here under a private namespace so the two builds never meet. This
// build also runs the resident plan's staged segments (plan_resident lowers
// 2..10-qubit programs to micro-ops: CX / SWAP relabelings, fast U layouts).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#define SSB_NT 32
#define SSB_RESIDENT_STAGED 1
#define ssb ssb_w32
#include "kernels.cuh"
#undef ssb

namespace ssb {

// view: a ProgView (identical layout in both builds).
int launch_resident_warp(const void* view, uint64_t seed, uint64_t shot_begin, uint64_t count, uint64_t* values,
                         int* err, cudaStream_t stream, size_t smem, int num_sms, void* exp) {
  const auto& P = *static_cast<const ssb_w32::ProgView*>(view);
  if (cudaFuncSetAttribute(ssb_w32::resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ssb_w32::resident_kernel, ssb_w32::NT, smem) !=
      cudaSuccess)
    return -1;
  const uint64_t grid = std::min<uint64_t>(count, static_cast<uint64_t>(std::max(1, per_sm)) * num_sms);
  ssb_w32::resident_kernel<<<static_cast<unsigned>(grid), ssb_w32::NT, smem, stream>>>(P, seed, nullptr, shot_begin,
                                                                                       count, values, err,
                                                                                       static_cast<double2*>(exp));
  return cudaGetLastError() == cudaSuccess ? static_cast<int>(grid) : -1;
}

}  // namespace ssb
