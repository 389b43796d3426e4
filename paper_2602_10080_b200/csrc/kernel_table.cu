// kernel_table.cu — instantiations of K1 for one distance kind per translation unit.
// Compiled three times with -DMLMQ_DK=0/1/2 (u32 / u64 / f32) so nvcc runs in parallel.
#include "kernels/mlmq_kernel.cuh"

#ifndef MLMQ_DK
#error "define MLMQ_DK"
#endif

namespace mlmq {

#define MLMQ_KFN_NAME_(k) kernel_for_dk##k
#define MLMQ_KFN_NAME(k) MLMQ_KFN_NAME_(k)

const void* MLMQ_KFN_NAME(MLMQ_DK)(int l2k, int cm) {
  if (cm <= 4) {
    switch (l2k) {
      case L2K_FIFO: return (const void*)mlmq_persistent_kernel<MLMQ_DK, L2K_FIFO, 4>;
      case L2K_BUCKET: return (const void*)mlmq_persistent_kernel<MLMQ_DK, L2K_BUCKET, 4>;
      default: return (const void*)mlmq_persistent_kernel<MLMQ_DK, L2K_HEAP, 4>;
    }
  }
  switch (l2k) {
    case L2K_FIFO: return (const void*)mlmq_persistent_kernel<MLMQ_DK, L2K_FIFO, 16>;
    case L2K_BUCKET: return (const void*)mlmq_persistent_kernel<MLMQ_DK, L2K_BUCKET, 16>;
    default: return (const void*)mlmq_persistent_kernel<MLMQ_DK, L2K_HEAP, 16>;
  }
}

}  // namespace mlmq
