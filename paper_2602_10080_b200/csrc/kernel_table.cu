// kernel_table.cu — one K1 instantiation per translation unit (distance kind x L2 family x
// L0 register capacity), compiled with -DMLMQ_DK/-DMLMQ_L2K/-DMLMQ_CM so nvcc runs in parallel.
#include "kernels/mlmq_kernel.cuh"

#if !defined(MLMQ_DK) || !defined(MLMQ_L2K) || !defined(MLMQ_CM)
#error "define MLMQ_DK, MLMQ_L2K and MLMQ_CM"
#endif

namespace mlmq {

#define MLMQ_KFN_NAME_(d, l, c) kernel_dk##d##_l##l##_c##c
#define MLMQ_KFN_NAME(d, l, c) MLMQ_KFN_NAME_(d, l, c)

const void* MLMQ_KFN_NAME(MLMQ_DK, MLMQ_L2K, MLMQ_CM)() {
  return (const void*)mlmq_persistent_kernel<MLMQ_DK, MLMQ_L2K, MLMQ_CM>;
}

}  // namespace mlmq
