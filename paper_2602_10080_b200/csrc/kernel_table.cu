// kernel_table.cu — one K1 instantiation per translation unit (distance kind x L2 family x
// L0 register capacity x L1 variant), compiled with -DMLMQ_DK/-DMLMQ_L2K/-DMLMQ_CM/-DMLMQ_L1
// so nvcc runs in parallel and each kernel carries only its own L1 code (i-cache footprint).
#include "kernels/mlmq_kernel.cuh"

#if !defined(MLMQ_DK) || !defined(MLMQ_L2K) || !defined(MLMQ_CM) || !defined(MLMQ_L1)
#error "define MLMQ_DK, MLMQ_L2K, MLMQ_CM and MLMQ_L1"
#endif

namespace mlmq {

#define MLMQ_KFN_NAME_(d, l, c, q) kernel_dk##d##_l##l##_c##c##_q##q
#define MLMQ_KFN_NAME(d, l, c, q) MLMQ_KFN_NAME_(d, l, c, q)

const void* MLMQ_KFN_NAME(MLMQ_DK, MLMQ_L2K, MLMQ_CM, MLMQ_L1)() {
  return (const void*)mlmq_persistent_kernel<MLMQ_DK, MLMQ_L2K, MLMQ_CM, MLMQ_L1>;
}

}  // namespace mlmq
