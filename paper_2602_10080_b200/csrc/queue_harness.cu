// queue_harness.cu — device harness for the L2 queues (reference
// pkg/tests/test_l2_queues.py and acceptance criterion 3, test_acceptance.py:282).
//
// The harness drives the SAME device code the persistent solve kernel runs
// (Worker<...>::write_back / l2_read, mlmq_kernel.cuh) outside a solve:
//   * op mode (one warp): one write of a host batch, or one try_read, by a given group --
//     the backing of the Python queue objects in paper_2602_10080_b200/l2.py;
//   * stress mode: W writer warps and R reader warps run concurrently on one queue,
//     writers publishing disjoint id ranges, readers appending everything they read to
//     one output array (multiset conservation), bucket readers logging the floor they saw
//     (monotonicity).
// Instantiated for u32 distances, the vector L1 (unused here) and each L2 family.
#include "kernels/mlmq_kernel.cuh"

namespace mlmq {

// the stress writers' distance for id v (any fixed function; the host recomputes it)
__host__ __device__ inline uint32_t harness_dist(unsigned long long v) {
  unsigned long long x = v * 0x9E3779B97F4A7C15ull;
  x ^= x >> 29;
  return (uint32_t)(x & ((1u << 18) - 1u));
}

template <int L2K>
__global__ void __launch_bounds__(288, 1) queue_harness_kernel(const __grid_constant__ KParams p, HarnessArgs h) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = blockIdx.x * (blockDim.x >> 5) + warp;
  using W = Worker<DK_U32, L2K, 4, L1K_VECTOR>;
  using E = Elem<uint32_t>;
  if (h.mode == 0 || h.mode == 1) {
    if (gid != 0) return;
    W w(p, smem, h.group, lane);
    if (h.cursors) w.mcursor = h.cursors[h.group];
    if (h.mode == 0) {
      w.write_back(reinterpret_cast<const E*>(h.in), 0, (int)h.n_in, W::LINEAR);
    } else {
      const int c = w.l2_read(w.batch);
      for (int k = lane; k < c; k += 32) h.out[k] = make_uint2(w.batch[k].v, w.batch[k].d);
      if (lane == 0) *h.out_n = (unsigned long long)c;
    }
    __syncwarp();
    if (h.cursors && lane == 0) h.cursors[h.group] = w.mcursor;
    return;
  }
  // stress
  if (gid >= h.readers + h.writers) return;
  W w(p, smem + (size_t)warp * p.smem_per_warp, gid, lane);
  if (gid >= h.readers) {
    const unsigned long long wi = (unsigned long long)(gid - h.readers);
    const unsigned long long lo = wi * h.w_stride + h.w_begin, hi = wi * h.w_stride + h.w_end;
    const int bs = p.bs;
    for (unsigned long long k = lo; k < hi; k += (unsigned long long)bs) {
      const int n = (int)min((unsigned long long)bs, hi - k);
      for (int i = lane; i < n; i += 32) {
        E e;
        e.v = (uint32_t)(k + i);
        e.d = harness_dist(k + i);
        w.batch[i] = e;
      }
      __syncwarp();
      w.write_back(w.batch, 0, n, W::LINEAR);
      __syncwarp();
      if (w.stopped_warp()) return;
    }
    return;
  }
  unsigned long long nlog = 0;
  for (;;) {
    unsigned long long seen = 0;
    if (lane == 0) seen = ld_relaxed(h.out_n);
    if (__shfl_sync(FULL, seen, 0) >= h.stop_at || w.stopped_warp()) break;
    const int c = w.l2_read(w.batch);
    if (c <= 0) {
      __nanosleep(128);
      continue;
    }
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(h.out_n, (unsigned long long)c);
    base = __shfl_sync(FULL, base, 0);
    for (int k = lane; k < c; k += 32)
      if (base + k < h.out_cap) h.out[base + k] = make_uint2(w.batch[k].v, w.batch[k].d);
    if (L2K == L2K_BUCKET && h.epoch_log && lane == 0 && nlog < h.log_cap)
      h.epoch_log[(size_t)gid * h.log_cap + nlog++] = ld_relaxed(p.ctl + C_EPOCH);
    __syncwarp();
  }
  if (lane == 0 && h.log_n) h.log_n[gid] = nlog;
}

int harness_launch(int l2k, const KParams& p, const HarnessArgs& h, int warps, int wpb, size_t smem_per_warp,
                   cudaStream_t stream) {
  const void* fn = l2k == L2K_FIFO ? (const void*)queue_harness_kernel<L2K_FIFO>
                   : l2k == L2K_BUCKET ? (const void*)queue_harness_kernel<L2K_BUCKET>
                                       : (const void*)queue_harness_kernel<L2K_HEAP>;
  const size_t smem = (size_t)wpb * smem_per_warp;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const int blocks = (warps + wpb - 1) / wpb;
  void* args[] = {(void*)&p, (void*)&h};
  // stress warps spin on each other: launch cooperatively so they are co-resident
  e = h.mode == 2 ? cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(wpb * 32), args, smem, stream)
                  : cudaLaunchKernel(fn, dim3(1), dim3(32), args, smem_per_warp, stream);
  return (int)e;
}

}  // namespace mlmq
