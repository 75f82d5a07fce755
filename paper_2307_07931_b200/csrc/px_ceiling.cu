// px_ceiling.cu -- K12: the streaming "ceiling" of this GPU for the relax
// sweep's access pattern: c = a + b over n doubles, 2
// reads + 1 write, 16-byte vector accesses, grid-stride with 4 independent
// 16-byte loads per array in flight per thread.  Also a 1-read/1-write copy
// (the pattern of MEASURED_PEAKS.json's torch copy).  Measurement helper only;
// not on the method's path.
#include <cuda_runtime.h>

#include "px_internal.h"

namespace px {

template <bool ADD>
__global__ void __launch_bounds__(256) k_triad(const double2* __restrict__ a, const double2* __restrict__ b,
                                               double2* __restrict__ c, int64_t n2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 x[4], y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldcs(a + i + k * stride);
    if (ADD) {
#pragma unroll
      for (int k = 0; k < 4; ++k) y[k] = __ldcs(b + i + k * stride);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double2 v = x[k];
      if (ADD) {
        v.x += y[k].x;
        v.y += y[k].y;
      }
      __stcs(c + i + k * stride, v);
    }
  }
  for (; i < n2; i += stride) {
    double2 v = __ldcs(a + i);
    if (ADD) {
      const double2 w = __ldcs(b + i);
      v.x += w.x;
      v.y += w.y;
    }
    __stcs(c + i, v);
  }
}

}  // namespace px

extern "C" px_status px_stream_ceiling(const double* a, const double* b, double* c, int64_t n,
                                        int32_t variant, void* stream) {
  using namespace px;
  if (!a || !c || (variant == 0 && !b) || n < 0 || (n & 1))
    return fail(PX_ERR_ARG, "px_stream_ceiling: bad arguments (n must be even)");
  if (((uintptr_t)a | (uintptr_t)c | (uintptr_t)(b ? b : a)) & 15)
    return fail(PX_ERR_ALIGN, "px_stream_ceiling: 16-byte alignment required");
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = nsm * 8;
  cudaStream_t s = (cudaStream_t)stream;
  if (variant == 0)
    k_triad<true><<<grid, 256, 0, s>>>((const double2*)a, (const double2*)b, (double2*)c, n / 2);
  else
    k_triad<false><<<grid, 256, 0, s>>>((const double2*)a, nullptr, (double2*)c, n / 2);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "ceiling kernel launch");
}
