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

// ---------------------------------------------------------------------------
// K10: Proto's UNFUSED pointwise update, forallInPlace(jacobiUpdate, φ, temp,
// ρ, λ) of figure `Proto` (Eq.3): φ ← φ + λ(temp − ρ) in place,
// temp = laplace(φ, wgt) from px_stencil_apply.  Together with
// px_stencil_apply and px_residual_norm it is the unfused Proto sequence the
// fused sweep replaces (the paper's own comparison, re-run on
// the GPU: scripts/fusion_gpu.py).  Every operation rounded as in the oracle,
// so the sequence is bit-identical to the fused sweep.  Baseline only.
namespace px {
__global__ void __launch_bounds__(256) k_update(double* phi, const double* temp, const double* rhs, int64_t ldp,
                                                int64_t ldt, int64_t ldr, int nx, int ny, double lambda) {
  for (int y = blockIdx.y; y < ny; y += gridDim.y) {
    double* p = phi + (int64_t)y * ldp;
    const double* t = temp + (int64_t)y * ldt;
    const double* f = rhs + (int64_t)y * ldr;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nx; x += gridDim.x * blockDim.x)
      p[x] = __dadd_rn(p[x], __dmul_rn(lambda, __dsub_rn(t[x], f[x])));
  }
}
}  // namespace px

extern "C" px_status px_pointwise_update(px_patch* phi, const px_patch* temp, const px_patch* rhs, double lambda,
                                         px_box region, void* stream) {
  using namespace px;
  clear_error();
  PX_TRY(check_patch(phi, "phi"));
  PX_TRY(check_patch(temp, "temp"));
  PX_TRY(check_patch(rhs, "rhs"));
  if (empty(region)) return PX_OK;
  if (!contains(phi->box, region) || !contains(temp->box, region) || !contains(rhs->box, region))
    return fail(PX_ERR_DOMAIN, "px_pointwise_update: region outside a patch");
  const int nx = ext(region, 0), ny = ext(region, 1);
  const int gx = (nx + 255) / 256 < 4 ? (nx + 255) / 256 : 4;
  const int gy = ny < 4096 ? ny : 4096;
  k_update<<<dim3(gx, gy), 256, 0, (cudaStream_t)stream>>>(
      at(*phi, region.lo.c[0], region.lo.c[1]), at(*temp, region.lo.c[0], region.lo.c[1]),
      at(*rhs, region.lo.c[0], region.lo.c[1]), phi->ld, temp->ld, rhs->ld, nx, ny, lambda);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "update kernel launch");
}
