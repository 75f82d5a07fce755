// px_device.cuh -- device helpers shared by the relax kernels (px_kernels.cu,
// px_bulk.cu): fused ghost images of owned cells and the deterministic
// fixed-order norm reduction.  Included by .cu files only.
#pragma once
#include <cuda_runtime.h>

#include "px_internal.h"

namespace px {

constexpr unsigned FULL_MASK = 0xffffffffu;

static __device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

// Ghost images of one owned cell (fused exchange).  Rarely executed: only
// cells within g of a face.
static __device__ __noinline__ void write_images(const StreamLaunch& a, int x, int y, double v) {
  const GhostSpec& g = a.gs;
  const int X = x + g.o[0], Y = y + g.o[1];
  int ix[3], iy[3];
  double sx[3], sy[3];
  int nxi = 1, nyi = 1;
  ix[0] = X;
  iy[0] = Y;
  sx[0] = sy[0] = 1.0;
  for (int d = 0; d < 2; ++d) {
    const int P = d ? Y : X, n = g.n[d];
    int* im = d ? iy : ix;
    double* sg = d ? sy : sx;
    int& cnt = d ? nyi : nxi;
    if (P < g.g && g.mode[d][0] != GH_NONE) {
      im[cnt] = g.mode[d][0] == GH_WRAP ? P + n : -P - 1;
      sg[cnt] = g.mode[d][0] == GH_REFLECT ? -1.0 : 1.0;
      ++cnt;
    }
    if (P >= n - g.g && g.mode[d][1] != GH_NONE) {
      im[cnt] = g.mode[d][1] == GH_WRAP ? P - n : 2 * n - 1 - P;
      sg[cnt] = g.mode[d][1] == GH_REFLECT ? -1.0 : 1.0;
      ++cnt;
    }
  }
  for (int j = 0; j < nyi; ++j)
    for (int i = 0; i < nxi; ++i) {
      if (i == 0 && j == 0) continue;
      a.dst[(int64_t)(ix[i] - g.o[0]) + (int64_t)(iy[j] - g.o[1]) * a.ld_dst] = v * sx[i] * sy[j];
    }
}

// Fused ghost images of one owned cell written along with it.  Inlined fast
// path for the common cases (no image; one x image); the rare y-face rows and
// corners go through write_images.
static __device__ __forceinline__ void images(const StreamLaunch& a, int x, int y, double v) {
  const GhostSpec& g = a.gs;
  const int X = x + g.o[0], Y = y + g.o[1];
  const bool yface = (Y < g.g) || (Y >= g.n[1] - g.g);
  const bool xlo = X < g.g, xhi = X >= g.n[0] - g.g;
  if (!(yface || xlo || xhi)) return;
  if (!yface && xlo != xhi) {
    const int m = xlo ? g.mode[0][0] : g.mode[0][1];
    if (m == GH_NONE) return;
    const int n = g.n[0];
    const int ix = xlo ? (m == GH_WRAP ? X + n : -X - 1) : (m == GH_WRAP ? X - n : 2 * n - 1 - X);
    a.dst[(int64_t)(ix - g.o[0]) + (int64_t)y * a.ld_dst] = (m == GH_REFLECT) ? -v : v;
    return;
  }
  write_images(a, x, y, v);
}

// Fixed-order block reduction of (max-bits, sum), then the last block of the
// slot reduces all partials.  Deterministic for a given launch geometry.
static __device__ void reduce_norms(const NormSlot& ns, unsigned long long mx, double ss) {
  __shared__ unsigned long long s_mx[32];
  __shared__ double s_ss[32];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nthreads = blockDim.x;
  for (int o = 16; o > 0; o >>= 1) {
    mx = umax64(mx, __shfl_xor_sync(FULL_MASK, mx, o));
    ss = ss + __shfl_xor_sync(FULL_MASK, ss, o);
  }
  if (lane == 0) {
    s_mx[warp] = mx;
    s_ss[warp] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = s_mx[0];
    double s = s_ss[0];
    for (int w = 1; w < nthreads / 32; ++w) {
      m = umax64(m, s_mx[w]);
      s = s + s_ss[w];
    }
    const int bid = ns.offset + blockIdx.x + blockIdx.y * gridDim.x;
    ns.partials[2 * bid] = __longlong_as_double((long long)m);
    ns.partials[2 * bid + 1] = s;
    __threadfence();
    unsigned t = atomicAdd(ns.counter, 1u);
    s_last = (t == (unsigned)ns.expected - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  unsigned long long m = 0;
  double s = 0.0;
  for (int i = threadIdx.x; i < ns.expected; i += nthreads) {
    m = umax64(m, (unsigned long long)__double_as_longlong(__ldcg(ns.partials + 2 * i)));
    s = s + __ldcg(ns.partials + 2 * i + 1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = umax64(m, __shfl_xor_sync(FULL_MASK, m, o));
    s = s + __shfl_xor_sync(FULL_MASK, s, o);
  }
  __syncthreads();
  if (lane == 0) {
    s_mx[warp] = m;
    s_ss[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    m = s_mx[0];
    s = s_ss[0];
    for (int w = 1; w < nthreads / 32; ++w) {
      m = umax64(m, s_mx[w]);
      s = s + s_ss[w];
    }
    *ns.out_max = __longlong_as_double((long long)m);
    *ns.out_sum = s;
    *ns.counter = 0u;
    __threadfence();
  }
}


}  // namespace px
