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

// Ghost images of one owned cell (fused exchange), general case (cells in
// the g rows next to a y face, corners).  Rare: called for 2g rows per sweep.
// Scalar arguments only, so the kernel parameters never need a local copy.
static __device__ __noinline__ void write_images(double* dst, int64_t ld, int X, int Y, int ox,
                                                 int oy, int n0, int n1, int g, int mx0, int mx1,
                                                 int my0, int my1, double v) {
  int ix[3], iy[3];
  double sx[3], sy[3];
  int nxi = 1, nyi = 1;
  ix[0] = X;
  iy[0] = Y;
  sx[0] = sy[0] = 1.0;
  if (X < g && mx0 != GH_NONE) {
    ix[nxi] = mx0 == GH_WRAP ? X + n0 : -X - 1;
    sx[nxi++] = mx0 == GH_REFLECT ? -1.0 : 1.0;
  }
  if (X >= n0 - g && mx1 != GH_NONE) {
    ix[nxi] = mx1 == GH_WRAP ? X - n0 : 2 * n0 - 1 - X;
    sx[nxi++] = mx1 == GH_REFLECT ? -1.0 : 1.0;
  }
  if (Y < g && my0 != GH_NONE) {
    iy[nyi] = my0 == GH_WRAP ? Y + n1 : -Y - 1;
    sy[nyi++] = my0 == GH_REFLECT ? -1.0 : 1.0;
  }
  if (Y >= n1 - g && my1 != GH_NONE) {
    iy[nyi] = my1 == GH_WRAP ? Y - n1 : 2 * n1 - 1 - Y;
    sy[nyi++] = my1 == GH_REFLECT ? -1.0 : 1.0;
  }
  for (int j = 0; j < nyi; ++j)
    for (int i = 0; i < nxi; ++i) {
      if (i == 0 && j == 0) continue;
      dst[(int64_t)(ix[i] - ox) + (int64_t)(iy[j] - oy) * ld] = v * sx[i] * sy[j];
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
  write_images(a.dst, a.ld_dst, X, Y, g.o[0], g.o[1], g.n[0], g.n[1], g.g, g.mode[0][0],
               g.mode[0][1], g.mode[1][0], g.mode[1][1], v);
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


// Canonical tap sums from register values (oracle order, each op rounded):
// the register-resident kernels (k_resident*, k_boxw).
template <int ST>
__device__ __forceinline__ double rs_taps(double w, double e, double s, double n, double c, double sw,
                                          double se, double nw, double ne) {
  if (ST == 0) return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(w, e), s), n), __dmul_rn(-4.0, c));
  double q = __dmul_rn(4.0, w);
  q = __dadd_rn(q, __dmul_rn(4.0, e));
  q = __dadd_rn(q, __dmul_rn(4.0, s));
  q = __dadd_rn(q, __dmul_rn(4.0, n));
  q = __dadd_rn(q, sw);
  q = __dadd_rn(q, se);
  q = __dadd_rn(q, nw);
  q = __dadd_rn(q, ne);
  return __dadd_rn(q, __dmul_rn(-20.0, c));
}

// Bounded spin for the cross-process waits of the peer-memory path: wait
// until *flag >= target (acquire, system scope); give up after
// PX_SPIN_TIMEOUT_NS of %globaltimer, or at once when an earlier wait of the
// communicator already gave up, and count it in *err (the synchronous solve
// reports PX_ERR_STATE; the bench's start-up self-check then falls back to
// NCCL).  A lost peer therefore ends the solve with an error, not a hang.
#ifndef PX_SPIN_TIMEOUT_NS
#define PX_SPIN_TIMEOUT_NS 2000000000ull
#endif
__device__ __forceinline__ unsigned long long px_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void px_spin_until(const unsigned long long* flag, unsigned long long target,
                                              unsigned long long* err) {
  unsigned long long v, t0 = 0;
  for (unsigned it = 0;; ++it) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) return;
    if ((it & 1023u) == 0u && err) {
      const unsigned long long t = px_globaltimer();
      if (it == 0) {
        t0 = t;
      } else if (t - t0 > PX_SPIN_TIMEOUT_NS || *(volatile unsigned long long*)err) {
        atomicAdd(err, 1ull);
        return;
      }
    }
  }
}

}  // namespace px
