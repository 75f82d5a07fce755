// px_smallbox.cu -- K9: a whole small single-box solve in ONE launch
// (BASELINE config 1: one 64x64 box, 100 sweeps).
//
// At 64² a sweep is 4096 cells: one kernel per sweep is pure launch latency.
// Here one CTA loads the box (φ with its ghost ring, and the right-hand side)
// into shared memory once, runs all N sweeps there -- stencil + update +
// residual norms in registers, the ghost ring refilled by the boundary rule
// from the new interior after every sweep (periodic wrap / odd reflection /
// fixed) -- and writes φ^N back.  Per cell the oracle's expression tree with
// every * and + rounded separately (bit-identical).  Norms of the recorded
// iterates are reduced per sweep in fixed order (warp shuffles, then warps in
// order) and written to the solve's norm ring.
#include <cuda_runtime.h>

#include <cstdint>

#include "px_device.cuh"
#include "px_internal.h"

namespace px {

constexpr int SB_THREADS = 512;

__device__ __forceinline__ int sb_map(int c, int n, int bc, double& sign) {
  if (c >= 0 && c < n) return c;
  if (bc == PX_BC_PERIODIC) return c < 0 ? c + n : c - n;
  sign = -sign;  // DIRICHLET_CC: odd reflection
  return c < 0 ? -c - 1 : 2 * n - 1 - c;
}

template <int ST>
__device__ __forceinline__ double sb_taps(const double* p, int P, int i) {
  // i = index of the cell in a padded array with row stride P
  if (ST == 0) {
    return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(p[i - 1], p[i + 1]), p[i - P]), p[i + P]),
                     __dmul_rn(-4.0, p[i]));
  } else {
    double q = __dmul_rn(4.0, p[i - 1]);
    q = __dadd_rn(q, __dmul_rn(4.0, p[i + 1]));
    q = __dadd_rn(q, __dmul_rn(4.0, p[i - P]));
    q = __dadd_rn(q, __dmul_rn(4.0, p[i + P]));
    q = __dadd_rn(q, p[i - P - 1]);
    q = __dadd_rn(q, p[i - P + 1]);
    q = __dadd_rn(q, p[i + P - 1]);
    q = __dadd_rn(q, p[i + P + 1]);
    return __dadd_rn(q, __dmul_rn(-20.0, p[i]));
  }
}

// fixed-order block reduction of (max bits, sum) by all threads; thread 0
// returns the result
__device__ __forceinline__ void sb_reduce(unsigned long long mx, double ss, unsigned long long* smx,
                                          double* sss, double* out_max, double* out_sum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    mx = umax64(mx, __shfl_xor_sync(FULL_MASK, mx, o));
    ss = ss + __shfl_xor_sync(FULL_MASK, ss, o);
  }
  if (lane == 0) {
    smx[warp] = mx;
    sss[warp] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = smx[0];
    double s = sss[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      m = umax64(m, smx[w]);
      s = s + sss[w];
    }
    *out_max = __longlong_as_double((long long)m);
    *out_sum = s;
  }
  __syncthreads();
}

template <int ST>
__global__ void __launch_bounds__(SB_THREADS, 1) k_smallbox(const SmallBox b) {
  extern __shared__ double sm[];
  const int P = b.nx + 2, Q = b.ny + 2;     // padded box (ghost width 1)
  double* A = sm;
  double* B = A + (size_t)P * Q;
  double* F = B + (size_t)P * Q;            // rhs, nx*ny
  __shared__ unsigned long long smx[SB_THREADS / 32];
  __shared__ double sss[SB_THREADS / 32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ncell = b.nx * b.ny, npad = P * Q;
  // load φ (interior + ghost ring as given) and the rhs
  for (int k = tid; k < npad; k += nt) {
    const int x = k % P - 1, y = k / P - 1;
    const double v = b.phi_in[x + (int64_t)y * b.ld_in];
    A[k] = v;
    B[k] = v;  // FIXED ghosts stay in both buffers
  }
  for (int k = tid; k < ncell; k += nt) {
    const int x = k % b.nx, y = k / b.nx;
    F[k] = b.rhs[x + (int64_t)y * b.ld_rhs];
  }
  __syncthreads();
  auto fill_ring = [&](double* D) {
    if (b.bc == PX_BC_FIXED_GHOSTS) return;
    const int ring = 2 * P + 2 * b.ny;
    for (int k = tid; k < ring; k += nt) {
      int x, y;
      if (k < P) { x = k - 1; y = -1; }
      else if (k < 2 * P) { x = k - P - 1; y = b.ny; }
      else if (k < 2 * P + b.ny) { x = -1; y = k - 2 * P; }
      else { x = b.nx; y = k - 2 * P - b.ny; }
      double sg = 1.0;
      const int xs = sb_map(x, b.nx, b.bc, sg), ys = sb_map(y, b.ny, b.bc, sg);
      D[(x + 1) + (y + 1) * P] = sg * D[(xs + 1) + (ys + 1) * P];
    }
  };
  fill_ring(A);
  __syncthreads();
  const double scale = b.scale, lambda = b.lambda;
  int entry = 0;
  // thread -> fixed column, rows strided: no integer division in the sweep loop
  const int tpr = b.nx < nt ? b.nx : nt;           // threads per row
  const int rstride = nt / tpr;                    // rows handled per pass
  const int tx = tid % tpr, ty = tid / tpr;
  const bool active = ty < rstride;
  for (int s = 0; s < b.nsweeps; ++s) {
    const bool rec = b.every > 0 && s % b.every == 0;
    unsigned long long mx = 0ull;
    double ss = 0.0;
    if (active) {
      for (int y = ty; y < b.ny; y += rstride) {
        for (int x = tx; x < b.nx; x += tpr) {
          const int i = (x + 1) + (y + 1) * P;
          const double L = sb_taps<ST>(A, P, i);
          const double r = __dsub_rn(__dmul_rn(scale, L), F[x + y * b.nx]);
          B[i] = __dadd_rn(A[i], __dmul_rn(lambda, r));
          mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r)));
          ss = fma(r, r, ss);
        }
      }
    }
    __syncthreads();
    fill_ring(B);
    if (rec) {
      sb_reduce(mx, ss, smx, sss, b.d_max + entry, b.d_sum + entry);
      ++entry;
    } else {
      __syncthreads();
    }
    double* t = A;
    A = B;
    B = t;
  }
  if (b.final_norm) {
    unsigned long long mx = 0ull;
    double ss = 0.0;
    for (int k = tid; k < ncell; k += nt) {
      const int x = k % b.nx, y = k / b.nx;
      const int i = (x + 1) + (y + 1) * P;
      const double r = __dsub_rn(__dmul_rn(scale, sb_taps<ST>(A, P, i)), F[k]);
      mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r)));
      ss = fma(r, r, ss);
    }
    sb_reduce(mx, ss, smx, sss, b.d_max + entry, b.d_sum + entry);
  }
  for (int k = tid; k < npad; k += nt) {
    const int x = k % P - 1, y = k / P - 1;
    b.phi_out[x + (int64_t)y * b.ld_out] = A[k];
  }
}

size_t smallbox_smem(int nx, int ny) {
  return ((size_t)2 * (nx + 2) * (ny + 2) + (size_t)nx * ny) * sizeof(double);
}

bool smallbox_fits(int nx, int ny) { return nx >= 1 && ny >= 1 && smallbox_smem(nx, ny) <= 200 * 1024; }

px_status launch_smallbox(const SmallBox& b, cudaStream_t s) {
  // 16+ rows: spread the box over a cluster of 8 SMs (px_cluster.cu)
  if (cluster_box_eligible(b)) return launch_cluster_box(b, s);
  const size_t smem = smallbox_smem(b.nx, b.ny);
  cudaError_t e;
  if (b.stencil == 0) {
    static bool attr0 = false;
    if (!attr0) {
      cudaFuncSetAttribute(k_smallbox<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr0 = true;
    }
    k_smallbox<0><<<1, SB_THREADS, smem, s>>>(b);
  } else {
    static bool attr1 = false;
    if (!attr1) {
      cudaFuncSetAttribute(k_smallbox<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr1 = true;
    }
    k_smallbox<1><<<1, SB_THREADS, smem, s>>>(b);
  }
  note_kernel("k_smallbox");
  e = cudaGetLastError();
  count_launches(1);
  return cuda_check(e, "small-box kernel launch");
}

}  // namespace px
