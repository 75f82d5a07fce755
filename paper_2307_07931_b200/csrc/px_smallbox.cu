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

// ---------------------------------------------------------------------------
// k_box1: the same whole-box solve on one CTA of 1024 threads, rebuilt for
// per-sweep latency (round 2; used for boxes the cluster kernel does not
// take -- fewer than 16 rows -- where it beats k_smallbox: at 64² 2.14 vs
// 2.92 µs per sweep; the 8-SM cluster kernel does 1.67).  A thread owns up to BX_MAXC cells at fixed
// positions (offsets computed once), so a sweep is: its cells' stencil and
// update -- independent chains the scheduler interleaves -- each cell at a
// face also writing its ghost images (periodic wrap / odd reflection,
// corners by the product rule) straight into the output buffer, then ONE
// block barrier.  A recorded sweep adds a warp-shuffle reduction whose 32
// per-warp partials go to shared memory; the entries are reduced over the
// warps in fixed order after the last sweep, off the sweep loop.
constexpr int BX_THREADS = 1024;
constexpr int BX_MAXC = 16;

// the images of interior cell (x, y) (value v) in the padded buffer D
static __device__ __noinline__ void bx_images(double* D, int P, int nx, int ny, int x, int y, int bc, double v) {
  int ix[3], iy[3];
  double sx[3], sy[3];
  int nxi = 1, nyi = 1;
  ix[0] = x;
  iy[0] = y;
  sx[0] = sy[0] = 1.0;
  const bool per = bc == PX_BC_PERIODIC;
  const double sg = per ? 1.0 : -1.0;
  if (x == 0) { ix[nxi] = per ? nx : -1; sx[nxi++] = sg; }       // the ghost column this cell defines
  if (x == nx - 1) { ix[nxi] = per ? -1 : nx; sx[nxi++] = sg; }
  if (y == 0) { iy[nyi] = per ? ny : -1; sy[nyi++] = sg; }
  if (y == ny - 1) { iy[nyi] = per ? -1 : ny; sy[nyi++] = sg; }
  for (int j = 0; j < nyi; ++j)
    for (int i = 0; i < nxi; ++i)
      if (i || j) D[(ix[i] + 1) + (iy[j] + 1) * P] = v * sx[i] * sy[j];
}

template <int ST, int MAXC>
__global__ void __launch_bounds__(BX_THREADS, 1) k_box1(const SmallBox b, int n_entries) {
  extern __shared__ double sm[];
  const int P = b.nx + 2, Q = b.ny + 2;
  double* A = sm;
  double* B = A + (size_t)P * Q;
  double* F = B + (size_t)P * Q;                                  // rhs, nx*ny
  double* part = F + (size_t)b.nx * b.ny;                          // [entry][warp][max bits, sum]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncell = b.nx * b.ny, npad = P * Q;
  for (int k = tid; k < npad; k += BX_THREADS) {
    const int x = k % P - 1, y = k / P - 1;
    const double v = b.phi_in[x + (int64_t)y * b.ld_in];
    A[k] = v;
    B[k] = v;  // FIXED ghosts stay in both buffers
  }
  for (int k = tid; k < ncell; k += BX_THREADS) F[k] = b.rhs[k % b.nx + (int64_t)(k / b.nx) * b.ld_rhs];
  __syncthreads();
  if (b.bc != PX_BC_FIXED_GHOSTS)  // the given ghost ring by the boundary rule (as the sweeps leave it)
    for (int k = tid; k < ncell; k += BX_THREADS) {
      const int x = k % b.nx, y = k / b.nx;
      if (x == 0 || y == 0 || x == b.nx - 1 || y == b.ny - 1) bx_images(A, P, b.nx, b.ny, x, y, b.bc, A[(x + 1) + (y + 1) * P]);
    }
  // this thread's cells: padded index, rhs index, face flag
  int ci[MAXC], fi[MAXC];
  int nc = 0;
  // 4 face bits per cell (x lo, x hi, y lo, y hi): the ghost images a cell
  // defines, written as shifts of its own index (no division in the loop)
  unsigned long long face = 0ull;
#pragma unroll
  for (int j = 0; j < MAXC; ++j) {
    const int k = tid + j * BX_THREADS;
    ci[j] = 0;
    fi[j] = 0;
    if (k < ncell) {
      const int x = k % b.nx, y = k / b.nx;
      ci[j] = (x + 1) + (y + 1) * P;
      fi[j] = k;
      if (b.bc != PX_BC_FIXED_GHOSTS) {
        const unsigned long long f = (x == 0 ? 1ull : 0ull) | (x == b.nx - 1 ? 2ull : 0ull) |
                                     (y == 0 ? 4ull : 0ull) | (y == b.ny - 1 ? 8ull : 0ull);
        face |= f << (4 * j);
      }
      nc = j + 1;
    }
  }
  const bool per = b.bc == PX_BC_PERIODIC;
  const double sg = per ? 1.0 : -1.0;
  const int dxl = per ? b.nx : -1, dxh = per ? -b.nx : 1;            // image column shifts
  const int dyl = per ? b.ny * P : -P, dyh = per ? -b.ny * P : P;    // image row shifts
  __syncthreads();
  const double scale = b.scale, lambda = b.lambda;
  int entry = 0;
  for (int s = 0; s < b.nsweeps; ++s) {
    const bool rec = b.every > 0 && s % b.every == 0;
    double mxd = 0.0, ss = 0.0;
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      if (j < nc) {
        const int i = ci[j];
        const double L = sb_taps<ST>(A, P, i);
        const double r = __dsub_rn(__dmul_rn(scale, L), F[fi[j]]);
        const double o = __dadd_rn(A[i], __dmul_rn(lambda, r));
        B[i] = o;
        const unsigned f = (unsigned)(face >> (4 * j)) & 15u;
        if (f) {
          const double so = sg * o;
          if (f & 1u) B[i + dxl] = so;
          if (f & 2u) B[i + dxh] = so;
          if (f & 12u) {
            const int dy = (f & 4u) ? dyl : dyh;
            B[i + dy] = so;
            if (f & 1u) B[i + dy + dxl] = sg * so;
            if (f & 2u) B[i + dy + dxh] = sg * so;
            if ((f & 12u) == 12u) {  // one-row box: its cells define both y images
              B[i + dyh] = so;
              if (f & 1u) B[i + dyh + dxl] = sg * so;
              if (f & 2u) B[i + dyh + dxh] = sg * so;
            }
          }
        }
        mxd = fmax(mxd, fabs(r));  // exact (one of its operands); NaN restored from Σr² below
        ss = fma(r, r, ss);
      }
    }
    if (rec) {
      unsigned long long mx = isnan(ss) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(mxd);
      for (int o = 16; o > 0; o >>= 1) {
        mx = umax64(mx, __shfl_xor_sync(FULL_MASK, mx, o));
        ss = ss + __shfl_xor_sync(FULL_MASK, ss, o);
      }
      if (lane == 0) {
        part[((size_t)entry * 32 + warp) * 2] = __longlong_as_double((long long)mx);
        part[((size_t)entry * 32 + warp) * 2 + 1] = ss;
      }
      ++entry;
    }
    __syncthreads();
    double* t = A;
    A = B;
    B = t;
  }
  if (b.final_norm) {
    double mxd = 0.0, ss = 0.0;
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      if (j >= nc) break;
      const double r = __dsub_rn(__dmul_rn(scale, sb_taps<ST>(A, P, ci[j])), F[fi[j]]);
      mxd = fmax(mxd, fabs(r));
      ss = fma(r, r, ss);
    }
    unsigned long long mx = isnan(ss) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(mxd);
    for (int o = 16; o > 0; o >>= 1) {
      mx = umax64(mx, __shfl_xor_sync(FULL_MASK, mx, o));
      ss = ss + __shfl_xor_sync(FULL_MASK, ss, o);
    }
    if (lane == 0) {
      part[((size_t)entry * 32 + warp) * 2] = __longlong_as_double((long long)mx);
      part[((size_t)entry * 32 + warp) * 2 + 1] = ss;
    }
    ++entry;
  }
  __syncthreads();
  for (int e = tid; e < entry; e += BX_THREADS) {  // entries over the warps in fixed order
    unsigned long long m = 0ull;
    double t = 0.0;
    for (int w = 0; w < 32; ++w) {
      m = umax64(m, (unsigned long long)__double_as_longlong(part[((size_t)e * 32 + w) * 2]));
      t = w ? __dadd_rn(t, part[((size_t)e * 32 + w) * 2 + 1]) : part[((size_t)e * 32 + w) * 2 + 1];
    }
    b.d_max[e] = __longlong_as_double((long long)m);
    b.d_sum[e] = t;
  }
  for (int k = tid; k < npad; k += BX_THREADS) {
    const int x = k % P - 1, y = k / P - 1;
    b.phi_out[x + (int64_t)y * b.ld_out] = A[k];
  }
}

static int box1_entries(const SmallBox& b) {
  return (b.every > 0 ? (b.nsweeps + b.every - 1) / b.every : 0) + (b.final_norm ? 1 : 0);
}
static size_t box1_smem(const SmallBox& b) {
  return ((size_t)2 * (b.nx + 2) * (b.ny + 2) + (size_t)b.nx * b.ny + (size_t)box1_entries(b) * 32 * 2) *
         sizeof(double);
}
// PROTOX_SMALLBOX (read once, A/B): unset = the 8-CTA cluster kernel when
// the box has 16+ rows, else k_box1, else k_smallbox; "box1" / "old" force
// k_box1 / k_smallbox
static int box1_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("PROTOX_SMALLBOX");
    m = !e ? 0 : (e[0] == 'b' ? 1 : (e[0] == 'o' ? 2 : 0));
  }
  return m;
}
static bool box1_eligible(const SmallBox& b) {
  return box1_mode() != 2 && b.g == 1 && (int64_t)b.nx * b.ny <= (int64_t)BX_THREADS * BX_MAXC &&
         box1_smem(b) <= 200 * 1024;
}

size_t smallbox_smem(int nx, int ny) {
  return ((size_t)2 * (nx + 2) * (ny + 2) + (size_t)nx * ny) * sizeof(double);
}

bool smallbox_fits(int nx, int ny) { return nx >= 1 && ny >= 1 && smallbox_smem(nx, ny) <= 200 * 1024; }

px_status launch_smallbox(const SmallBox& b, cudaStream_t s) {
  // 16+ rows: spread the box over a cluster of 8 SMs (px_cluster.cu): one SM
  // running k_box1 is issue-bound (73 % issue-active at 1.76 µs per 64² sweep)
  if (box1_mode() == 0 && cluster_box_eligible(b)) return launch_cluster_box(b, s);
  if (box1_eligible(b)) {
    const size_t smem = box1_smem(b);
    const bool small = (int64_t)b.nx * b.ny <= 4 * BX_THREADS;  // up to 4 cells per thread: all in registers
    void (*fn)(const SmallBox, int) = b.stencil ? (small ? k_box1<1, 4> : k_box1<1, BX_MAXC>)
                                                : (small ? k_box1<0, 4> : k_box1<0, BX_MAXC>);
    static bool attr[4] = {false, false, false, false};
    const int ai = (b.stencil ? 2 : 0) + (small ? 1 : 0);
    if (!attr[ai]) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr[ai] = true;
    }
    fn<<<1, BX_THREADS, smem, s>>>(b, box1_entries(b));
    note_kernel("k_box1");
    count_launches(1);
    return cuda_check(cudaGetLastError(), "small-box kernel launch");
  }

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
