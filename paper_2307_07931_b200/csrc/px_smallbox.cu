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

#include <cmath>
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
// PROTOX_SMALLBOX (read once, A/B): unset = k_boxw (nx <= 64, ny <= 128),
// else the 8-CTA cluster kernel when the box has 16+ rows, else k_box1, else
// k_smallbox; "cluster" skips k_boxw; "box1" / "old" force k_box1 / k_smallbox
static int box1_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("PROTOX_SMALLBOX");
    m = !e ? 0 : (e[0] == 'b' ? 1 : (e[0] == 'o' ? 2 : (e[0] == 'c' ? 3 : 0)));
  }
  return m;
}
static bool box1_eligible(const SmallBox& b) {
  return box1_mode() != 2 && b.g == 1 && (int64_t)b.nx * b.ny <= (int64_t)BX_THREADS * BX_MAXC &&
         box1_smem(b) <= 200 * 1024;
}

// ---------------------------------------------------------------------------
// k_boxw: the whole-box solve with the box IN REGISTERS, one warp per row
// group (round 2, BASELINE config 1).  Lane l of warp w owns column pair l
// (columns 2l, 2l+1; nx <= 64) of rows w·RW .. w·RW + RW - 1 of its CTA's
// ny/CL rows (16 warps, ny/CL <= 16·RW, RW <= 4; CL CTAs form a cluster,
// below), φ and ρ in registers for the whole solve.  W/E neighbours are indexed
// shuffles inside the warp (the periodic wrap falls out of the lane index;
// odd reflection / fixed ghosts are a select at lanes 0 and np-1); N/S
// neighbours inside the row group are registers, across groups one 16-B
// shared load per row group edge from a double-buffered row board that every
// warp writes its first and last rows into (with the y images at the domain
// faces) before the ONE block barrier per sweep.  A recorded sweep adds a
// warp butterfly of (max bits, Σr²) whose per-warp partials go to shared
// memory, reduced over the warps in fixed order after the last sweep.  Per
// cell the oracle's expression tree (power-of-two h and λ: the exact fused
// multiply-adds of k_resident_reg): bit-identical φ and max-norm.  The max
// per warp by two redux.sync steps on the bit pattern, not a 64-bit
// butterfly (the norm is recorded every sweep at BJ.C1).  Over a cluster of
// CL CTAs (default 8 at 64²: 0.79 µs per sweep, one CTA 1.14) the halo rows a
// CTA reads from its neighbours arrive by st.async counted on a per-buffer
// mbarrier that only the reading warps wait on, and the per-sweep barrier is
// the CTA's own.
constexpr int BW_THREADS = 512;  // 16 warps: 128 registers a thread, up to 4 rows of φ, ρ in registers
constexpr int BW_WARPS = BW_THREADS / 32;
constexpr int BW_CL_DEFAULT = 8;  // 64² (BJ.C1): 1 / 2 / 4 / 8 CTAs 1.14 / 1.26 / 0.955 / 0.89 µs per sweep
// rows per warp (1, 2 or 4) of an nx x ny box; 0: not eligible
static int bw_rows_per_warp(int nx, int ny) {
  if (nx < 2 || nx > 64 || (nx & 1) || ny < 1) return 0;
  for (int rw = 1; rw <= 4; rw *= 2)
    if (ny <= BW_WARPS * rw && ny % rw == 0) return rw;
  return 0;
}
// CL > 1: the box over a cluster of CL CTAs (CTA rank cr owns rows cr·ny/CL ..),
// each keeping a full-height row board; a row another CTA reads (the CTA's
// first / last row, the periodic y images) is also stored into that CTA's
// board through DSMEM, and the per-sweep barrier is the cluster barrier.
__device__ __forceinline__ unsigned bw_cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void bw_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16-B store of v at local shared address p into CTA t's copy of the same slot
__device__ __forceinline__ void bw_st_remote(const double* p, unsigned t, double2 v) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(p);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(t));
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(v.x), "d"(v.y) : "memory");
}
// the same store as st.async, counted (16 bytes) on CTA t's mbarrier `bar`
__device__ __forceinline__ void bw_st_async(const double* p, unsigned t, double2 v, const uint64_t* bar) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(p), lb = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(t));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(t));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra),
               "d"(v.x), "d"(v.y), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void bw_mbar_wait(const uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double2 bw_ld_remote(const double* p, unsigned t) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(p);
  unsigned ra;
  double2 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(t));
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}

template <int ST, bool P2, int RW, int CL>
__global__ void __launch_bounds__(BW_THREADS, 1) k_boxw(const SmallBox b, int n_entries, int mb) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t hb[2];  // mb: the remote halo rows of board buffer 0 / 1 (bytes counted)
  const int nx = b.nx, ny = b.ny, np = nx / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cr = CL > 1 ? (int)bw_cta_rank() : 0;
  const int nyl = ny / CL, yb = cr * nyl;  // this CTA's rows yb .. yb + nyl - 1
  if (CL > 1) bw_cluster_sync();           // every CTA of the cluster runs before any DSMEM store
  double* board = sm;                                   // [2][ny + 2][nx]: rows -1 .. ny
  double* part = board + (size_t)2 * (ny + 2) * nx;     // [entry][BW_WARPS][max bits, sum]
  double* gcor = part + (size_t)n_entries * BW_WARPS * 2;  // [4] fixed corners (-1,-1) (nx,-1) (-1,ny) (nx,ny)
  const int bsz = (ny + 2) * nx;
  const int y0 = yb + warp * RW;
  const bool wact = warp * RW < nyl;                    // warp-uniform
  const bool act = wact && lane < np;
  const int xs = lane < np ? 2 * lane : 0;              // clamped column (inactive lanes read valid memory)
  const bool per = b.bc == PX_BC_PERIODIC, refl = b.bc == PX_BC_DIRICHLET_CC, fixed = b.bc == PX_BC_FIXED_GHOSTS;
  const int srcW = lane == 0 ? np - 1 : lane - 1, srcE = lane >= np - 1 ? 0 : lane + 1;
  const bool edgeW = lane == 0, edgeE = lane == np - 1;
  double2 cur[RW], rho[RW];
  double gW[RW], gE[RW];
#pragma unroll
  for (int j = 0; j < RW; ++j) {
    const int y = y0 + j;
    cur[j] = rho[j] = make_double2(0.0, 0.0);
    gW[j] = gE[j] = 0.0;
    if (act) {
      const double* src = b.phi_in + (int64_t)y * b.ld_in + xs;
      cur[j] = make_double2(src[0], src[1]);
      const double* f = b.rhs + (int64_t)y * b.ld_rhs + xs;
      rho[j] = make_double2(f[0], f[1]);
      if (fixed) {
        gW[j] = b.phi_in[(int64_t)y * b.ld_in - 1];
        gE[j] = b.phi_in[(int64_t)y * b.ld_in + nx];
      }
    }
  }
  // fixed ghost rows (both buffers) and corners
  if (fixed) {
    for (int i = tid; i < nx; i += BW_THREADS) {
      const double lo = b.phi_in[-b.ld_in + i], hi = b.phi_in[(int64_t)ny * b.ld_in + i];
      board[i] = board[bsz + i] = lo;
      board[(size_t)(ny + 1) * nx + i] = board[bsz + (size_t)(ny + 1) * nx + i] = hi;
    }
    if (tid == 0) {
      gcor[0] = b.phi_in[-b.ld_in - 1];
      gcor[1] = b.phi_in[-b.ld_in + nx];
      gcor[2] = b.phi_in[(int64_t)ny * b.ld_in - 1];
      gcor[3] = b.phi_in[(int64_t)ny * b.ld_in + nx];
    }
  }
  // board row Y (-1 .. ny) of buffer bb := v, locally and, when Y is a halo
  // row of a neighbouring CTA of the cluster, in that CTA's board too
  auto put = [&](double* B, int Y, double2 v) {
    double* q = B + (size_t)(Y + 1) * nx + xs;
    *reinterpret_cast<double2*>(q) = v;
    if (CL > 1) {
      const int up = cr > 0 ? cr - 1 : CL - 1, dn = cr < CL - 1 ? cr + 1 : 0;
      // Y read as a halo row by CTA t: Y == t·nyl - 1 or Y == (t+1)·nyl
      const uint64_t* bar = &hb[B == board ? 0 : 1];
      if (up != cr && (Y == up * nyl - 1 || Y == (up + 1) * nyl)) {
        if (mb) bw_st_async(q, (unsigned)up, v, bar);
        else bw_st_remote(q, (unsigned)up, v);
      }
      if (dn != cr && dn != up && (Y == dn * nyl - 1 || Y == (dn + 1) * nyl)) {
        if (mb) bw_st_async(q, (unsigned)dn, v, bar);
        else bw_st_remote(q, (unsigned)dn, v);
      }
    }
  };
  // the warp's first and last rows (and the y images at the faces) into board buffer bb
  auto post = [&](int bb) {
    if (!act) return;
    double* B = board + (size_t)bb * bsz;
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      if (j != 0 && j != RW - 1) continue;
      const int y = y0 + j;
      put(B, y, cur[j]);
      if (y == 0 && !fixed) {
        if (per) put(B, ny, cur[j]);
        else put(B, -1, make_double2(-cur[j].x, -cur[j].y));
      }
      if (y == ny - 1 && !fixed) {
        if (per) put(B, -1, cur[j]);
        else put(B, ny, make_double2(-cur[j].x, -cur[j].y));
      }
    }
  };
  // mb: the halo rows another CTA writes arrive by st.async, counted on the
  // board buffer's mbarrier; the warps that read them wait for its phase, the
  // others only need the CTA barrier (no cluster barrier per sweep)
  const bool up_remote = CL > 1 && (cr > 0 || per), dn_remote = CL > 1 && (cr < CL - 1 || per);
  const uint32_t E = (uint32_t)((up_remote ? 1 : 0) + (dn_remote ? 1 : 0)) * (uint32_t)np * 16u;
  const bool waiter = mb && CL > 1 && wact && (warp == 0 || (warp + 1) * RW >= nyl);
  uint32_t ph[2] = {0u, 0u};
  if (CL > 1 && mb) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&hb[0])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&hb[1])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int k = 0; k < 2; ++k)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&hb[k])),
                     "r"(E)
                     : "memory");
    }
    bw_cluster_sync();  // every CTA's barriers armed before any st.async
  }
  auto halo_wait = [&](int bb, bool rearm) {
    if (!waiter) return;
    bw_mbar_wait(&hb[bb], ph[bb]);
    ph[bb] ^= 1u;
    if (rearm && tid == 0)  // the next use of this buffer (two sweeps on)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&hb[bb])),
                   "r"(E)
                   : "memory");
  };
  post(0);
  if (CL > 1 && !mb) bw_cluster_sync();
  else __syncthreads();
  // W of column 2l / E of column 2l+1 of a row v (gw / ge: its fixed ghosts)
  auto west = [&](double2 v, double gw) -> double {
    const double sh = __shfl_sync(FULL_MASK, v.y, srcW);
    return edgeW && !per ? (refl ? -v.x : gw) : sh;
  };
  auto east = [&](double2 v, double ge) -> double {
    const double sh = __shfl_sync(FULL_MASK, v.x, srcE);
    return edgeE && !per ? (refl ? -v.y : ge) : sh;
  };
  // fixed ghost columns of the board rows next to the group (rows y0-1 and
  // y0+RW lie in the domain or its ghost ring)
  double gWs = 0.0, gEs = 0.0, gWn = 0.0, gEn = 0.0;
  if (fixed && wact) {
    gWs = b.phi_in[(int64_t)(y0 - 1) * b.ld_in - 1];
    gEs = b.phi_in[(int64_t)(y0 - 1) * b.ld_in + nx];
    gWn = b.phi_in[(int64_t)(y0 + RW) * b.ld_in - 1];
    gEn = b.phi_in[(int64_t)(y0 + RW) * b.ld_in + nx];
  }
  auto update = [&](double2 S, double2 C, double2 N, double2 f, double sw_g, double se_g, double cw_g, double ce_g,
                    double nw_g, double ne_g, double2& res) -> double2 {
    const double cw = west(C, cw_g), ce = east(C, ce_g);
    double sw = 0.0, se = 0.0, nw = 0.0, ne = 0.0;
    if (ST) {
      sw = west(S, sw_g);
      se = east(S, se_g);
      nw = west(N, nw_g);
      ne = east(N, ne_g);
    }
    double2 o;
    if (P2) {
      const double L0 = fma(-4.0, C.x, __dadd_rn(__dadd_rn(__dadd_rn(cw, C.y), S.x), N.x));
      const double L1 = fma(-4.0, C.y, __dadd_rn(__dadd_rn(__dadd_rn(C.x, ce), S.y), N.y));
      res.x = fma(b.scale, L0, -f.x);
      res.y = fma(b.scale, L1, -f.y);
      o = make_double2(fma(b.lambda, res.x, C.x), fma(b.lambda, res.y, C.y));
    } else {
      const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
      const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
      res.x = __dsub_rn(__dmul_rn(b.scale, L0), f.x);
      res.y = __dsub_rn(__dmul_rn(b.scale, L1), f.y);
      o = make_double2(__dadd_rn(C.x, __dmul_rn(b.lambda, res.x)), __dadd_rn(C.y, __dmul_rn(b.lambda, res.y)));
    }
    if (!act) res = make_double2(0.0, 0.0);
    return o;
  };
  // max|r| by fmax (exact: one of its operands; a NaN r is restored from
  // Σr², which it makes NaN), Σr² by fused multiply-add
  auto acc = [&](double2 res, double& mx, double& ss) {
    mx = fmax(mx, fabs(res.x));
    ss = fma(res.x, res.x, ss);
    mx = fmax(mx, fabs(res.y));
    ss = fma(res.y, res.y, ss);
  };
  // warp partial: the max as two 32-bit redux.sync steps over the bit pattern
  // (high word, then the low word among the lanes holding the high maximum),
  // Σ by a fixed butterfly
  auto warp_partial = [&](double mxd, double ss, int e, bool store) {
    const unsigned long long mb =
        isnan(ss) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(mxd);
    const unsigned hi = (unsigned)(mb >> 32);
    const unsigned mhi = __reduce_max_sync(FULL_MASK, hi);
    const unsigned mlo = __reduce_max_sync(FULL_MASK, hi == mhi ? (unsigned)mb : 0u);
    for (int o = 16; o > 0; o >>= 1) ss = ss + __shfl_xor_sync(FULL_MASK, ss, o);
    if (store && lane == 0) {
      part[((size_t)e * BW_WARPS + warp) * 2] = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
      part[((size_t)e * BW_WARPS + warp) * 2 + 1] = ss;
    }
  };
  // one pass over the group's rows of buffer bb's iterate: WRITE = update
  // (the new rows replace cur), else residuals only
  auto pass = [&](int bb, bool write, bool rec, double& mx, double& ss) {
    const double* B = board + (size_t)bb * bsz;
    const double2 s_row = *reinterpret_cast<const double2*>(B + (size_t)y0 * nx + xs);        // row y0 - 1
    const double2 n_row = *reinterpret_cast<const double2*>(B + (size_t)(y0 + RW + 1) * nx + xs);  // row y0 + RW
    double2 o[RW];
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      const double2 S = j == 0 ? s_row : cur[j - 1];
      const double2 N = j == RW - 1 ? n_row : cur[j + 1];
      const double sg_w = j == 0 ? gWs : gW[j - 1], sg_e = j == 0 ? gEs : gE[j - 1];
      const double ng_w = j == RW - 1 ? gWn : gW[j + 1], ng_e = j == RW - 1 ? gEn : gE[j + 1];
      double2 res;
      o[j] = update(S, cur[j], N, rho[j], sg_w, sg_e, gW[j], gE[j], ng_w, ng_e, res);
      if (rec) acc(res, mx, ss);
    }
    if (write)
#pragma unroll
      for (int j = 0; j < RW; ++j) cur[j] = o[j];
  };
  // a recorded sweep's warp reduction runs after the barrier, overlapping the
  // next sweep's loads and shuffles (it is off the sweep-to-sweep chain)
  int entry = 0, phase = 0;
  bool pend = false;
  double pmx = 0.0, pss = 0.0;
  for (int s = 0; s < b.nsweeps; ++s) {
    const bool rec = b.every > 0 && phase == 0;
    if (++phase == b.every) phase = 0;
    if (wact) {
      // the previous recorded sweep's reduction in the same block as this
      // sweep's update (the compiler interleaves the two chains)
      warp_partial(pmx, pss, entry - 1, pend);
      double mx = 0.0, ss = 0.0;
      halo_wait(s & 1, true);
      pass(s & 1, true, rec, mx, ss);
      post((s + 1) & 1);
      pend = rec;
      pmx = mx;
      pss = ss;
    } else if (rec && lane == 0) {
      part[((size_t)entry * BW_WARPS + warp) * 2] = 0.0;
      part[((size_t)entry * BW_WARPS + warp) * 2 + 1] = 0.0;
    }
    if (rec) ++entry;
    if (CL > 1 && !mb) bw_cluster_sync();
    else __syncthreads();
  }
  if (wact) warp_partial(pmx, pss, entry - 1, pend);
  const int bN = b.nsweeps & 1;
  halo_wait(bN, false);  // φ^N's remote halo rows (final residual, ghost rows)
  __syncthreads();
  if (b.final_norm) {
    if (wact) {
      double mx = 0.0, ss = 0.0;
      pass(bN, false, true, mx, ss);
      warp_partial(mx, ss, entry, true);
    } else if (lane == 0) {
      part[((size_t)entry * BW_WARPS + warp) * 2] = 0.0;
      part[((size_t)entry * BW_WARPS + warp) * 2 + 1] = 0.0;
    }
    ++entry;
  }
  if (CL > 1) bw_cluster_sync();
  else __syncthreads();
  // entries over the warps (of CTA 0, 1, .. of the cluster) in fixed order, by CTA 0
  if (cr == 0)
    for (int e = tid; e < entry; e += BW_THREADS) {
      unsigned long long m = 0ull;
      double t = 0.0;
      for (int k = 0; k < CL * BW_WARPS; ++k) {
        const double* pp = part + ((size_t)e * BW_WARPS + (k % BW_WARPS)) * 2;
        const double2 v = CL > 1 ? bw_ld_remote(pp, (unsigned)(k / BW_WARPS)) : *reinterpret_cast<const double2*>(pp);
        m = umax64(m, (unsigned long long)__double_as_longlong(v.x));
        t = k ? __dadd_rn(t, v.y) : v.y;
      }
      b.d_max[e] = __longlong_as_double((long long)m);
      b.d_sum[e] = t;
    }
  // φ^N with its ghost ring: own rows (+ ghost columns = the W/E images), and
  // warp 0 the ghost rows -1 / ny from the board (+ the corners)
  if (wact) {
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      const double w = west(cur[j], gW[j]), e = east(cur[j], gE[j]);
      if (act) {
        double* dst = b.phi_out + (int64_t)(y0 + j) * b.ld_out + xs;
        dst[0] = cur[j].x;
        dst[1] = cur[j].y;
        if (edgeW) dst[-1] = w;
        if (edgeE) dst[2] = e;
      }
    }
  }
  if (warp == 0) {
    const double* B = board + (size_t)bN * bsz;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if ((k == 0 && cr != 0) || (k == 1 && cr != CL - 1)) continue;  // the face CTAs hold the ghost rows
      const int y = k ? ny : -1;
      const double2 v = *reinterpret_cast<const double2*>(B + (size_t)(y + 1) * nx + xs);
      const double w = west(v, gcor[2 * k]), e = east(v, gcor[2 * k + 1]);
      if (lane < np) {
        double* dst = b.phi_out + (int64_t)y * b.ld_out + xs;
        dst[0] = v.x;
        dst[1] = v.y;
        if (edgeW) dst[-1] = w;
        if (edgeE) dst[2] = e;
      }
    }
  }
  if (CL > 1) bw_cluster_sync();  // no CTA leaves while CTA 0 may still read its partials
}

static size_t bw_smem(const SmallBox& b, int n_entries) {
  return ((size_t)2 * (b.ny + 2) * b.nx + (size_t)n_entries * BW_WARPS * 2 + 4) * sizeof(double);
}
static bool bw_pow2(double v) {
  if (!(v > 0.0) || !std::isfinite(v)) return false;
  int e;
  return std::frexp(v, &e) == 0.5;
}
// PROTOX_BOXW_MB=0 (read once, A/B): the cluster k_boxw exchanges its halo
// rows with plain DSMEM stores and a cluster barrier per sweep instead of
// st.async counted on per-buffer mbarriers
static int bw_mb_env() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("PROTOX_BOXW_MB");
    m = (e && e[0] == '0') ? 0 : 1;
  }
  return m;
}
template <int RW, int CL>
static cudaError_t bw_launch(const SmallBox& b, int ne, size_t smem, cudaStream_t s) {
  const bool p2 = b.stencil == 0 && bw_pow2(b.scale) && bw_pow2(b.lambda);
  void (*fn)(const SmallBox, int, int) =
      b.stencil ? k_boxw<1, false, RW, CL> : (p2 ? k_boxw<0, true, RW, CL> : k_boxw<0, false, RW, CL>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  if (CL > 8) {  // 16 CTAs: a non-portable cluster size
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (CL == 1) {
    fn<<<1, BW_THREADS, smem, s>>>(b, ne, 0);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(BW_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, b, ne, bw_mb_env());
}
template <int CL>
static cudaError_t bw_launch_rw(const SmallBox& b, int rw, int ne, size_t smem, cudaStream_t s) {
  return rw == 1 ? bw_launch<1, CL>(b, ne, smem, s)
                 : (rw == 2 ? bw_launch<2, CL>(b, ne, smem, s) : bw_launch<4, CL>(b, ne, smem, s));
}
// CTAs of the k_boxw cluster (PROTOX_BOXW_CL = 1, 2, 4, 8 or 16, read once; the box
// rows must split evenly)
static int bw_cl_env() {
  static int c = -1;
  if (c < 0) {
    const char* e = getenv("PROTOX_BOXW_CL");
    c = e ? atoi(e) : BW_CL_DEFAULT;
    if (c != 1 && c != 2 && c != 4 && c != 8 && c != 16) c = BW_CL_DEFAULT;
  }
  return c;
}

size_t smallbox_smem(int nx, int ny) {
  return ((size_t)2 * (nx + 2) * (ny + 2) + (size_t)nx * ny) * sizeof(double);
}

bool smallbox_fits(int nx, int ny) { return nx >= 1 && ny >= 1 && smallbox_smem(nx, ny) <= 200 * 1024; }

px_status launch_smallbox(const SmallBox& b, cudaStream_t s) {
  // 16+ rows: spread the box over a cluster of 8 SMs (px_cluster.cu): one SM
  // running k_box1 is issue-bound (73 % issue-active at 1.76 µs per 64² sweep)
  if (box1_mode() == 0 && b.g == 1) {
    int cl = bw_cl_env();
    while (cl > 1 && (b.ny % cl || bw_rows_per_warp(b.nx, b.ny / cl) == 0)) cl /= 2;
    const int rw = bw_rows_per_warp(b.nx, b.ny / cl);
    const int ne = box1_entries(b) > 0 ? box1_entries(b) : 1;
    const size_t smem = bw_smem(b, ne);
    if (rw > 0 && smem <= 200 * 1024) {
      const cudaError_t e = cl == 1   ? bw_launch_rw<1>(b, rw, ne, smem, s)
                            : cl == 2 ? bw_launch_rw<2>(b, rw, ne, smem, s)
                            : cl == 4 ? bw_launch_rw<4>(b, rw, ne, smem, s)
                            : cl == 8 ? bw_launch_rw<8>(b, rw, ne, smem, s)
                                      : bw_launch_rw<16>(b, rw, ne, smem, s);
      note_kernel("k_boxw");
      count_launches(1);
      return cuda_check(e, "small-box kernel launch");
    }
  }
  if ((box1_mode() == 0 || box1_mode() == 3) && cluster_box_eligible(b)) return launch_cluster_box(b, s);
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
