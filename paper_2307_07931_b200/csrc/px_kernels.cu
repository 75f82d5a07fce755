// px_kernels.cu -- the hot path of libprotox: one fused, register-streaming
// pass per sweep of
//     L   = S(φ)                 5-point (Eq.1, taps P:198) or 9-point
//     r   = scale·L − rhs        residual (Eq.7)
//     φ'  = φ + λ·r              point-Jacobi update (Eq.3)
//     max|r|, Σr²                norms, warp-shuffle + fixed-order
//                                block/grid reduction
// plus the fused ghost images of the new iterate (exchange).
//
// Design: the sweep is HBM-bound (24 B/cell-update: read φ,
// read rhs, write φ'), so the kernel streams each array through the SM once.
// A warp owns a 64-column strip (lane = 2 adjacent cells, 16-byte ld/st.v2.f64)
// and walks down SW_ROWS rows keeping the rows S, C, N in registers; W/E
// neighbours come from the adjacent lane by __shfl (lanes 0/31 load the one
// halo cell).  Loads are issued SW_PF rows ahead of use so each thread keeps
// several 16-byte requests in flight.  Every cell is evaluated with the
// oracle's expression tree, each * and + rounded separately (__dmul_rn /
// __dadd_rn), so results are bit-identical to oracle/ for any h and λ.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include <cooperative_groups.h>

#include "px_internal.h"
#include "px_device.cuh"

namespace cg = cooperative_groups;

namespace px {

constexpr int SW_WARPS = 8;
constexpr int SW_THREADS = SW_WARPS * 32;
constexpr int SW_COLS = SW_WARPS * 64;
constexpr int SW_ROWS = 32;
constexpr int SW_PF = 4;                  // prefetch distance in rows (= ring slots)
constexpr unsigned FULL = 0xffffffffu;

static int ldg_nsm() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// Rows per CTA: SW_ROWS, reduced in steps of SW_PF (down to SW_PF) until the
// grid has >= 4 CTAs per SM -- small (L2-resident) problems such as 1024²
// would otherwise leave most SMs idle.
static int32_t ldg_rows(int32_t nx, int32_t ny, int32_t phase) {
  const int64_t gx = (nx + phase + SW_COLS - 1) / SW_COLS;
  const int64_t target = 4 * (int64_t)ldg_nsm();
  int32_t rows = SW_ROWS;
  while (rows > SW_PF && gx * ((ny + rows - 1) / rows) < target) rows -= SW_PF;
  return rows;
}

static int32_t ldg_blocks(int32_t nx, int32_t ny, int32_t phase) {
  if (nx <= 0 || ny <= 0) return 0;
  const int32_t rows = ldg_rows(nx, ny, phase);
  return ((nx + phase + SW_COLS - 1) / SW_COLS) * ((ny + rows - 1) / rows);
}

// upper bound of the blocks any relax/residual launch over the region uses
// (sizes norm buffers; host-only: no device query)
int32_t stream_blocks(int32_t nx, int32_t ny, int32_t phase) {
  if (nx <= 0 || ny <= 0) return BULK_MAX_GRID;
  const int32_t b = ((nx + phase + SW_COLS - 1) / SW_COLS) * ((ny + SW_PF - 1) / SW_PF);
  return b > BULK_MAX_GRID ? b : BULK_MAX_GRID;
}

int32_t launch_blocks(int mode, const StreamLaunch& a) {
  if (bulk_eligible(mode, a)) return bulk_blocks(a);
  return ldg_blocks(a.nx, a.ny, a.phase);
}

// --------------------------------------------------------------- helpers
struct Raw {            // a row as loaded: the lane's pair plus its halo cell
  double a, b, h;       // h: column c-1 on lane 0, c+2 on lane 31
};
struct Fin {            // a row after the neighbour exchange
  double w, a, b, e;    // columns c-1, c, c+1, c+2
};

__device__ __forceinline__ Raw load_raw(const double* __restrict__ row, int c, int lane, int x0,
                                        int x1) {
  Raw v;
  if (c >= x0 && c + 1 <= x1) {
    double2 p = __ldg(reinterpret_cast<const double2*>(row + c));
    v.a = p.x;
    v.b = p.y;
  } else {
    v.a = (c >= x0 && c <= x1) ? __ldg(row + c) : 0.0;
    v.b = (c + 1 >= x0 && c + 1 <= x1) ? __ldg(row + c + 1) : 0.0;
  }
  v.h = 0.0;
  if (lane == 0) {
    if (c - 1 >= x0 && c - 1 <= x1) v.h = __ldg(row + c - 1);
  } else if (lane == 31) {
    if (c + 2 >= x0 && c + 2 <= x1) v.h = __ldg(row + c + 2);
  }
  return v;
}

__device__ __forceinline__ Fin finish(const Raw& v, int lane) {
  Fin f;
  f.a = v.a;
  f.b = v.b;
  double w = __shfl_up_sync(FULL, v.b, 1);
  double e = __shfl_down_sync(FULL, v.a, 1);
  f.w = (lane == 0) ? v.h : w;
  f.e = (lane == 31) ? v.h : e;
  return f;
}

// Undivided stencil sums for the two cells of a lane, tap order fixed
// (R10):  5-point  W, E, S, N, C(-4);
//                   9-point  W, E, S, N (4), SW, SE, NW, NE (1), C(-20).
template <int ST>
__device__ __forceinline__ void taps(const Fin& S, const Fin& C, const Fin& N, double& L0,
                                     double& L1) {
  if (ST == 0) {
    L0 = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(C.w, C.b), S.a), N.a), __dmul_rn(-4.0, C.a));
    L1 = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(C.a, C.e), S.b), N.b), __dmul_rn(-4.0, C.b));
  } else {
    double t;
    t = __dmul_rn(4.0, C.w);
    t = __dadd_rn(t, __dmul_rn(4.0, C.b));
    t = __dadd_rn(t, __dmul_rn(4.0, S.a));
    t = __dadd_rn(t, __dmul_rn(4.0, N.a));
    t = __dadd_rn(t, S.w);
    t = __dadd_rn(t, S.b);
    t = __dadd_rn(t, N.w);
    t = __dadd_rn(t, N.b);
    L0 = __dadd_rn(t, __dmul_rn(-20.0, C.a));
    t = __dmul_rn(4.0, C.a);
    t = __dadd_rn(t, __dmul_rn(4.0, C.e));
    t = __dadd_rn(t, __dmul_rn(4.0, S.b));
    t = __dadd_rn(t, __dmul_rn(4.0, N.b));
    t = __dadd_rn(t, S.a);
    t = __dadd_rn(t, S.e);
    t = __dadd_rn(t, N.a);
    t = __dadd_rn(t, N.e);
    L1 = __dadd_rn(t, __dmul_rn(-20.0, C.b));
  }
}

// ------------------------------------------------------- the stream kernel
// One tile (column group bx x row chunk by) of a sweep; accumulates the
// residual norms of the tile's cells into mx / ss.
template <int MODE, int ST>
__device__ __forceinline__ void stream_tile(const StreamLaunch& a, const int bx, const int by, const int rows,
                                            unsigned long long& mx, double& ss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = -a.phase + (bx * SW_WARPS + warp) * 64 + 2 * lane;
  const int r0 = by * rows;
  const int rend = min(a.ny, r0 + rows);      // rows computed: [r0, rend)
  const int rlast = rend;                      // last φ row needed (N of rend-1)
  const bool need_rhs = (MODE == MODE_RELAX || MODE == MODE_RESID);
  const bool warp_live = (-a.phase + (int)(bx * SW_WARPS + warp) * 64) < a.nx;

  if (warp_live) {
    // Ring of SW_PF raw φ rows and SW_PF rhs rows in flight.  φ row
    // r0-1+q lives in slot q % SW_PF; a slot is refilled right after the
    // row in it has been consumed (finish-then-load), so SW_PF loads of each
    // array are always outstanding.  The row loop is unrolled by SW_PF only
    // (slot indices stay compile-time; code stays small for the I-cache).
    Raw raw[SW_PF];
    double2 rr[SW_PF];
    auto load_rhs = [&](int r) {
      const double* q = a.rhs + (int64_t)r * a.ld_rhs;
      if (c >= 0 && c + 1 < a.nx) return __ldcs(reinterpret_cast<const double2*>(q + c));
      return make_double2((c >= 0 && c < a.nx) ? __ldcs(q + c) : 0.0,
                          (c + 1 >= 0 && c + 1 < a.nx) ? __ldcs(q + c + 1) : 0.0);
    };
    raw[0] = load_raw(a.src + (int64_t)(r0 - 1) * a.ld_src, c, lane, a.src_x0, a.src_x1);
    raw[1] = load_raw(a.src + (int64_t)r0 * a.ld_src, c, lane, a.src_x0, a.src_x1);
    Fin fS = finish(raw[0], lane);
    Fin fC = finish(raw[1], lane);
#pragma unroll
    for (int q = 2; q < SW_PF + 2; ++q) {
      const int r = r0 - 1 + q;
      if (r <= rlast) raw[q % SW_PF] = load_raw(a.src + (int64_t)r * a.ld_src, c, lane, a.src_x0, a.src_x1);
    }
    if (need_rhs) {
#pragma unroll
      for (int k = 0; k < SW_PF; ++k)
        if (r0 + k < rend) rr[k] = load_rhs(r0 + k);
    }

#pragma unroll 1
    for (int i0 = 0; i0 < rows; i0 += SW_PF) {
#pragma unroll
    for (int jj = 0; jj < SW_PF; ++jj) {
      const int i = i0 + jj;
      const int r = r0 + i;
      if (r >= rend) break;
      // row N = φ row r+1 (slot (i+2) % SW_PF), then refill that slot
      const Fin fN = finish(raw[(jj + 2) % SW_PF], lane);
      {
        const int rp = r + 1 + SW_PF;
        if (rp <= rlast)
          raw[(jj + 2) % SW_PF] = load_raw(a.src + (int64_t)rp * a.ld_src, c, lane, a.src_x0, a.src_x1);
      }
      double2 f = make_double2(0.0, 0.0);
      if (need_rhs) {
        f = rr[jj];
        if (r + SW_PF < rend) rr[jj] = load_rhs(r + SW_PF);
      }
      double L0, L1;
      taps<ST>(fS, fC, fN, L0, L1);
      const bool va = (c >= 0 && c < a.nx), vb = (c + 1 >= 0 && c + 1 < a.nx);
      double o0 = 0.0, o1 = 0.0;
      if (MODE == MODE_RELAX || MODE == MODE_RESID) {
        const double d0 = __dmul_rn(a.scale, L0), d1 = __dmul_rn(a.scale, L1);
        const double e0 = __dsub_rn(d0, f.x), e1 = __dsub_rn(d1, f.y);
        if (va) {
          mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(e0)));
          ss = fma(e0, e0, ss);
        }
        if (vb) {
          mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(e1)));
          ss = fma(e1, e1, ss);
        }
        if (MODE == MODE_RELAX) {
          o0 = __dadd_rn(fC.a, __dmul_rn(a.lambda, e0));
          o1 = __dadd_rn(fC.b, __dmul_rn(a.lambda, e1));
        }
      } else if (MODE == MODE_APPLY) {
        o0 = __dmul_rn(a.scale, L0);
        o1 = __dmul_rn(a.scale, L1);
      } else {  // MODE_MRHS: f = ρ + c12·S5(ρ)
        o0 = __dadd_rn(fC.a, __dmul_rn(a.scale, L0));
        o1 = __dadd_rn(fC.b, __dmul_rn(a.scale, L1));
      }
      if (MODE != MODE_RESID) {
        double* dp = a.dst + (int64_t)r * a.ld_dst;
        if (va && vb) {
          *reinterpret_cast<double2*>(dp + c) = make_double2(o0, o1);
        } else {
          if (va) dp[c] = o0;
          if (vb) dp[c + 1] = o1;
        }
        if (MODE == MODE_RELAX && a.gs.g > 0) {
          if (va) images(a, c, r, o0);
          if (vb) images(a, c + 1, r, o1);
        }
      }
      fS = fC;
      fC = fN;
    }
    }
  }
}

template <int MODE, int ST>
__global__ void __launch_bounds__(SW_THREADS, 2) k_stream(const StreamLaunch a, const int rows) {
  unsigned long long mx = 0ull;
  double ss = 0.0;
  stream_tile<MODE, ST>(a, blockIdx.x, blockIdx.y, rows, mx, ss);
  if (MODE == MODE_RELAX || MODE == MODE_RESID) {
    if (a.norms.out_max) reduce_norms(a.norms, mx, ss);
  }
}

// Block 0 reduces n per-CTA partials in fixed order into *out_max / *out_sum.
__device__ void reduce_partials(const double* part, int n, double* out_max, double* out_sum,
                                unsigned long long* s_mx, double* s_ss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long m = 0ull;
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    m = umax64(m, (unsigned long long)__double_as_longlong(__ldcg(part + 2 * i)));
    t = t + __ldcg(part + 2 * i + 1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = umax64(m, __shfl_xor_sync(FULL_MASK, m, o));
    t = t + __shfl_xor_sync(FULL_MASK, t, o);
  }
  if (lane == 0) {
    s_mx[warp] = m;
    s_ss[warp] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    m = s_mx[0];
    t = s_ss[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      m = umax64(m, s_mx[w]);
      t = t + s_ss[w];
    }
    *out_max = __longlong_as_double((long long)m);
    *out_sum = t;
  }
  __syncthreads();
}

// ------------------------------------------- persistent whole-solve kernel
// All sweeps of a single-rank solve in ONE cooperative launch (C2-sized,
// L2-resident problems, where one launch per sweep is latency): each CTA
// sweeps its tiles, then the grid synchronises (the fused ghost images of
// the new iterate become visible) and the two buffers swap.  Norms of a
// recorded sweep: each CTA's fixed-order partial, then CTA 0 reduces them in
// fixed order after the barrier (partials double-buffered by entry parity).
template <int ST>
__global__ void __launch_bounds__(SW_THREADS, 2) k_persist(const PersistLaunch p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long s_mx[32];
  __shared__ double s_ss[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ntiles = p.gx * p.gy;
  auto block_partial = [&](unsigned long long mx, double ss, double* part) {
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
      double t = s_ss[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        m = umax64(m, s_mx[w]);
        t = t + s_ss[w];
      }
      part[2 * blockIdx.x] = __longlong_as_double((long long)m);
      part[2 * blockIdx.x + 1] = t;
    }
    __syncthreads();
  };
  int entry = 0;
  for (int s = 0; s < p.nsweeps; ++s) {
    const StreamLaunch& a = (s & 1) ? p.a1 : p.a0;
    const bool rec = p.every > 0 && s % p.every == 0;
    unsigned long long mx = 0ull;
    double ss = 0.0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) stream_tile<MODE_RELAX, ST>(a, t % p.gx, t / p.gx, p.rows, mx, ss);
    double* part = p.partials + (size_t)(entry & 1) * 2 * gridDim.x;
    if (rec) block_partial(mx, ss, part);
    grid.sync();
    if (rec) {
      if (blockIdx.x == 0) reduce_partials(part, gridDim.x, p.d_max + entry, p.d_sum + entry, s_mx, s_ss);
      ++entry;
    }
  }
  if (p.final_norm) {
    const StreamLaunch& a = (p.nsweeps & 1) ? p.r1 : p.r0;
    unsigned long long mx = 0ull;
    double ss = 0.0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) stream_tile<MODE_RESID, ST>(a, t % p.gx, t / p.gx, p.rows, mx, ss);
    double* part = p.partials + (size_t)(entry & 1) * 2 * gridDim.x;
    block_partial(mx, ss, part);
    grid.sync();
    if (blockIdx.x == 0) reduce_partials(part, gridDim.x, p.d_max + entry, p.d_sum + entry, s_mx, s_ss);
  }
}

static int64_t g_launches = 0;
void count_launches(int64_t n) { g_launches += n; }

// names of the sweep kernels enqueued since the last take (px_last_solve_kernels)
static thread_local std::string tl_kernels;
void note_kernel(const char* name) {
  if (tl_kernels.find(name) != std::string::npos) return;
  if (!tl_kernels.empty()) tl_kernels += "+";
  tl_kernels += name;
}
std::string take_noted_kernels() {
  std::string s;
  s.swap(tl_kernels);
  return s;
}

px_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PX_OK;
  return fail(PX_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

template <int MODE, int ST>
static void launch_t(const StreamLaunch& a, dim3 grid, cudaStream_t s) {
  k_stream<MODE, ST><<<grid, SW_THREADS, 0, s>>>(a, ldg_rows(a.nx, a.ny, a.phase));
}

px_status launch_stream(int mode, int stencil, const StreamLaunch& a, cudaStream_t s) {
  if (a.nx <= 0 || a.ny <= 0) return PX_OK;
  if (bulk_eligible(mode, a)) return launch_bulk(mode, stencil, a, s);
  if (a.ps.on) return fail(PX_ERR_UNSUPPORTED, "peer-memory push needs the TMA kernel (even width, aligned rows)");
  return launch_stream_ldg(mode, stencil, a, s);
}

int32_t stream_launch_blocks_ldg(const StreamLaunch& a) { return ldg_blocks(a.nx, a.ny, a.phase); }

// ---- fused halo push over peer memory: per-solve helpers (px_solve P2P mode)
__global__ void k_wait(const PushSpec ps) {
  if (ps.rel)  // the previous kernel (the last sweep) has completed: its pushes are performed
    for (int side = 0; side < 2; ++side)
      if (ps.rflag[side])
        asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(ps.rflag[side]), "l"(1ull) : "memory");
  const unsigned long long target = *ps.epoch + ps.wcount;
  for (int side = 0; side < 2; ++side)
    if (ps.wflag[side]) px_spin_until(ps.wflag[side], target, ps.err);
}
// e[0] = arrival base of this solve, e[1] = arrivals per side of the previous
// solve: every solve adds its own count, so solves of different lengths mix.
__global__ void k_epoch_bump(unsigned long long* e, unsigned long long per_solve) {
  e[0] += e[1];
  e[1] = per_solve;
}

// φ^0's boundary rows (full padded rows) into both buffers of each neighbour.
// CTA b copies a column slice of every row; then it counts one arrival per
// side (PX_PUSH_INIT_CTAS arrivals per side in all).
__global__ void __launch_bounds__(256) k_push_init(const PushInit pi) {
  const int per = (pi.row_len + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per, i1 = min(pi.row_len, i0 + per);
  for (int side = 0; side < 2; ++side) {
    const double* src = side ? pi.src_hi : pi.src_lo;
    for (int b = 0; b < 2; ++b) {
      double* dst = pi.dst[side][b];
      if (!dst) continue;
      for (int r = 0; r < pi.g; ++r)
        for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x)
          dst[(int64_t)r * pi.ld + i] = src[(int64_t)r * pi.ld + i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int side = 0; side < 2; ++side)
      if (pi.rflag[side])
        asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(pi.rflag[side]), "l"(1ull) : "memory");
  }
}

// Norm all-reduce over peer memory (PeerAllreduce, px_internal.h); one CTA.
__global__ void __launch_bounds__(256) k_peer_allreduce(const PeerAllreduce ar) {
  __shared__ unsigned long long q;
  const int P = ar.nranks;
  for (int c0 = 0; c0 < ar.n; c0 += PX_MBOX_ENTRIES) {
    const int m = min(PX_MBOX_ENTRIES, ar.n - c0);
    if (threadIdx.x == 0) q = ++*ar.round;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      ar.mbox_own[2 * i] = ar.d_max[c0 + i];
      ar.mbox_own[2 * i + 1] = ar.d_sum[c0 + i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int p = 0; p < P; ++p)
        if (p != ar.rank)
          asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(ar.arrive[p]), "l"(1ull) : "memory");
      px_spin_until(ar.own_arrive, q * (unsigned long long)(P - 1), ar.err);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      // every rank combines the mailboxes in rank order: identical bits everywhere
      unsigned long long mx = 0ull;
      double ss = 0.0;
      for (int p = 0; p < P; ++p) {
        const double* mb = ar.mbox[p];
        const double vm = __ldcv(mb + 2 * i), vs = __ldcv(mb + 2 * i + 1);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(vm);
        mx = bits > mx ? bits : mx;  // |r| >= 0 (or NaN, sign clear): the bit order is the value order
        ss = p == 0 ? vs : __dadd_rn(ss, vs);
      }
      ar.d_max[c0 + i] = __longlong_as_double((long long)mx);
      ar.d_sum[c0 + i] = ss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // every peer has read this mailbox before the next round rewrites it
      __threadfence_system();
      for (int p = 0; p < P; ++p)
        if (p != ar.rank)
          asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(ar.done[p]), "l"(1ull) : "memory");
      px_spin_until(ar.own_done, q * (unsigned long long)(P - 1), ar.err);
    }
    __syncthreads();
  }
}

px_status launch_wait(const PushSpec& ps, cudaStream_t s) {
  k_wait<<<1, 1, 0, s>>>(ps);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "wait kernel launch");
}

px_status launch_push_init(const PushInit& pi, cudaStream_t s) {
  k_push_init<<<PX_PUSH_INIT_CTAS, 256, 0, s>>>(pi);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "push-init kernel launch");
}

px_status launch_peer_allreduce(const PeerAllreduce& ar, cudaStream_t s) {
  if (ar.n <= 0 || ar.nranks <= 1) return PX_OK;
  k_peer_allreduce<<<1, 256, 0, s>>>(ar);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "peer all-reduce kernel launch");
}

px_status launch_epoch_bump(unsigned long long* epoch, unsigned long long per_solve, cudaStream_t s) {
  k_epoch_bump<<<1, 1, 0, s>>>(epoch, per_solve);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "epoch kernel launch");
}

px_status launch_stream_ldg(int mode, int stencil, const StreamLaunch& a, cudaStream_t s) {
  if (a.nx <= 0 || a.ny <= 0) return PX_OK;
  const int32_t rows = ldg_rows(a.nx, a.ny, a.phase);
  dim3 grid((a.nx + a.phase + SW_COLS - 1) / SW_COLS, (a.ny + rows - 1) / rows);
  if (grid.y > 65535) return fail(PX_ERR_UNSUPPORTED, "region too tall (%d rows)", a.ny);
  switch (mode * 2 + stencil) {
    case MODE_RELAX * 2 + 0: launch_t<MODE_RELAX, 0>(a, grid, s); break;
    case MODE_RELAX * 2 + 1: launch_t<MODE_RELAX, 1>(a, grid, s); break;
    case MODE_RESID * 2 + 0: launch_t<MODE_RESID, 0>(a, grid, s); break;
    case MODE_RESID * 2 + 1: launch_t<MODE_RESID, 1>(a, grid, s); break;
    case MODE_APPLY * 2 + 0: launch_t<MODE_APPLY, 0>(a, grid, s); break;
    case MODE_APPLY * 2 + 1: launch_t<MODE_APPLY, 1>(a, grid, s); break;
    case MODE_MRHS * 2 + 0: launch_t<MODE_MRHS, 0>(a, grid, s); break;
    default: return fail(PX_ERR_ARG, "bad stream mode %d / stencil %d", mode, stencil);
  }
  if (mode == MODE_RELAX) note_kernel("k_stream");
  count_launches(1);
  return cuda_check(cudaGetLastError(), "stream kernel launch");
}

int32_t persist_rows(int32_t nx, int32_t ny, int32_t grid) {
  const int64_t gx = (nx + SW_COLS - 1) / SW_COLS;
  int32_t rows = (int32_t)((gx * ny + grid - 1) / grid);
  rows = (rows + SW_PF - 1) / SW_PF * SW_PF;
  return rows < SW_PF ? SW_PF : rows;
}

// co-resident grid of the persistent kernel (cooperative launch limit)
int32_t persist_grid() {
  static int g = 0;
  if (!g) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_persist<0>, SW_THREADS, 0) != cudaSuccess ||
        per < 1)
      per = 1;
    int per9 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per9, k_persist<1>, SW_THREADS, 0) != cudaSuccess ||
        per9 < 1)
      per9 = 1;
    g = ldg_nsm() * (per < per9 ? per : per9);
  }
  return g;
}

px_status launch_persist(int stencil, const PersistLaunch& p, int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SW_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = stencil ? cudaLaunchKernelEx(&cfg, k_persist<1>, p) : cudaLaunchKernelEx(&cfg, k_persist<0>, p);
  note_kernel("k_persist");
  if (e == cudaSuccess) e = cudaGetLastError();
  count_launches(1);
  return cuda_check(e, "persistent solve kernel launch");
}

// ------------------------------------------------------------ ghost fill
// Phase x: for rows [0, ny) fill columns [-g, 0) and [nx, nx+g).
__global__ void k_ghost_x(double* o, int64_t ld, int nx, int ny, int g, int mlo, int mhi) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)ny * g * 2;
  if (idx >= total) return;
  const int side = (int)(idx & 1);
  const int t = (int)((idx >> 1) % g) + 1;
  const int y = (int)((idx >> 1) / g);
  double* row = o + (int64_t)y * ld;
  if (side == 0) {
    if (mlo == GH_WRAP) row[-t] = row[nx - t];
    else if (mlo == GH_REFLECT) row[-t] = -row[t - 1];
  } else {
    if (mhi == GH_WRAP) row[nx - 1 + t] = row[t - 1];
    else if (mhi == GH_REFLECT) row[nx - 1 + t] = -row[nx - t];
  }
}
// Phase y: full rows x in [-g, nx+g) of ghost rows [-g, 0) and [ny, ny+g).
__global__ void k_ghost_y(double* o, int64_t ld, int nx, int ny, int g, int mlo, int mhi) {
  const int64_t W = nx + 2 * g;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= W * g * 2) return;
  const int x = (int)(idx % W) - g;
  const int t = (int)((idx / W) % g) + 1;
  const int side = (int)(idx / (W * g));
  if (side == 0) {
    if (mlo == GH_WRAP) o[x - (int64_t)t * ld] = o[x + (int64_t)(ny - t) * ld];
    else if (mlo == GH_REFLECT) o[x - (int64_t)t * ld] = -o[x + (int64_t)(t - 1) * ld];
  } else {
    if (mhi == GH_WRAP) o[x + (int64_t)(ny - 1 + t) * ld] = o[x + (int64_t)(t - 1) * ld];
    else if (mhi == GH_REFLECT) o[x + (int64_t)(ny - 1 + t) * ld] = -o[x + (int64_t)(ny - t) * ld];
  }
}

px_status launch_fill_ghosts(const px_layout* l, int32_t rank, const px_patch& p, cudaStream_t s) {
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  const int nx = ext(li.owned, 0), ny = ext(li.owned, 1), g = l->ghost;
  double* o = at(p, li.owned.lo.c[0], li.owned.lo.c[1]);
  int mx = GH_NONE, my_lo = GH_NONE, my_hi = GH_NONE;
  if (l->bc == PX_BC_PERIODIC) mx = GH_WRAP;
  else if (l->bc == PX_BC_DIRICHLET_CC) mx = GH_REFLECT;
  if (li.nbr_lo < 0 && l->bc == PX_BC_DIRICHLET_CC) my_lo = GH_REFLECT;
  if (li.nbr_hi < 0 && l->bc == PX_BC_DIRICHLET_CC) my_hi = GH_REFLECT;
  if (l->bc == PX_BC_PERIODIC && l->nranks == 1) my_lo = my_hi = GH_WRAP;
  return launch_fill_ghosts_raw(o, p.ld, nx, ny, g, mx, my_lo, my_hi, s);
}

px_status launch_fill_ghosts_raw(double* o, int64_t ld, int nx, int ny, int g, int mx, int my_lo, int my_hi,
                                 cudaStream_t s) {
  if (mx != GH_NONE) {
    int64_t n = (int64_t)ny * g * 2;
    k_ghost_x<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(o, ld, nx, ny, g, mx, mx);
    count_launches(1);
    PX_TRY(cuda_check(cudaGetLastError(), "ghost x launch"));
  }
  if (my_lo != GH_NONE || my_hi != GH_NONE) {
    int64_t n = (int64_t)(nx + 2 * g) * g * 2;
    k_ghost_y<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(o, ld, nx, ny, g, my_lo, my_hi);
    count_launches(1);
    PX_TRY(cuda_check(cudaGetLastError(), "ghost y launch"));
  }
  return PX_OK;
}

// ------------------------------------------------------ synthetic fields
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_init(double* o, int64_t ld, int nx, int ny, int gx0, int gy0, int n0, int n1,
                       int kind, uint64_t seed, int kw, int lw) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= nx) return;
  const int64_t i = gx0 + x, j = gy0 + y;
  double v = 0.0;
  if (kind == PX_FIELD_HASH) {
    const uint64_t u = splitmix64(seed ^ (uint64_t)(i + j * (int64_t)n0));
    v = ((double)(u >> 11) * 0x1p-53) * 2.0 - 1.0;
  } else if (kind == PX_FIELD_SINE) {
    v = sin(kw * M_PI * ((i + 0.5) / n0)) * sin(lw * M_PI * ((j + 0.5) / n1));
  }
  o[x + (int64_t)y * ld] = v;
}

px_status launch_init_field(const px_layout* l, int32_t rank, const px_patch& p, int kind,
                            uint64_t seed, int k, int lw, cudaStream_t s) {
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  const int nx = ext(li.owned, 0), ny = ext(li.owned, 1);
  double* o = at(p, li.owned.lo.c[0], li.owned.lo.c[1]);
  dim3 grid((nx + 255) / 256, ny);
  if (ny > 65535 * 32) return fail(PX_ERR_UNSUPPORTED, "too many rows");
  // grid.y is limited to 65535: split tall slabs
  for (int y0 = 0; y0 < ny; y0 += 65535) {
    int h = ny - y0 < 65535 ? ny - y0 : 65535;
    dim3 g2((nx + 255) / 256, h);
    k_init<<<g2, 256, 0, s>>>(o + (int64_t)y0 * p.ld, p.ld, nx, h,
                              li.owned.lo.c[0] - l->domain.lo.c[0],
                              li.owned.lo.c[1] - l->domain.lo.c[1] + y0, ext(l->domain, 0),
                              ext(l->domain, 1), kind, seed, k, lw);
    count_launches(1);
    PX_TRY(cuda_check(cudaGetLastError(), "init launch"));
  }
  return PX_OK;
}

}  // namespace px

extern "C" int64_t px_kernel_launch_count(void) { return px::g_launches; }
