// px_resident.cu -- all sweeps of an L2-sized single-rank solve with the
// iterate RESIDENT IN SHARED MEMORY (BASELINE config 2: 1024², 1000 sweeps;
// SURVEY §8(d) "C2 is L2-bound and launch-bound").
//
// One cooperative launch of G <= #SM CTAs.  CTA c owns the rows
// [c·ny/G, (c+1)·ny/G) and keeps them in shared memory for the whole solve:
// two copies of its rows plus one halo row above and below (with the ghost
// columns), and its rows of the right-hand side.  A sweep reads and writes
// shared memory only.  The CTA sweeps its first and last row first; each
// thread publishes its own cells of them to an L2 mailbox straight from
// registers as LL entries (every 8-byte half carries the sweep tag, so the
// data is its own flag: no barrier, fence or flag word before the
// publication), sweeps its inner rows while they travel, then fetches its
// cells of the neighbours' rows (spinning until both tags match) into its
// halo rows.  One block barrier per sweep; no grid-wide barrier: a CTA
// synchronises with its two neighbours only.  Domain faces: periodic wrap
// (the ring of CTAs), odd reflection (halo row = −own row, written by the
// thread that computed it), fixed ghosts (kept from φ^0); the thread holding
// column 0 / nx−1 of a row also writes the ghost columns that copy or
// reflect it.
//
// Per cell the oracle's expression tree with every * and + rounded
// separately (bit-identical).  Norms: per thread in row order, per CTA in
// fixed warp order into partials[entry][cta]; after the last sweep one grid
// barrier, then entry e is reduced over the CTAs in fixed order by CTA
// e mod G.  Deterministic for a given (nx, ny, #SM).
//
// Safety of the two publication slots: CTA c writes φ^{s+1} rows into slot
// (s+1)&1 during sweep s; it writes slot (s+1)&1 again (φ^{s+3}, sweep s+2)
// only after it fetched its neighbours' φ^{s+2} rows, which they published
// in their sweep s+1, i.e. after they fetched φ^{s+1}.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <cstdlib>

#include "px_device.cuh"
#include "px_internal.h"

namespace cg = cooperative_groups;

namespace px {

constexpr int RS_THREADS = 512;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}


// Rows rlo..rhi of the CTA's shared block: B = A + λ(scale·L(A) − F)
// (WRITE), or residual norms of A only.  A thread walks a column pair down
// the rows with the S/C rows (and their outer neighbours) in registers.
// NORM = false: a sweep whose norm is not recorded skips the accumulation.
template <int ST, bool WRITE, bool NORM = true>
__device__ __forceinline__ void rs_rows(const double* A, double* B, const double* F, int P, int nx, int rlo,
                                        int rhi, double scale, double lambda, unsigned long long& mx,
                                        double& ss) {
  for (int q = threadIdx.x; q < nx / 2; q += blockDim.x) {
    const int x = 2 * q + 2;  // shared index of column 2q
    const double* a0 = A + (size_t)(rlo - 1) * P + x;
    double2 S = *reinterpret_cast<const double2*>(a0);
    double2 C = *reinterpret_cast<const double2*>(a0 + P);
    double sw = a0[-1], se = a0[2], cw = a0[P - 1], ce = a0[P + 2];
    for (int r = rlo; r <= rhi; ++r) {
      const double* an = A + (size_t)(r + 1) * P + x;
      const double2 N = *reinterpret_cast<const double2*>(an);
      const double nw = an[-1], ne = an[2];
      const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
      const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
      const double2 f = *reinterpret_cast<const double2*>(F + (size_t)(r - 1) * nx + (x - 2));
      const double r0 = __dsub_rn(__dmul_rn(scale, L0), f.x);
      const double r1 = __dsub_rn(__dmul_rn(scale, L1), f.y);
      if (WRITE) {
        double2 o;
        o.x = __dadd_rn(C.x, __dmul_rn(lambda, r0));
        o.y = __dadd_rn(C.y, __dmul_rn(lambda, r1));
        *reinterpret_cast<double2*>(B + (size_t)r * P + x) = o;
      }
      if (NORM) {
        mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r0)));
        ss = fma(r0, r0, ss);
        mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r1)));
        ss = fma(r1, r1, ss);
      }
      S = C;
      sw = cw;
      se = ce;
      C = N;
      cw = nw;
      ce = ne;
    }
  }
}

// fixed-order block reduction of (max bits, Σ) into out[0..1] (thread 0)
__device__ __forceinline__ void rs_block_reduce(unsigned long long mx, double ss, double* out) {
  __shared__ unsigned long long s_mx[RS_THREADS / 32];
  __shared__ double s_ss[RS_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    out[0] = __longlong_as_double((long long)m);
    out[1] = t;
  }
  __syncthreads();
}

// ghost columns -1 and nx of one shared row (x rule; GH_NONE keeps them)
__device__ __forceinline__ void rs_xghost(double* row, int nx, const int (&xm)[2]) {
  if (xm[0] == GH_WRAP) row[1] = row[nx + 1];
  else if (xm[0] == GH_REFLECT) row[1] = -row[2];
  if (xm[1] == GH_WRAP) row[nx + 2] = row[2];
  else if (xm[1] == GH_REFLECT) row[nx + 2] = -row[nx + 1];
}

// ---- LL exchange (the row mailbox carries its own flags) -------------------
// One double per 16-byte entry, each 8-byte half = (sweep tag << 32) | one
// 32-bit half of the double (NCCL's LL idea), stored as one u64 element of a
// v2.u64 access, i.e. single-copy atomic: a reader that sees the tag in both
// halves has the whole value of that sweep -- no release fence, no flag word,
// no barrier before the publication.
#ifndef PX_LL_SYS
#define PX_LL_SYS 0  // A/B: 1 = the round-2 volatile (system-scope) mailbox accesses
#endif
__device__ __forceinline__ void ll_put(double* e, double v, uint32_t tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long t = (unsigned long long)tag << 32;
#if PX_LL_SYS
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(e), "l"(t | (b & 0xffffffffull)), "l"(t | (b >> 32))
               : "memory");
#else
  // gpu scope (the mailbox never leaves the device): STG.STRONG.GPU, not .SYS
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(e), "l"(t | (b & 0xffffffffull)),
               "l"(t | (b >> 32))
               : "memory");
#endif
}
#ifndef PX_RR_PROF
#define PX_RR_PROF 0  // per-phase clock64 totals of k_resident_reg (printf; scripts/build_variant.py)
#endif
#ifndef PX_RS_DIAG
#define PX_RS_DIAG 0  // A/B diagnostics only (scripts/build_variant.py): 1 no tag wait, 2 no row compute
#endif
#ifndef LL_BACKOFF_NS
#define LL_BACKOFF_NS 100
#endif
struct LL {
  unsigned long long lo, hi;  // (tag << 32) | low / high half of the double
};
__device__ __forceinline__ LL ll_load(const double* e) {
  LL v;
#if PX_LL_SYS
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.lo), "=l"(v.hi) : "l"(e) : "memory");
#else
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.lo), "=l"(v.hi) : "l"(e) : "memory");
#endif
  return v;
}
__device__ __forceinline__ bool ll_ok(const LL& v, uint32_t tag) {
  return (uint32_t)(v.lo >> 32) == tag && (uint32_t)(v.hi >> 32) == tag;
}
__device__ __forceinline__ double ll_val(const LL& v) {
  return __longlong_as_double((long long)((v.hi << 32) | (v.lo & 0xffffffffull)));
}
// A column pair as ONE 32-B LL entry (sm_100 v4.u64 access; each u64 element
// = tag << 32 | one half of a double, single-copy atomic as above): one store
// and one poll per pair and row instead of two.
__device__ __forceinline__ void ll_put2(double* e, double2 v, uint32_t tag) {
  const unsigned long long a = (unsigned long long)__double_as_longlong(v.x);
  const unsigned long long b = (unsigned long long)__double_as_longlong(v.y);
  const unsigned long long t = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(e), "l"(t | (a & 0xffffffffull)),
               "l"(t | (a >> 32)), "l"(t | (b & 0xffffffffull)), "l"(t | (b >> 32))
               : "memory");
}
struct LL2 {
  unsigned long long w[4];
};
__device__ __forceinline__ LL2 ll_load2(const double* e) {
  LL2 v;
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3])
               : "l"(e)
               : "memory");
  return v;
}
__device__ __forceinline__ bool ll2_ok(const LL2& v, uint32_t tag) {
  return (uint32_t)(v.w[0] >> 32) == tag && (uint32_t)(v.w[1] >> 32) == tag && (uint32_t)(v.w[2] >> 32) == tag &&
         (uint32_t)(v.w[3] >> 32) == tag;
}
__device__ __forceinline__ double2 ll2_val(const LL2& v) {
  return make_double2(__longlong_as_double((long long)((v.w[1] << 32) | (v.w[0] & 0xffffffffull))),
                      __longlong_as_double((long long)((v.w[3] << 32) | (v.w[2] & 0xffffffffull))));
}
// the n (<= M) pair entries e[i], loads in flight together, re-polled until
// every tag matches
template <int n, int M>
__device__ __forceinline__ void ll_get2(const double* const (&e)[M], uint32_t tag, double2 (&out)[M]) {
  LL2 v[M];
#pragma unroll
  for (int i = 0; i < n; ++i) v[i] = ll_load2(e[i]);
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < n; ++i) ok = ok && ll2_ok(v[i], tag);
    if (ok) break;
    if (LL_BACKOFF_NS) __nanosleep(LL_BACKOFF_NS);
#pragma unroll
    for (int i = 0; i < n; ++i)
      if (!ll2_ok(v[i], tag)) v[i] = ll_load2(e[i]);
  }
#pragma unroll
  for (int i = 0; i < n; ++i) out[i] = ll2_val(v[i]);
}

// the n (<= 4) entries e[i], all loads in flight together; re-poll until
// every tag matches
template <int n, int M>
__device__ __forceinline__ void ll_get(const double* const (&e)[M], uint32_t tag, double (&out)[M]) {
  LL v[M];
#pragma unroll
  for (int i = 0; i < n; ++i) v[i] = ll_load(e[i]);
#if PX_RS_DIAG == 1
  for (int it = 0; it < 0; ++it) {  // diagnostic: take whatever the mailbox holds
#else
  for (;;) {
#endif
    bool ok = true;
#pragma unroll
    for (int i = 0; i < n; ++i) ok = ok && ll_ok(v[i], tag);
    if (ok) break;
    if (LL_BACKOFF_NS) __nanosleep(LL_BACKOFF_NS);  // fewer polls in flight: L2 stays free for the publications
#pragma unroll
    for (int i = 0; i < n; ++i)
      if (!ll_ok(v[i], tag)) v[i] = ll_load(e[i]);
  }
#pragma unroll
  for (int i = 0; i < n; ++i) out[i] = ll_val(v[i]);
}

// The x images of one row's pair (columns 2q, 2q+1 at shared index x): the
// thread holding column 0 / nx-1 also writes the ghost columns that copy or
// reflect it (periodic: -1 <- nx-1, nx <- 0; reflection: -1 <- -0, nx <- -(nx-1)).
__device__ __forceinline__ void ll_ximg(double* row, int x, int nx, double v0, double v1, const int (&xm)[2]) {
  if (x == 2) {
    if (xm[1] == GH_WRAP) row[nx + 2] = v0;
    if (xm[0] == GH_REFLECT) row[1] = -v0;
  }
  if (x == nx) {
    if (xm[0] == GH_WRAP) row[1] = v1;
    if (xm[1] == GH_REFLECT) row[nx + 2] = -v1;
  }
}

// Rows rlo..rhi of B = A + λ(scale·L(A) − F) (as rs_rows), with each row's x
// images, and -- for row 1 / row R -- the row published to the mailbox (pub_first
// / pub_last, 2 doubles per column) or, at a reflecting y face, its odd image
// written into the halo row 0 / R+1 of B.
template <int ST, bool NORM>
__device__ __forceinline__ void ll_rows(const double* A, double* B, const double* F, int P, int nx, int R, int rlo,
                                        int rhi, double scale, double lambda, const int (&xm)[2],
                                        double* pub_first, double* pub_last, bool refl_top, bool refl_bot,
                                        uint32_t tag, unsigned long long& mx, double& ss) {
  for (int q = threadIdx.x; q < nx / 2; q += blockDim.x) {
    const int x = 2 * q + 2;
    const double* a0 = A + (size_t)(rlo - 1) * P + x;
    double2 S = *reinterpret_cast<const double2*>(a0);
    double2 C = *reinterpret_cast<const double2*>(a0 + P);
    double sw = a0[-1], se = a0[2], cw = a0[P - 1], ce = a0[P + 2];
    for (int r = rlo; r <= rhi; ++r) {
      const double* an = A + (size_t)(r + 1) * P + x;
      const double2 N = *reinterpret_cast<const double2*>(an);
      const double nw = an[-1], ne = an[2];
      const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
      const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
      const double2 f = *reinterpret_cast<const double2*>(F + (size_t)(r - 1) * nx + (x - 2));
      const double r0 = __dsub_rn(__dmul_rn(scale, L0), f.x);
      const double r1 = __dsub_rn(__dmul_rn(scale, L1), f.y);
      double2 o;
      o.x = __dadd_rn(C.x, __dmul_rn(lambda, r0));
      o.y = __dadd_rn(C.y, __dmul_rn(lambda, r1));
      double* brow = B + (size_t)r * P;
      *reinterpret_cast<double2*>(brow + x) = o;
      ll_ximg(brow, x, nx, o.x, o.y, xm);
      if (r == 1) {
        if (pub_first) {
          ll_put(pub_first + (x - 2), o.x, tag);
          ll_put(pub_first + (x - 2) + nx, o.y, tag);
        } else if (refl_top) {
          *reinterpret_cast<double2*>(B + x) = make_double2(-o.x, -o.y);
          ll_ximg(B, x, nx, -o.x, -o.y, xm);
        }
      }
      if (r == R) {
        if (pub_last) {
          ll_put(pub_last + (x - 2), o.x, tag);
          ll_put(pub_last + (x - 2) + nx, o.y, tag);
        } else if (refl_bot) {
          double* h = B + (size_t)(R + 1) * P;
          *reinterpret_cast<double2*>(h + x) = make_double2(-o.x, -o.y);
          ll_ximg(h, x, nx, -o.x, -o.y, xm);
        }
      }
      if (NORM) {
        mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r0)));
        ss = fma(r0, r0, ss);
        mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r1)));
        ss = fma(r1, r1, ss);
      }
      S = C;
      sw = cw;
      se = ce;
      C = N;
      cw = nw;
      ce = ne;
    }
  }
}

// Store of row r's pair o (with its x images) into B and, for row 1 / row R,
// the publication (or the reflected halo row) -- the per-row epilogue of
// ll_rows, shared by the unrolled walk below.
__device__ __forceinline__ void ll_emit(double* B, int P, int nx, int R, int r, int x, double2 o,
                                        const int (&xm)[2], double* pub_first, double* pub_last, bool refl_top,
                                        bool refl_bot, uint32_t tag) {
  double* brow = B + (size_t)r * P;
  *reinterpret_cast<double2*>(brow + x) = o;
  ll_ximg(brow, x, nx, o.x, o.y, xm);
  if (r == 1) {
    if (pub_first) {
      ll_put(pub_first + (x - 2), o.x, tag);
      ll_put(pub_first + (x - 2) + nx, o.y, tag);
    } else if (refl_top) {
      *reinterpret_cast<double2*>(B + x) = make_double2(-o.x, -o.y);
      ll_ximg(B, x, nx, -o.x, -o.y, xm);
    }
  }
  if (r == R) {
    if (pub_last) {
      ll_put(pub_last + (x - 2), o.x, tag);
      ll_put(pub_last + (x - 2) + nx, o.y, tag);
    } else if (refl_bot) {
      double* h = B + (size_t)(R + 1) * P;
      *reinterpret_cast<double2*>(h + x) = make_double2(-o.x, -o.y);
      ll_ximg(h, x, nx, -o.x, -o.y, xm);
    }
  }
}

// One pair of row r from the register copies of rows r-1, r, r+1 (oracle
// expression tree, every op rounded).
template <int ST, bool NORM>
__device__ __forceinline__ double2 ll_pair(double2 S, double sw, double se, double2 C, double cw, double ce,
                                           double2 N, double nw, double ne, double2 f, double scale,
                                           double lambda, unsigned long long& mx, double& ss) {
  const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
  const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
  const double r0 = __dsub_rn(__dmul_rn(scale, L0), f.x);
  const double r1 = __dsub_rn(__dmul_rn(scale, L1), f.y);
  double2 o;
  o.x = __dadd_rn(C.x, __dmul_rn(lambda, r0));
  o.y = __dadd_rn(C.y, __dmul_rn(lambda, r1));
  if (NORM) {
    mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r0)));
    ss = fma(r0, r0, ss);
    mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r1)));
    ss = fma(r1, r1, ss);
  }
  return o;
}

// ll_rows for a CTA of R <= RM rows with the whole column walk UNROLLED: a
// thread loads its pair of all R + 2 rows up front, so the R rows' expression trees are independent streams
// the scheduler interleaves (the rolled walk of ll_rows issues one row's
// chain at a time and shuffles its registers between rows).  Same rows in
// the same order as ll_rows (row 1, row R, rows 2..R-1) -- same stores, same
// publications, same per-thread norm order: bit-identical.
template <int ST, bool NORM, int RM>
__device__ __forceinline__ void ll_rows_u(const double* A, double* B, const double* F, int P, int nx, int R,
                                          double scale, double lambda, const int (&xm)[2], double* pub_first,
                                          double* pub_last, bool refl_top, bool refl_bot, uint32_t tag,
                                          unsigned long long& mx, double& ss) {
  for (int q = threadIdx.x; q < nx / 2; q += blockDim.x) {
    const int x = 2 * q + 2;
    double2 a[RM + 2];
#pragma unroll
    for (int i = 0; i < RM + 2; ++i)
      if (i <= R + 1) a[i] = *reinterpret_cast<const double2*>(A + (size_t)i * P + x);
    // the W/E neighbour columns (and ρ) are loaded where a row uses them:
    // keeping them for every row would spill at 128 registers per thread
#define LL_ROW(r)                                                                                            \
  {                                                                                                          \
    const double* ac = A + (size_t)(r) * P + x;                                                              \
    const double sw = ST ? ac[-P - 1] : 0.0, se = ST ? ac[-P + 2] : 0.0;                                     \
    const double nw = ST ? ac[P - 1] : 0.0, ne = ST ? ac[P + 2] : 0.0;                                       \
    ll_emit(B, P, nx, R, r, x,                                                                               \
            ll_pair<ST, NORM>(a[r - 1], sw, se, a[r], ac[-1], ac[2], a[r + 1], nw, ne,                       \
                              *reinterpret_cast<const double2*>(F + (size_t)((r) - 1) * nx + (x - 2)), scale, \
                              lambda, mx, ss),                                                               \
            xm, pub_first, pub_last, refl_top, refl_bot, tag);                                               \
  }
    LL_ROW(1);
#pragma unroll
    for (int r = 2; r <= RM; ++r)
      if (r == R) LL_ROW(r);
#pragma unroll
    for (int r = 2; r < RM; ++r)
      if (r < R) LL_ROW(r);
#undef LL_ROW
  }
}
constexpr int LL_UNROLL_ROWS = 7;  // BJ.C2: 1024 rows over 148 CTAs = 6 or 7 rows each

template <int ST>
__global__ void __launch_bounds__(RS_THREADS, 1) k_resident(const ResidentLaunch p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int nx = p.nx, P = nx + 4;
  const int y0 = (int)((int64_t)c * p.ny / G), y1 = (int)((int64_t)(c + 1) * p.ny / G), R = y1 - y0;
  double* A = sm;
  double* B = A + (size_t)(p.rmax + 2) * P;
  double* F = B + (size_t)(p.rmax + 2) * P;
  // [slot][cta][first, last][nx] LL entries (16 B each); the row's pair q puts
  // its cells in entries q and nx/2 + q, so every warp-wide store and poll
  // covers whole 32-B sectors (16-B entries at a 32-B stride -- a pair's two
  // cells side by side -- double the hop latency: scripts/ll_latency.cu)
  double* pub = p.ws + ((G + 1) & ~1);
  double* part = pub + (size_t)2 * G * 2 * 2 * nx; // [entry][cta][max, sum]
  const int up = c > 0 ? c - 1 : G - 1, dn = c < G - 1 ? c + 1 : 0;
  const bool top_x = c > 0 || p.ymode[0] == GH_WRAP;      // halo row 0 from CTA `up`
  const bool bot_x = c < G - 1 || p.ymode[1] == GH_WRAP;  // halo row R+1 from CTA `dn`
  const int xm[2] = {p.xmode[0], p.xmode[1]};

  // φ^0 rows y0-1 .. y1 with their ghost columns (ghost ring filled by the
  // caller's exchange) into both copies; the rhs rows.
  for (int r = 0; r < R + 2; ++r) {
    const double* src = p.phi_in + (int64_t)(y0 - 1 + r) * p.ld_in;
    for (int x = tid - 1; x <= nx; x += nt) {
      const double v = src[x];
      A[(size_t)r * P + x + 2] = v;
      B[(size_t)r * P + x + 2] = v;
    }
  }
  for (int r = 0; r < R; ++r)
    for (int x = tid; x < nx; x += nt) F[(size_t)r * nx + x] = p.rhs[(int64_t)(y0 + r) * p.ld_rhs + x];
  // this CTA's mailbox entries start with tag 0 (a solve's tags are 1..N)
  for (int sl = 0; sl < 2; ++sl)
    for (int i = tid; i < 2 * 2 * nx; i += nt) pub[(size_t)(sl * G + c) * 2 * 2 * nx + i] = 0.0;
  __threadfence();
  grid.sync();

  int entry = 0;
  const bool refl_top = !top_x && p.ymode[0] == GH_REFLECT, refl_bot = !bot_x && p.ymode[1] == GH_REFLECT;
  const bool unrolled = p.unroll && p.rmax <= LL_UNROLL_ROWS;
  for (int s = 0; s < p.nsweeps; ++s) {
    const bool rec = p.every > 0 && s % p.every == 0;
    const uint32_t tag = (uint32_t)s + 1u;
    unsigned long long mx = 0ull;
    double ss = 0.0;
    // the first and last rows first, each thread publishing its own cells of
    // them straight from registers (LL entries: no barrier, no fence, no
    // flag), so the neighbours' copies overlap the sweep of the inner rows
    const int slot = (s + 1) & 1;
    double* mine = pub + (size_t)(slot * G + c) * 2 * 2 * nx;
    double* pf = top_x ? mine : nullptr;
    double* pl = bot_x ? mine + 2 * nx : nullptr;
    auto sweep = [&](int lo, int hi) {
      if (rec) ll_rows<ST, true>(A, B, F, P, nx, R, lo, hi, p.scale, p.lambda, xm, pf, pl, refl_top, refl_bot, tag, mx, ss);
      else ll_rows<ST, false>(A, B, F, P, nx, R, lo, hi, p.scale, p.lambda, xm, pf, pl, refl_top, refl_bot, tag, mx, ss);
    };
#if PX_RS_DIAG == 2
    if (true) {  // diagnostic: publish the rows without computing any
      for (int q = tid; q < nx / 2; q += nt) {
        const int x = 2 * q + 2;
        if (pf) { ll_put(pf + (x - 2), 0.0, tag); ll_put(pf + (x - 2) + nx, 0.0, tag); }
        if (pl) { ll_put(pl + (x - 2), 0.0, tag); ll_put(pl + (x - 2) + nx, 0.0, tag); }
      }
    } else
#endif
    if (unrolled) {
      if (rec)
        ll_rows_u<ST, true, LL_UNROLL_ROWS>(A, B, F, P, nx, R, p.scale, p.lambda, xm, pf, pl, refl_top, refl_bot,
                                            tag, mx, ss);
      else
        ll_rows_u<ST, false, LL_UNROLL_ROWS>(A, B, F, P, nx, R, p.scale, p.lambda, xm, pf, pl, refl_top, refl_bot,
                                             tag, mx, ss);
    } else {
      sweep(1, 1);
      if (R > 1) sweep(R, R);
      if (R > 2) sweep(2, R - 1);
    }
    if (rec) {
      rs_block_reduce(mx, ss, part + ((size_t)entry * G + c) * 2);
      ++entry;
    }
    // the neighbours' rows of φ^{s+1}: each thread fetches its own cells
    // (spinning on the tags) and writes them, with their x images, into the
    // halo rows
    const double* fu = pub + ((size_t)(slot * G + up) * 2 + 1) * 2 * nx;  // up's last row
    const double* fd = pub + ((size_t)(slot * G + dn) * 2) * 2 * nx;      // dn's first row
    for (int q = tid; q < nx / 2; q += nt) {
      const int x = 2 * q + 2;
      double v[4];
      if (top_x && bot_x) {
        const double* const e[4] = {fu + 2 * q, fu + 2 * q + nx, fd + 2 * q, fd + 2 * q + nx};
        ll_get<4>(e, tag, v);
      } else if (top_x || bot_x) {
        const double* f = top_x ? fu : fd;
        const double* const e[4] = {f + 2 * q, f + 2 * q + nx, f, f};
        ll_get<2>(e, tag, v);
        if (!top_x) {
          v[2] = v[0];
          v[3] = v[1];
        }
      }
      if (top_x) {
        *reinterpret_cast<double2*>(B + x) = make_double2(v[0], v[1]);
        ll_ximg(B, x, nx, v[0], v[1], xm);
      }
      if (bot_x) {
        double* h = B + (size_t)(R + 1) * P;
        *reinterpret_cast<double2*>(h + x) = make_double2(v[2], v[3]);
        ll_ximg(h, x, nx, v[2], v[3], xm);
      }
    }
    __syncthreads();
    double* t = A;
    A = B;
    B = t;
  }
  if (p.final_norm) {
    unsigned long long mx = 0ull;
    double ss = 0.0;
    rs_rows<ST, false>(A, nullptr, F, P, nx, 1, R, p.scale, p.lambda, mx, ss);
    rs_block_reduce(mx, ss, part + ((size_t)entry * G + c) * 2);
    ++entry;
  }
  __threadfence();
  grid.sync();
  // entries reduced over the CTAs in fixed order
  for (int e = c; e < entry; e += G) {
    unsigned long long m = 0ull;
    double t = 0.0;
    for (int i = tid; i < G; i += nt) {
      m = umax64(m, (unsigned long long)__double_as_longlong(__ldcg(part + ((size_t)e * G + i) * 2)));
      t = t + __ldcg(part + ((size_t)e * G + i) * 2 + 1);
    }
    double out[2];
    rs_block_reduce(m, t, out);
    if (tid == 0) {
      p.d_max[e] = out[0];
      p.d_sum[e] = out[1];
    }
  }
  // φ^N (with its ghost columns) back to HBM; the face ghost rows too
  for (int r = 1; r <= R; ++r) {
    double* dst = p.phi_out + (int64_t)(y0 - 1 + r) * p.ld_out;
    for (int x = tid - 1; x <= nx; x += nt) dst[x] = A[(size_t)r * P + x + 2];
  }
  if (c == 0)
    for (int x = tid - 1; x <= nx; x += nt) p.phi_out[-p.ld_out + x] = A[x + 2];
  if (c == G - 1)
    for (int x = tid - 1; x <= nx; x += nt) p.phi_out[(int64_t)p.ny * p.ld_out + x] = A[(size_t)(R + 1) * P + x + 2];
}

// ---------------------------------------------------------------------------
// k_resident_reg<ST>: the resident solve with the iterate in REGISTERS.
// Thread q owns column pair q (columns 2q, 2q+1) of every row of its CTA
// plus the two halo rows, as double2 registers that persist across sweeps;
// only ρ stays in shared memory.  W/E neighbours come from the adjacent
// lanes (__shfl_up/down) and, across warp boundaries, from per-warp edge
// arrays in shared memory (lane 0's first and the last active lane's second
// column of every row, double-buffered by sweep parity, written before the
// one block barrier per sweep); at the domain's x faces from the edge of the
// last / first warp (periodic), the cell itself (odd reflection) or the fixed
// ghost columns of φ^0.  Every thread reads its W/E candidates the same way
// (one shuffle and one shared load, a dummy broadcast address where it has
// no edge) and selects: no divergent branch per row.  The row count is a
// template parameter (the CTA's R dispatched once), so the column walk has
// no per-row predicates.  A sweep: row R, then row 1 (both published to the
// L2 mailbox at once, as k_resident), then rows 2..R-1 in place with one
// rolling register of the old row above; then the neighbours' rows of the
// new iterate are fetched into the halo registers, the edges written, one
// barrier.  Per cell the same expression tree, per thread the same norm order
// (row 1, row R, rows 2..R-1; final pass rows 1..R) and the same thread ->
// pair map as k_resident: bit-identical to it.
constexpr int RR_RM = 7;  // BJ.C2: 1024 rows over 148 CTAs = 6 or 7 rows each
struct RrCtx {
  const double* F;                 // ρ rows [R][nx]
  double *eL, *eR;                 // [2][NWP][RE]
  const double* wp;                // west candidate (buffer 0, row 0); dummy broadcast if none
  const double* ep;                // east candidate
  int wbs, ebs;                    // buffer stride of wp / ep (0: not double-buffered)
  bool wld, eld;                   // take the shared candidate instead of the shuffle
  bool st_l, st_r;                 // this lane stores the warp's left / right edge
  double *gW, *gE;                 // [2][RE] ghost columns -1 / nx: fixed (both buffers), or the
  bool st_gw, st_ge;               // odd reflections the first / last pair stores with its edges
  int warp, x, xs, nx, G, c, up, dn;
  bool act, top_x, bot_x, refl_top, refl_bot;
  double *pub, *part;
};
template <int ST, int RR, bool P2>
__device__ __forceinline__ void rr_body(const ResidentLaunch& p, const RrCtx& k, cg::grid_group& grid) {
  constexpr int NWP = RS_THREADS / 32, RE = RR_RM + 2, BS = NWP * RE;
  const int tid = threadIdx.x, nx = k.nx, x = k.x, G = k.G, c = k.c;
  const int y0 = (int)((int64_t)c * p.ny / G);
  double2 cur[RR + 2];
#pragma unroll
  for (int r = 0; r < RR + 2; ++r) {
    cur[r] = make_double2(0.0, 0.0);
    if (k.act) {
      const double* src = p.phi_in + (int64_t)(y0 - 1 + r) * p.ld_in + x;
      cur[r] = make_double2(src[0], src[1]);
    }
  }
  auto put_edges = [&](int b) {
#pragma unroll
    for (int r = 0; r < RR + 2; ++r) {
      if (k.st_l) k.eL[b * BS + k.warp * RE + r] = cur[r].x;
      if (k.st_r) k.eR[b * BS + k.warp * RE + r] = cur[r].y;
      if (k.st_gw) k.gW[b * RE + r] = -cur[r].x;
      if (k.st_ge) k.gE[b * RE + r] = -cur[r].y;
    }
  };
  put_edges(0);
  __threadfence();
  grid.sync();

  // every lane loads (a broadcast dummy where it has no edge) and selects:
  // no divergence around the shuffles
  auto west = [&](double2 v, int r, int b) -> double {
    const double sh = __shfl_up_sync(FULL_MASK, v.y, 1);
    const double t = k.wp[b * k.wbs + r];
    return k.wld ? t : sh;
  };
  auto east = [&](double2 v, int r, int b) -> double {
    const double sh = __shfl_down_sync(FULL_MASK, v.x, 1);
    const double t = k.ep[b * k.ebs + r];
    return k.eld ? t : sh;
  };
  // one pair of row r from rows S (r-1), C (r), N (r+1) of buffer b's iterate;
  // res = the residuals (0 on lanes past the last pair)
  auto pair = [&](double2 S, double2 C, double2 N, int r, int b, double2& res) -> double2 {
    const double cw = west(C, r, b), ce = east(C, r, b);
    double sw = 0.0, se = 0.0, nw = 0.0, ne = 0.0;
    if (ST) {
      sw = west(S, r - 1, b);
      se = east(S, r - 1, b);
      nw = west(N, r + 1, b);
      ne = east(N, r + 1, b);
    }
    const double2 f = *reinterpret_cast<const double2*>(k.F + (size_t)(r - 1) * nx + k.xs);
    double2 o;
    if (P2) {
      // power-of-two h and λ, 5-point: -4c, scale·L and λr are exact, so
      // each fused multiply-add rounds exactly like the separate ops
      const double L0 = fma(-4.0, C.x, __dadd_rn(__dadd_rn(__dadd_rn(cw, C.y), S.x), N.x));
      const double L1 = fma(-4.0, C.y, __dadd_rn(__dadd_rn(__dadd_rn(C.x, ce), S.y), N.y));
      res.x = fma(p.scale, L0, -f.x);
      res.y = fma(p.scale, L1, -f.y);
      o = make_double2(fma(p.lambda, res.x, C.x), fma(p.lambda, res.y, C.y));
    } else {
      const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
      const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
      res.x = __dsub_rn(__dmul_rn(p.scale, L0), f.x);
      res.y = __dsub_rn(__dmul_rn(p.scale, L1), f.y);
      o = make_double2(__dadd_rn(C.x, __dmul_rn(p.lambda, res.x)), __dadd_rn(C.y, __dmul_rn(p.lambda, res.y)));
    }
    if (!k.act) res = make_double2(0.0, 0.0);
    return o;
  };
  auto acc = [&](double2 res, unsigned long long& mx, double& ss) {
    mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(res.x)));
    ss = fma(res.x, res.x, ss);
    mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(res.y)));
    ss = fma(res.y, res.y, ss);
  };

  int entry = 0, phase = 0;  // phase = s mod every (no division per sweep)
#if PX_RR_PROF
  long long tp[7] = {0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define RR_T(i)                  \
  {                              \
    const long long t_ = clock64(); \
    tp[i] += t_ - tq;            \
    tq = t_;                     \
  }
#else
#define RR_T(i)
#endif
  for (int s = 0; s < p.nsweeps; ++s) {
    const int b = s & 1;
    const bool rec = p.every > 0 && phase == 0;
    if (++phase == p.every) phase = 0;
    const uint32_t tag = (uint32_t)s + 1u;
    const int slot = (s + 1) & 1;
    double* mine = k.pub + (size_t)(slot * G + c) * 2 * 2 * nx;
    // the update of the CTA's rows, compiled once with and once without the
    // norm accumulation: no branch between the rows, so the scheduler
    // interleaves their independent expression trees
    auto rows = [&](auto rec_c) {
      constexpr bool REC = decltype(rec_c)::value;
      unsigned long long mx = 0ull;
      double ss = 0.0;
      // row R, then row 1: both published at once
      double2 rR = make_double2(0.0, 0.0), r1;
      const double2 nR = RR > 1 ? pair(cur[RR - 1], cur[RR], cur[RR + 1], RR, b, rR) : make_double2(0.0, 0.0);
      const double2 n1 = pair(cur[0], cur[1], cur[2], 1, b, r1);
      if (REC) {
        acc(r1, mx, ss);
        if (RR > 1) acc(rR, mx, ss);
      }
#if PX_RR_PROF
      {  // the compute of rows R and 1 complete (consume the results)
        if (__double_as_longlong(n1.x) == 1 && __double_as_longlong(nR.y) == 3) tp[0] += 1;
      }
      RR_T(6)
#endif
      // pair q of a published row = the 32-B entry at 4q (a warp writes 1 KB contiguously)
      if (k.act) {
        if (k.top_x) ll_put2(mine + 2 * x, n1, tag);
        if (k.bot_x) ll_put2(mine + 2 * nx + 2 * x, RR > 1 ? nR : n1, tag);
      }
      RR_T(0)
      // rows 2..R-1 from the old iterate (written back after the last of them)
      double2 o[RR > 2 ? RR - 2 : 1];
#pragma unroll
      for (int r = 2; r < RR; ++r) {
        double2 res;
        o[r - 2] = pair(cur[r - 1], cur[r], cur[r + 1], r, b, res);
        if (REC) acc(res, mx, ss);
      }
#pragma unroll
      for (int r = 2; r < RR; ++r) cur[r] = o[r - 2];
      cur[1] = n1;
      if (RR > 1) cur[RR] = nR;
      RR_T(1)
      if (REC) {
        rs_block_reduce(mx, ss, k.part + ((size_t)entry * G + c) * 2);
        ++entry;
      }
    };
    if (rec)
      rows(std::true_type{});
    else
      rows(std::false_type{});
    RR_T(2)
    // halo rows of φ^{s+1}
    if (k.act && (k.top_x || k.bot_x)) {
      const double* fu = k.pub + ((size_t)(slot * G + k.up) * 2 + 1) * 2 * nx;  // up's last row
      const double* fd = k.pub + ((size_t)(slot * G + k.dn) * 2) * 2 * nx;      // dn's first row
      double2 v[2];
      if (k.top_x && k.bot_x) {
        const double* const e[2] = {fu + 2 * x, fd + 2 * x};
        ll_get2<2>(e, tag, v);
      } else {
        const double* const e[2] = {(k.top_x ? fu : fd) + 2 * x, fu};
        ll_get2<1>(e, tag, v);
        v[1] = v[0];
      }
      if (k.top_x) cur[0] = v[0];
      if (k.bot_x) cur[RR + 1] = v[1];
    }
    RR_T(3)
    if (k.refl_top) cur[0] = make_double2(-cur[1].x, -cur[1].y);
    if (k.refl_bot) cur[RR + 1] = make_double2(-cur[RR].x, -cur[RR].y);
    put_edges(b ^ 1);
    RR_T(4)
    __syncthreads();
    RR_T(5)
  }
#if PX_RR_PROF
  if ((threadIdx.x == 0 || threadIdx.x == 480) && (c == 0 || c == 74))
    printf("RRPROF cta %d thr %d R %d: rows1R %.0f publish %.0f inner %.0f reduce %.0f poll %.0f edges %.0f bar %.0f cycles/sweep\n", c,
           threadIdx.x, RR, (double)tp[6] / p.nsweeps, (double)tp[0] / p.nsweeps, (double)tp[1] / p.nsweeps, (double)tp[2] / p.nsweeps,
           (double)tp[3] / p.nsweeps, (double)tp[4] / p.nsweeps, (double)tp[5] / p.nsweeps);
#endif
#undef RR_T
  const int bN = p.nsweeps & 1;  // the edge buffer of φ^N
  if (p.final_norm) {            // rows 1..R in order (k_resident's final pass)
    unsigned long long mx = 0ull;
    double ss = 0.0;
#pragma unroll
    for (int r = 1; r <= RR; ++r) {
      double2 res;
      pair(cur[r - 1], cur[r], cur[r + 1], r, bN, res);
      acc(res, mx, ss);
    }
    rs_block_reduce(mx, ss, k.part + ((size_t)entry * G + c) * 2);
    ++entry;
  }
  __threadfence();
  grid.sync();
  for (int e = c; e < entry; e += G) {
    unsigned long long m = 0ull;
    double t = 0.0;
    for (int i = tid; i < G; i += RS_THREADS) {
      m = umax64(m, (unsigned long long)__double_as_longlong(__ldcg(k.part + ((size_t)e * G + i) * 2)));
      t = t + __ldcg(k.part + ((size_t)e * G + i) * 2 + 1);
    }
    double out[2];
    rs_block_reduce(m, t, out);
    if (tid == 0) {
      p.d_max[e] = out[0];
      p.d_sum[e] = out[1];
    }
  }
  // φ^N with its ghost columns; the face CTAs also write their halo row (the
  // domain's ghost row)
  const bool first = x == 0, last = x == nx - 2;
#pragma unroll
  for (int r = 0; r < RR + 2; ++r) {
    if ((r == 0 && c != 0) || (r == RR + 1 && c != G - 1)) continue;
    const double w = west(cur[r], r, bN), e = east(cur[r], r, bN);
    if (k.act) {
      double* dst = p.phi_out + (int64_t)(y0 - 1 + r) * p.ld_out + x;
      dst[0] = cur[r].x;
      dst[1] = cur[r].y;
      if (first) dst[-1] = w;
      if (last) dst[2] = e;
    }
  }
}

// Shared layout and per-thread context of the register-resident kernels
// (H halo rows per side, RE row slots): ρ rows | eL[2][NWP][RE] |
// eR[2][NWP][RE] | gW[2][RE] | gE[2][RE]; the LL mailbox (H rows per side)
// and the norm partials in the workspace.
template <int RE, int H>
__device__ __forceinline__ void rr_setup(const ResidentLaunch& p, RrCtx& k, double* sm) {
  constexpr int NWP = RS_THREADS / 32, BS = NWP * RE;
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = p.nx, np = nx / 2;
  const int y0 = (int)((int64_t)c * p.ny / G), y1 = (int)((int64_t)(c + 1) * p.ny / G), R = y1 - y0;
  double* F = sm;
  k.F = F;
  k.eL = F + (size_t)(p.rmax + 2 * (H - 1)) * nx;
  k.eR = k.eL + 2 * BS;
  k.gW = k.eR + 2 * BS;
  k.gE = k.gW + 2 * RE;
  // [slot][cta][side][H rows][2 nx doubles], 32-B aligned (the workspace is cudaMalloc'ed)
  k.pub = p.ws + ((G + 3) & ~3);
  k.part = k.pub + (size_t)2 * G * 2 * H * 2 * nx;  // [entry][cta][max, sum]
  k.G = G;
  k.c = c;
  k.nx = nx;
  k.warp = warp;
  k.up = c > 0 ? c - 1 : G - 1;
  k.dn = c < G - 1 ? c + 1 : 0;
  k.top_x = c > 0 || p.ymode[0] == GH_WRAP;
  k.bot_x = c < G - 1 || p.ymode[1] == GH_WRAP;
  k.refl_top = !k.top_x && p.ymode[0] == GH_REFLECT;
  k.refl_bot = !k.bot_x && p.ymode[1] == GH_REFLECT;
  const int q = tid;
  k.act = q < np;
  k.x = 2 * q;
  k.xs = k.act ? k.x : 0;
  const bool first = q == 0, last = q == np - 1;
  const int wlast = (np - 1) >> 5;  // the warp holding column nx-1
  k.st_l = lane == 0;
  k.st_r = (lane == 31 && k.act) || last;
  k.st_gw = first && p.xmode[0] == GH_REFLECT;
  k.st_ge = last && p.xmode[1] == GH_REFLECT;
  // west candidate of column 2q: the previous warp's right edge, or at the
  // domain face the last warp's right edge (periodic) / the ghost column
  k.wp = k.gW;
  k.wbs = 0;
  k.wld = false;
  if (first) {
    k.wld = true;
    k.wbs = p.xmode[0] == GH_WRAP ? BS : RE;
    if (p.xmode[0] == GH_WRAP) k.wp = k.eR + wlast * RE;
  } else if (lane == 0) {
    k.wp = k.eR + (warp - 1) * RE;
    k.wbs = BS;
    k.wld = true;
  }
  k.ep = k.gE;
  k.ebs = 0;
  k.eld = false;
  if (last) {
    k.eld = true;
    k.ebs = p.xmode[1] == GH_WRAP ? BS : RE;
    if (p.xmode[1] == GH_WRAP) k.ep = k.eL;
  } else if (lane == 31 && k.act) {
    k.ep = k.eL + (warp + 1) * RE;
    k.ebs = BS;
    k.eld = true;
  }
  // ρ of the owned rows, and with H = 2 also of the inner halo rows (level 1
  // updates them): F row r = global row y0 - (H-1) + r (periodic wrap; rows
  // outside a non-periodic domain are never used)
  for (int r = 0; r < R + 2 * (H - 1); ++r) {
    int y = y0 - (H - 1) + r;
    y = y < 0 ? y + p.ny : (y >= p.ny ? y - p.ny : y);
    for (int i = tid; i < nx; i += RS_THREADS) F[(size_t)r * nx + i] = p.rhs[(int64_t)y * p.ld_rhs + i];
  }
  if (tid < RE) {  // fixed ghost columns of slots 0 .. R+2H-1 (both buffers)
    const int y = y0 - H + tid;
    const bool ok = tid < R + 2 * H && y >= -1 && y <= p.ny;
    const double w = ok ? p.phi_in[(int64_t)y * p.ld_in - 1] : 0.0;
    const double e = ok ? p.phi_in[(int64_t)y * p.ld_in + nx] : 0.0;
    k.gW[tid] = k.gW[RE + tid] = w;
    k.gE[tid] = k.gE[RE + tid] = e;
  }
  for (int sl = 0; sl < 2; ++sl)
    for (int i = tid; i < 2 * H * 2 * nx; i += RS_THREADS) k.pub[(size_t)(sl * G + c) * 2 * H * 2 * nx + i] = 0.0;
  __syncthreads();
}

template <int ST, bool P2>
__global__ void __launch_bounds__(RS_THREADS, 1) k_resident_reg(const ResidentLaunch p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  RrCtx k;
  rr_setup<RR_RM + 2, 1>(p, k, sm);
  const int R = (int)((int64_t)(blockIdx.x + 1) * p.ny / gridDim.x) - (int)((int64_t)blockIdx.x * p.ny / gridDim.x);
  switch (R) {
    case 1: rr_body<ST, 1, P2>(p, k, grid); break;
    case 2: rr_body<ST, 2, P2>(p, k, grid); break;
    case 3: rr_body<ST, 3, P2>(p, k, grid); break;
    case 4: rr_body<ST, 4, P2>(p, k, grid); break;
    case 5: rr_body<ST, 5, P2>(p, k, grid); break;
    case 6: rr_body<ST, 6, P2>(p, k, grid); break;
    default: rr_body<ST, 7, P2>(p, k, grid); break;
  }
}

// ---------------------------------------------------------------------------
// k_resident_reg2<ST>: k_resident_reg with TEMPORAL BLOCKING of the mailbox
// handshake -- two sweeps per hop.  A thread keeps its pair of the CTA's rows
// and of TWO halo rows on each side (rows -1 .. R+2) in registers.  A pass of
// two levels: level 1 updates rows 0 .. R+1 (the inner halo rows redundantly,
// exactly as their owners update them; at a non-periodic domain face the
// ghost row is re-derived instead: odd reflection of row 1 / R, or the fixed
// φ^0 row), edges, barrier; level 2 updates rows 1 .. R -- rows 1, 2, R-1, R
// first, published to the L2 mailbox at once (2 rows per side), then the
// inner rows -- then the neighbours' rows are fetched into the four halo
// rows, edges, barrier.  The L2 hop (≈ 1.6 µs with its barrier on the B200,
// scripts/ll_latency.cu) is paid once per two sweeps for two redundant row
// updates per pass.  An odd sweep count ends with a one-level pass.  φ and
// the max-norm bit-identical to k_resident; the per-thread Σr² order is row
// order (within the oracle tolerance, not bitwise equal to k_resident's).
template <int ST, int RR, bool P2>
__device__ __forceinline__ void rr2_body(const ResidentLaunch& p, const RrCtx& k, cg::grid_group& grid) {
  constexpr int NWP = RS_THREADS / 32, RE = RR_RM + 4, BS = NWP * RE, NI = RR + 4;  // i = row + 1
  const int tid = threadIdx.x, nx = k.nx, x = k.x, G = k.G, c = k.c;
  const int y0 = (int)((int64_t)c * p.ny / G);
  const bool wrap_y = p.ymode[0] == GH_WRAP;
  double2 cur[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    cur[i] = make_double2(0.0, 0.0);
    int y = y0 - 2 + i;
    if (wrap_y) y = y < -1 ? y + p.ny : (y > p.ny ? y - p.ny : y);
    if (k.act && y >= -1 && y <= p.ny) {
      const double* src = p.phi_in + (int64_t)y * p.ld_in + x;
      cur[i] = make_double2(src[0], src[1]);
    }
  }
  auto put_edges = [&](int b) {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (k.st_l) k.eL[b * BS + k.warp * RE + i] = cur[i].x;
      if (k.st_r) k.eR[b * BS + k.warp * RE + i] = cur[i].y;
      if (k.st_gw) k.gW[b * RE + i] = -cur[i].x;
      if (k.st_ge) k.gE[b * RE + i] = -cur[i].y;
    }
  };
  put_edges(0);
  __threadfence();
  grid.sync();

  auto west = [&](double2 v, int i, int b) -> double {
    const double sh = __shfl_up_sync(FULL_MASK, v.y, 1);
    const double t = k.wp[b * k.wbs + i];
    return k.wld ? t : sh;
  };
  auto east = [&](double2 v, int i, int b) -> double {
    const double sh = __shfl_down_sync(FULL_MASK, v.x, 1);
    const double t = k.ep[b * k.ebs + i];
    return k.eld ? t : sh;
  };
  // one pair of slot i (row i-1) from slots i-1, i, i+1 of buffer b's level
  auto pair = [&](double2 S, double2 C, double2 N, int i, int b, double2& res) -> double2 {
    const double cw = west(C, i, b), ce = east(C, i, b);
    double sw = 0.0, se = 0.0, nw = 0.0, ne = 0.0;
    if (ST) {
      sw = west(S, i - 1, b);
      se = east(S, i - 1, b);
      nw = west(N, i + 1, b);
      ne = east(N, i + 1, b);
    }
    const double2 f = *reinterpret_cast<const double2*>(k.F + (size_t)(i - 1) * nx + k.xs);  // ρ of row i-1
    double2 o;
    if (P2) {  // as k_resident_reg
      const double L0 = fma(-4.0, C.x, __dadd_rn(__dadd_rn(__dadd_rn(cw, C.y), S.x), N.x));
      const double L1 = fma(-4.0, C.y, __dadd_rn(__dadd_rn(__dadd_rn(C.x, ce), S.y), N.y));
      res.x = fma(p.scale, L0, -f.x);
      res.y = fma(p.scale, L1, -f.y);
      o = make_double2(fma(p.lambda, res.x, C.x), fma(p.lambda, res.y, C.y));
    } else {
      const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
      const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
      res.x = __dsub_rn(__dmul_rn(p.scale, L0), f.x);
      res.y = __dsub_rn(__dmul_rn(p.scale, L1), f.y);
      o = make_double2(__dadd_rn(C.x, __dmul_rn(p.lambda, res.x)), __dadd_rn(C.y, __dmul_rn(p.lambda, res.y)));
    }
    if (!k.act) res = make_double2(0.0, 0.0);
    return o;
  };
  auto acc = [&](double2 res, unsigned long long& mx, double& ss) {
    mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(res.x)));
    ss = fma(res.x, res.x, ss);
    mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(res.y)));
    ss = fma(res.y, res.y, ss);
  };
  const bool top_face = !k.top_x, bot_face = !k.bot_x;  // non-periodic domain faces
  // ghost row of a domain face after a level: reflection of the first / last
  // owned row, or (fixed ghosts) untouched
  auto face_rows = [&]() {
    if (k.refl_top) cur[1] = make_double2(-cur[2].x, -cur[2].y);
    if (k.refl_bot) cur[RR + 2] = make_double2(-cur[RR + 1].x, -cur[RR + 1].y);
  };
  int entry = 0, cb = 0;
  int pass = 0;
  for (int s = 0; s < p.nsweeps; s += 2, ++pass) {
    const int L = p.nsweeps - s >= 2 ? 2 : 1;
    const uint32_t tag = (uint32_t)pass + 1u;
    const int slot = (pass + 1) & 1;
    double* mine = k.pub + (size_t)(slot * G + c) * 2 * 2 * 2 * nx;  // [side][row][2 nx]
    // rows 1, 2 (f0, f1) to the first side, rows R-1, R (l0, l1) to the last
    // (a pair as one 32-B LL entry at 4q = 2x doubles of its row)
    auto publish = [&](double2 f0, double2 f1, double2 l0, double2 l1) {
      if (k.act) {
        if (k.top_x) {
          ll_put2(mine + 2 * x, f0, tag);
          ll_put2(mine + 2 * nx + 2 * x, f1, tag);
        }
        if (k.bot_x) {
          ll_put2(mine + 4 * nx + 2 * x, l0, tag);
          ll_put2(mine + 6 * nx + 2 * x, l1, tag);
        }
      }
    };
    // ---- level 1: rows 0 .. R+1 (slots 1 .. R+2), in place with a rolling old row
    {
      const bool rec = p.every > 0 && s % p.every == 0;
      unsigned long long mx = 0ull;
      double ss = 0.0;
      double2 prev = cur[0];  // the old row above (level 1 updates in place, in row order)
#pragma unroll
      for (int i = 1; i <= RR + 2; ++i) {
        const bool skip = (i == 1 && top_face) || (i == RR + 2 && bot_face);
        if (!skip) {
          double2 res;
          const double2 o = pair(prev, cur[i], cur[i + 1], i, cb, res);
          if (rec && i >= 2 && i <= RR + 1) acc(res, mx, ss);
          prev = cur[i];
          cur[i] = o;
        } else {
          prev = cur[i];
        }
      }
      face_rows();
      if (rec) {
        rs_block_reduce(mx, ss, k.part + ((size_t)entry * G + c) * 2);
        ++entry;
      }
    }
    if (L == 2) {
      put_edges(cb ^ 1);
      __syncthreads();
      cb ^= 1;
      // ---- level 2: rows 1 .. R; rows 1, 2, R-1, R first (published), then 3 .. R-2
      const bool rec = p.every > 0 && (s + 1) % p.every == 0;
      unsigned long long mx = 0ull;
      double ss = 0.0;
      double2 t[4], rt[4];
      // boundary slots 2, 3, RR, RR+1 (the distinct ones)
      constexpr int b0 = 2, b1 = 3, b2 = RR, b3 = RR + 1;
      constexpr bool u2 = b2 > b1, u3 = b3 > b1 && b3 > b2;
      t[0] = pair(cur[b0 - 1], cur[b0], cur[b0 + 1], b0, cb, rt[0]);
      t[1] = pair(cur[b1 - 1], cur[b1], cur[b1 + 1], b1, cb, rt[1]);
      if (u2) t[2] = pair(cur[b2 - 1], cur[b2], cur[b2 + 1], b2, cb, rt[2]);
      if (u3) t[3] = pair(cur[b3 - 1], cur[b3], cur[b3 + 1], b3, cb, rt[3]);
      // the last two rows: slots RR, RR+1
      const double2 l0 = RR == 2 ? t[0] : (RR == 3 ? t[1] : t[2]);
      const double2 l1 = RR == 2 ? t[1] : t[3];
      publish(t[0], t[1], l0, l1);
      // inner rows 3 .. R-2 (slots 4 .. RR-1) from the old level
      double2 inner[RR > 4 ? RR - 4 : 1];
#pragma unroll
      for (int i = 4; i <= RR - 1; ++i) {
        double2 res;
        inner[i - 4] = pair(cur[i - 1], cur[i], cur[i + 1], i, cb, res);
        if (rec) acc(res, mx, ss);
      }
      cur[b0] = t[0];
      cur[b1] = t[1];
      if (u2) cur[b2] = t[2];
      if (u3) cur[b3] = t[3];
#pragma unroll
      for (int i = 4; i <= RR - 1; ++i) cur[i] = inner[i - 4];
      if (rec) {
        acc(rt[0], mx, ss);
        acc(rt[1], mx, ss);
        if (u2) acc(rt[2], mx, ss);
        if (u3) acc(rt[3], mx, ss);
        rs_block_reduce(mx, ss, k.part + ((size_t)entry * G + c) * 2);
        ++entry;
      }
    } else {
      publish(cur[2], cur[3], cur[RR], cur[RR + 1]);
    }
    face_rows();
    // the neighbours' rows of this pass's iterate into the halo slots 0, 1 / R+2, R+3
    if (k.act && (k.top_x || k.bot_x)) {
      const double* fu = k.pub + ((size_t)(slot * G + k.up) * 2 + 1) * 2 * 2 * nx;  // up's last rows
      const double* fd = k.pub + ((size_t)(slot * G + k.dn) * 2) * 2 * 2 * nx;      // dn's first rows
      if (k.top_x && k.bot_x) {
        const double* const e[4] = {fu + 2 * x, fu + 2 * nx + 2 * x, fd + 2 * x, fd + 2 * nx + 2 * x};
        double2 v[4];
        ll_get2<4>(e, tag, v);
        cur[0] = v[0];
        cur[1] = v[1];
        cur[RR + 2] = v[2];
        cur[RR + 3] = v[3];
      } else {
        const double* f = k.top_x ? fu : fd;
        const double* const e[2] = {f + 2 * x, f + 2 * nx + 2 * x};
        double2 v[2];
        ll_get2<2>(e, tag, v);
        if (k.top_x) {
          cur[0] = v[0];
          cur[1] = v[1];
        } else {
          cur[RR + 2] = v[0];
          cur[RR + 3] = v[1];
        }
      }
    }
    put_edges(cb ^ 1);
    __syncthreads();
    cb ^= 1;
  }
  const int bN = cb;  // the edge buffer of φ^N
  if (p.final_norm) {  // rows 1..R in order (k_resident's final pass)
    unsigned long long mx = 0ull;
    double ss = 0.0;
#pragma unroll
    for (int i = 2; i <= RR + 1; ++i) {
      double2 res;
      pair(cur[i - 1], cur[i], cur[i + 1], i, bN, res);
      acc(res, mx, ss);
    }
    rs_block_reduce(mx, ss, k.part + ((size_t)entry * G + c) * 2);
    ++entry;
  }
  __threadfence();
  grid.sync();
  for (int e = c; e < entry; e += G) {
    unsigned long long m = 0ull;
    double t = 0.0;
    for (int i = tid; i < G; i += RS_THREADS) {
      m = umax64(m, (unsigned long long)__double_as_longlong(__ldcg(k.part + ((size_t)e * G + i) * 2)));
      t = t + __ldcg(k.part + ((size_t)e * G + i) * 2 + 1);
    }
    double out[2];
    rs_block_reduce(m, t, out);
    if (tid == 0) {
      p.d_max[e] = out[0];
      p.d_sum[e] = out[1];
    }
  }
  const bool first = x == 0, last = x == nx - 2;
#pragma unroll
  for (int i = 1; i <= RR + 2; ++i) {
    if ((i == 1 && c != 0) || (i == RR + 2 && c != G - 1)) continue;
    const double w = west(cur[i], i, bN), e = east(cur[i], i, bN);
    if (k.act) {
      double* dst = p.phi_out + (int64_t)(y0 - 2 + i) * p.ld_out + x;
      dst[0] = cur[i].x;
      dst[1] = cur[i].y;
      if (first) dst[-1] = w;
      if (last) dst[2] = e;
    }
  }
}

template <int ST, bool P2>
__global__ void __launch_bounds__(RS_THREADS, 1) k_resident_reg2(const ResidentLaunch p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  RrCtx k;
  rr_setup<RR_RM + 4, 2>(p, k, sm);
  const int R = (int)((int64_t)(blockIdx.x + 1) * p.ny / gridDim.x) - (int)((int64_t)blockIdx.x * p.ny / gridDim.x);
  switch (R) {
    case 2: rr2_body<ST, 2, P2>(p, k, grid); break;
    case 3: rr2_body<ST, 3, P2>(p, k, grid); break;
    case 4: rr2_body<ST, 4, P2>(p, k, grid); break;
    case 5: rr2_body<ST, 5, P2>(p, k, grid); break;
    case 6: rr2_body<ST, 6, P2>(p, k, grid); break;
    default: rr2_body<ST, 7, P2>(p, k, grid); break;
  }
}

// ---------------------------------------------------------------------------
// k_resident_tb<ST, K>: the same resident solve with TEMPORAL BLOCKING of the
// row exchange -- K sweeps per neighbour handshake.  CTA c keeps its rows and
// K halo rows on each neighbour side (shared rows i = 0 .. R+2K-1, owned
// i = K .. K+R-1, global row y0-K+i).  A round of K levels computes, at level
// t, the rows whose inputs are still valid: on a side exchanged with a
// neighbour the valid range shrinks by one row per level (redundant halo
// compute -- the halo rows are advanced exactly like the neighbour advances
// its own rows, so the owned results are bit-identical); on a reflecting or
// fixed domain face the owned rows are computed at every level and the
// first ghost row is re-derived (reflection) or kept (fixed).  Then the CTA
// publishes its first and last K owned rows and copies its neighbours' into
// its halo: one handshake per K sweeps instead of one per sweep.  The
// right-hand side is read from global memory (L2-resident) so that the two
// copies of the taller row block fit in shared memory.
constexpr int RT_MAXROWS = 16;  // rows a thread walks per level (ρ prefetched into registers)
template <int ST, bool WRITE>
__device__ __forceinline__ void rt_rows(const double* A, double* B, const double* rhs, int64_t ld_rhs, int P, int nx,
                                        int rlo, int rhi, int y_of_i0, int ny, bool wrap, double scale,
                                        double lambda, bool norm, int nlo, int nhi, unsigned long long& mx,
                                        double& ss) {
  for (int q = threadIdx.x; q < nx / 2; q += blockDim.x) {
    const int x = 2 * q + 2;
    // the right-hand side of the whole column walk first: one L2 round trip
    // per level instead of one per row
    double2 fr[RT_MAXROWS];
#pragma unroll
    for (int j = 0; j < RT_MAXROWS; ++j) {
      const int r = rlo + j;
      if (r <= rhi) {
        int y = y_of_i0 + r;
        if (wrap) y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
        fr[j] = __ldg(reinterpret_cast<const double2*>(rhs + (int64_t)y * ld_rhs + (x - 2)));
      }
    }
    const double* a0 = A + (size_t)(rlo - 1) * P + x;
    double2 S = *reinterpret_cast<const double2*>(a0);
    double2 C = *reinterpret_cast<const double2*>(a0 + P);
    double sw = a0[-1], se = a0[2], cw = a0[P - 1], ce = a0[P + 2];
#pragma unroll
    for (int j = 0; j < RT_MAXROWS; ++j) {
      const int r = rlo + j;
      if (r > rhi) break;
      const double* an = A + (size_t)(r + 1) * P + x;
      const double2 N = *reinterpret_cast<const double2*>(an);
      const double nw = an[-1], ne = an[2];
      const double L0 = rs_taps<ST>(cw, C.y, S.x, N.x, C.x, sw, S.y, nw, N.y);
      const double L1 = rs_taps<ST>(C.x, ce, S.y, N.y, C.y, S.x, se, N.x, ne);
      const double2 f = fr[j];
      const double r0 = __dsub_rn(__dmul_rn(scale, L0), f.x);
      const double r1 = __dsub_rn(__dmul_rn(scale, L1), f.y);
      if (WRITE) {
        double2 o;
        o.x = __dadd_rn(C.x, __dmul_rn(lambda, r0));
        o.y = __dadd_rn(C.y, __dmul_rn(lambda, r1));
        *reinterpret_cast<double2*>(B + (size_t)r * P + x) = o;
      }
      if (norm && r >= nlo && r <= nhi) {
        mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r0)));
        ss = fma(r0, r0, ss);
        mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(r1)));
        ss = fma(r1, r1, ss);
      }
      S = C;
      sw = cw;
      se = ce;
      C = N;
      cw = nw;
      ce = ne;
    }
  }
}

template <int ST, int K>
__global__ void __launch_bounds__(RS_THREADS, 1) k_resident_tb(const ResidentLaunch p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int nx = p.nx, ny = p.ny, P = nx + 4;
  const int y0 = (int)((int64_t)c * ny / G), y1 = (int)((int64_t)(c + 1) * ny / G), R = y1 - y0;
  const int NR = R + 2 * K;  // shared rows
  double* A = sm;
  double* B = A + (size_t)(p.rmax + 2 * K) * P;
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(p.ws);
  double* pub = p.ws + G;                                // [slot][cta][first, last][K][nx]
  double* part = pub + (size_t)2 * G * 2 * K * nx;       // [entry][cta][max, sum]
  const int up = c > 0 ? c - 1 : G - 1, dn = c < G - 1 ? c + 1 : 0;
  const bool wrap = p.ymode[0] == GH_WRAP;
  const bool top_x = c > 0 || wrap;       // halo rows 0..K-1 from CTA `up`
  const bool bot_x = c < G - 1 || wrap;   // halo rows R+K..R+2K-1 from CTA `dn`
  const int xm[2] = {p.xmode[0], p.xmode[1]};
  const int yb = y0 - K;                  // global row of shared row 0

  // φ^0: owned rows, the neighbour halos (global rows, wrapped on the
  // periodic ring) and the first ghost row at a domain face, into both copies
  for (int i = 0; i < NR; ++i) {
    int y = yb + i;
    const bool own = i >= K && i < K + R;
    bool load = own || (i < K && top_x) || (i >= K + R && bot_x) || (i == K - 1 && !top_x) || (i == K + R && !bot_x);
    if (!load) continue;
    if (wrap) y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
    const double* src = p.phi_in + (int64_t)y * p.ld_in;
    for (int x = tid - 1; x <= nx; x += nt) {
      const double v = src[x];
      A[(size_t)i * P + x + 2] = v;
      B[(size_t)i * P + x + 2] = v;
    }
  }
  if (tid == 0) flags[c] = 0ull;
  __threadfence();
  grid.sync();

  int entry = 0, s = 0, round = 0;
  while (s < p.nsweeps) {
    const int kk = p.nsweeps - s < K ? p.nsweeps - s : K;  // levels of this round
    for (int t = 1; t <= kk; ++t) {
      // valid range at level t (shrinks on exchanged sides only)
      const int lo = top_x ? t : K, hi = bot_x ? NR - 1 - t : K + R - 1;
      const bool rec = p.every > 0 && (s % p.every) == 0;
      unsigned long long mx = 0ull;
      double ss = 0.0;
      rt_rows<ST, true>(A, B, p.rhs, p.ld_rhs, P, nx, lo, hi, yb, ny, wrap, p.scale, p.lambda, rec, K, K + R - 1,
                        mx, ss);
      __syncthreads();
      // domain faces: the first ghost row by reflection (fixed: kept)
      for (int x = tid; x < nx; x += nt) {
        if (!top_x && p.ymode[0] == GH_REFLECT) B[(size_t)(K - 1) * P + x + 2] = -B[(size_t)K * P + x + 2];
        if (!bot_x && p.ymode[1] == GH_REFLECT) B[(size_t)(K + R) * P + x + 2] = -B[(size_t)(K + R - 1) * P + x + 2];
      }
      __syncthreads();
      const int glo = top_x ? lo : K - 1, ghi = bot_x ? hi : K + R;
      for (int r = glo + tid; r <= ghi; r += nt) rs_xghost(B + (size_t)r * P, nx, xm);
      if (rec) {
        rs_block_reduce(mx, ss, part + ((size_t)entry * G + c) * 2);
        ++entry;
      } else {
        __syncthreads();
      }
      double* tmp = A;
      A = B;
      B = tmp;
      ++s;
    }
    // handshake: publish the first and last K owned rows, take the neighbours'
    const int slot = (round + 1) & 1;
    double* mine = pub + (size_t)(slot * G + c) * 2 * K * nx;
    for (int j = 0; j < K; ++j)
      for (int x = tid; x < nx; x += nt) {
        __stcg(mine + (size_t)j * nx + x, A[(size_t)(K + j) * P + x + 2]);
        __stcg(mine + (size_t)(K + j) * nx + x, A[(size_t)(R + j) * P + x + 2]);
      }
    __syncthreads();
    ++round;
    if (tid == 0) st_release(flags + c, (unsigned long long)round);
    if (tid == 0 && top_x)
      while (ld_acquire(flags + up) < (unsigned long long)round) {
      }
    if (tid == 32 && bot_x)
      while (ld_acquire(flags + dn) < (unsigned long long)round) {
      }
    __syncthreads();
    const double* fu = pub + ((size_t)(slot * G + up) * 2 + 1) * K * nx;  // up's last K rows
    const double* fd = pub + ((size_t)(slot * G + dn) * 2) * K * nx;      // dn's first K rows
    for (int j = 0; j < K; ++j)
      for (int x = tid; x < nx; x += nt) {
        if (top_x) A[(size_t)j * P + x + 2] = __ldcg(fu + (size_t)j * nx + x);
        if (bot_x) A[(size_t)(K + R + j) * P + x + 2] = __ldcg(fd + (size_t)j * nx + x);
      }
    __syncthreads();
    for (int r = tid; r < NR; r += nt)
      if ((r < K && top_x) || (r >= K + R && bot_x)) rs_xghost(A + (size_t)r * P, nx, xm);
    __syncthreads();
  }
  if (p.final_norm) {
    unsigned long long mx = 0ull;
    double ss = 0.0;
    rt_rows<ST, false>(A, nullptr, p.rhs, p.ld_rhs, P, nx, K, K + R - 1, yb, ny, wrap, p.scale, p.lambda, true, K,
                       K + R - 1, mx, ss);
    rs_block_reduce(mx, ss, part + ((size_t)entry * G + c) * 2);
    ++entry;
  }
  __threadfence();
  grid.sync();
  for (int e = c; e < entry; e += G) {
    unsigned long long m = 0ull;
    double t = 0.0;
    for (int i = tid; i < G; i += nt) {
      m = umax64(m, (unsigned long long)__double_as_longlong(__ldcg(part + ((size_t)e * G + i) * 2)));
      t = t + __ldcg(part + ((size_t)e * G + i) * 2 + 1);
    }
    double out[2];
    rs_block_reduce(m, t, out);
    if (tid == 0) {
      p.d_max[e] = out[0];
      p.d_sum[e] = out[1];
    }
  }
  for (int i = K; i < K + R; ++i) {
    double* dst = p.phi_out + (int64_t)(yb + i) * p.ld_out;
    for (int x = tid - 1; x <= nx; x += nt) dst[x] = A[(size_t)i * P + x + 2];
  }
  if (c == 0)
    for (int x = tid - 1; x <= nx; x += nt) p.phi_out[-p.ld_out + x] = A[(size_t)(K - 1) * P + x + 2];
  if (c == G - 1)
    for (int x = tid - 1; x <= nx; x += nt) p.phi_out[(int64_t)ny * p.ld_out + x] = A[(size_t)(K + R) * P + x + 2];
}

// rounds of the temporally blocked resident solve: K sweeps per handshake
// (PROTOX_RESIDENT_K = 1, 2 or 3), limited by shared memory and by the rows a
// CTA owns.  Default 1: measured at BASELINE config 2 (1024², 1000 sweeps)
// K = 1 / 2 / 3 run at 252 / 207 / 218 Gcell-updates/s -- the per-level
// barriers and the redundant halo rows cost more than the saved handshakes
// (DESIGN.md §6), so the blocked variant is an A/B option only.
constexpr int RS_KMAX = 3;
static int rs_k_env() {
  static int k = -1;
  if (k < 0) {
    const char* e = getenv("PROTOX_RESIDENT_K");
    k = e ? atoi(e) : 1;
    if (k < 1) k = 1;
    if (k > RS_KMAX) k = RS_KMAX;
  }
  return k;
}

size_t resident_ws_doubles(int nx, int grid, int n_entries) {
  // flags (k_resident_tb) or padding, the row mailboxes (k_resident: 2 slots x 2 rows x nx LL entries
  // of 2 doubles; k_resident_tb: 2 slots x 2K rows x nx), the norm partials
  // k_resident_reg2: 2 slots x 2 sides x 2 rows x nx LL entries of 2 doubles
  return (size_t)grid + 4 + (size_t)2 * grid * 2 * (RS_KMAX > 4 ? RS_KMAX : 4) * nx +
         (size_t)(n_entries > 0 ? n_entries : 1) * grid * 2;
}

static int rs_nsm(int* smem_optin) {
  static int n = 0, opt = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    if (cudaDeviceGetAttribute(&opt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || opt <= 0)
      opt = 227 * 1024;
    cudaGetLastError();
  }
  *smem_optin = opt;
  return n;
}

// K of the resident solve of an nx x ny problem (0: does not fit)
static int resident_k(int nx, int ny, int* grid, int* rmax, size_t* smem) {
  if (nx < 2 || ny < 1 || (nx & 1)) return 0;
  int optin = 0;
  const int nsm = rs_nsm(&optin);
  const int G = ny < nsm ? ny : nsm;
  const int R = (ny + G - 1) / G;
  const int Rmin = ny / G;  // the smallest block: it publishes K owned rows
  for (int K = rs_k_env(); K >= 1; --K) {
    if (K > 1 && R + 2 * K - 2 > RT_MAXROWS) continue;  // rows per level walk
    size_t bytes;
    if (K == 1)
      bytes = ((size_t)2 * (R + 2) * (nx + 4) + (size_t)R * nx) * sizeof(double);
    else
      bytes = (size_t)2 * (R + 2 * K) * (nx + 4) * sizeof(double);
    // leave room for the static shared arrays of the reduction
    if (bytes + 1024 > (size_t)optin || (K > 1 && Rmin < K)) continue;
    *grid = G;
    *rmax = R;
    *smem = bytes;
    return K;
  }
  return 0;
}

bool resident_plan(int nx, int ny, int* grid, int* rmax, size_t* smem) {
  return resident_k(nx, ny, grid, rmax, smem) > 0;
}

template <typename F>
static cudaError_t rs_attr(F* fn, size_t smem, size_t& set) {
  if (set >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) set = smem;
  return e;
}

// PROTOX_RESIDENT_UNROLL=0 selects the rolled column walk (A/B)
static int rs_unroll_env() {
  static int u = -1;
  if (u < 0) {
    const char* e = getenv("PROTOX_RESIDENT_UNROLL");
    u = (e && e[0] == '0') ? 0 : 1;
  }
  return u;
}

static bool rs_pow2(double v) {
  if (!(v > 0.0) || !std::isfinite(v)) return false;
  int e;
  return std::frexp(v, &e) == 0.5;
}

// PROTOX_RESIDENT_REG: 0 = the shared-memory row walk (k_resident), 1 = the
// register-resident kernel, 2 = its two-sweeps-per-hop variant (A/B)
static int rs_reg_env() {
  static int u = -1;
  if (u < 0) {
    const char* e = getenv("PROTOX_RESIDENT_REG");
    u = e ? atoi(e) : 1;
    if (u < 0 || u > 2) u = 1;
  }
  return u;
}

px_status launch_resident(int stencil, const ResidentLaunch& r_in, int grid, size_t smem, cudaStream_t s) {
  ResidentLaunch r = r_in;
  r.unroll = rs_unroll_env();
  int g2 = 0, rm = 0;
  size_t sm2 = 0;
  const int K = resident_k(r.nx, r.ny, &g2, &rm, &sm2);
  if (K < 1 || g2 != grid || sm2 != smem) return fail(PX_ERR_STATE, "resident plan changed");
  static size_t attr_set[2][RS_KMAX] = {};
  const int k = stencil ? 1 : 0;
  void* fn = nullptr;
  cudaError_t e = cudaSuccess;
  const bool reg = K == 1 && rs_reg_env() > 0 && r.rmax <= RR_RM && r.nx / 2 <= RS_THREADS;
  // two sweeps per mailbox hop: every CTA needs two own rows to publish
  const bool reg2 = reg && rs_reg_env() == 2 && r.ny / grid >= 2;
  if (reg2) {
    constexpr int RE = RR_RM + 4;
    smem = ((size_t)(r.rmax + 2) * r.nx + 2 * 2 * (RS_THREADS / 32) * RE + 4 * RE) * sizeof(double);
    static size_t reg2_set[3] = {};
    if (k) {
      e = rs_attr(k_resident_reg2<1, false>, smem, reg2_set[1]);
      fn = (void*)k_resident_reg2<1, false>;
    } else if (rs_pow2(r.scale) && rs_pow2(r.lambda)) {
      e = rs_attr(k_resident_reg2<0, true>, smem, reg2_set[2]);
      fn = (void*)k_resident_reg2<0, true>;
    } else {
      e = rs_attr(k_resident_reg2<0, false>, smem, reg2_set[0]);
      fn = (void*)k_resident_reg2<0, false>;
    }
  } else if (reg) {
    // ρ rows + edge arrays + fixed ghost columns (k_resident_reg's shared layout)
    constexpr int RE = RR_RM + 2;
    smem = ((size_t)r.rmax * r.nx + 2 * 2 * (RS_THREADS / 32) * RE + 4 * RE) * sizeof(double);
    static size_t reg_set[3] = {};
    if (k) {
      e = rs_attr(k_resident_reg<1, false>, smem, reg_set[1]);
      fn = (void*)k_resident_reg<1, false>;
    } else if (rs_pow2(r.scale) && rs_pow2(r.lambda)) {
      e = rs_attr(k_resident_reg<0, true>, smem, reg_set[2]);
      fn = (void*)k_resident_reg<0, true>;
    } else {
      e = rs_attr(k_resident_reg<0, false>, smem, reg_set[0]);
      fn = (void*)k_resident_reg<0, false>;
    }
  } else switch (k * 4 + K) {
    case 1: e = rs_attr(k_resident<0>, smem, attr_set[0][0]); fn = (void*)k_resident<0>; break;
    case 2: e = rs_attr(k_resident_tb<0, 2>, smem, attr_set[0][1]); fn = (void*)k_resident_tb<0, 2>; break;
    case 3: e = rs_attr(k_resident_tb<0, 3>, smem, attr_set[0][2]); fn = (void*)k_resident_tb<0, 3>; break;
    case 5: e = rs_attr(k_resident<1>, smem, attr_set[1][0]); fn = (void*)k_resident<1>; break;
    case 6: e = rs_attr(k_resident_tb<1, 2>, smem, attr_set[1][1]); fn = (void*)k_resident_tb<1, 2>; break;
    case 7: e = rs_attr(k_resident_tb<1, 3>, smem, attr_set[1][2]); fn = (void*)k_resident_tb<1, 3>; break;
    default: return fail(PX_ERR_STATE, "bad resident configuration");
  }
  if (e != cudaSuccess) return cuda_check(e, "resident kernel smem attribute");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(RS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&r};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e == cudaSuccess) e = cudaGetLastError();
  note_kernel(reg2 ? "k_resident_reg2" : (reg ? "k_resident_reg" : (K == 1 ? "k_resident" : "k_resident_tb")));
  count_launches(1);
  return cuda_check(e, "resident solve kernel launch");
}

}  // namespace px
