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

#include <cstdint>
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

// Canonical tap sums (oracle order, each op rounded).
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
// One double per 16-byte entry, each 8-byte half = half the double + the
// sweep tag (NCCL's LL idea): a 16-byte store writes each 8-byte half
// atomically, so a reader that sees the tag in both halves has the whole
// value of that sweep -- no release fence, no flag word, no barrier before
// the publication.
__device__ __forceinline__ void ll_put(double* e, double v, uint32_t tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(e), "r"((uint32_t)b), "r"(tag),
               "r"((uint32_t)(b >> 32)), "r"(tag)
               : "memory");
}
#ifndef LL_BACKOFF_NS
#define LL_BACKOFF_NS 100
#endif
struct LL {
  uint32_t lo, t0, hi, t1;
};
__device__ __forceinline__ LL ll_load(const double* e) {
  LL v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.lo), "=r"(v.t0), "=r"(v.hi), "=r"(v.t1)
               : "l"(e)
               : "memory");
  return v;
}
__device__ __forceinline__ double ll_val(const LL& v) {
  return __longlong_as_double((long long)(((unsigned long long)v.hi << 32) | v.lo));
}
// the n (<= 4) entries e[i], all loads in flight together; re-poll until
// every tag matches
template <int n>
__device__ __forceinline__ void ll_get(const double* const (&e)[4], uint32_t tag, double (&out)[4]) {
  LL v[4];
#pragma unroll
  for (int i = 0; i < n; ++i) v[i] = ll_load(e[i]);
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < n; ++i) ok = ok && v[i].t0 == tag && v[i].t1 == tag;
    if (ok) break;
    if (LL_BACKOFF_NS) __nanosleep(LL_BACKOFF_NS);  // fewer polls in flight: L2 stays free for the publications
#pragma unroll
    for (int i = 0; i < n; ++i)
      if (v[i].t0 != tag || v[i].t1 != tag) v[i] = ll_load(e[i]);
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
          ll_put(pub_first + 2 * (x - 2), o.x, tag);
          ll_put(pub_first + 2 * (x - 1), o.y, tag);
        } else if (refl_top) {
          *reinterpret_cast<double2*>(B + x) = make_double2(-o.x, -o.y);
          ll_ximg(B, x, nx, -o.x, -o.y, xm);
        }
      }
      if (r == R) {
        if (pub_last) {
          ll_put(pub_last + 2 * (x - 2), o.x, tag);
          ll_put(pub_last + 2 * (x - 1), o.y, tag);
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
  double* pub = p.ws + ((G + 1) & ~1);             // [slot][cta][first, last][nx] LL entries (16 B each)
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
    sweep(1, 1);
    if (R > 1) sweep(R, R);
    if (R > 2) sweep(2, R - 1);
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
        const double* const e[4] = {fu + 4 * q, fu + 4 * q + 2, fd + 4 * q, fd + 4 * q + 2};
        ll_get<4>(e, tag, v);
      } else if (top_x || bot_x) {
        const double* f = top_x ? fu : fd;
        const double* const e[4] = {f + 4 * q, f + 4 * q + 2, f, f};
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
  return (size_t)grid + 1 + (size_t)2 * grid * 2 * (RS_KMAX > 2 ? RS_KMAX : 2) * nx +
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

px_status launch_resident(int stencil, const ResidentLaunch& r, int grid, size_t smem, cudaStream_t s) {
  int g2 = 0, rm = 0;
  size_t sm2 = 0;
  const int K = resident_k(r.nx, r.ny, &g2, &rm, &sm2);
  if (K < 1 || g2 != grid || sm2 != smem) return fail(PX_ERR_STATE, "resident plan changed");
  static size_t attr_set[2][RS_KMAX] = {};
  const int k = stencil ? 1 : 0;
  void* fn = nullptr;
  cudaError_t e = cudaSuccess;
  switch (k * 4 + K) {
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
  void* args[] = {const_cast<ResidentLaunch*>(&r)};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e == cudaSuccess) e = cudaGetLastError();
  note_kernel(K == 1 ? "k_resident" : "k_resident_tb");
  count_launches(1);
  return cuda_check(e, "resident solve kernel launch");
}

}  // namespace px
