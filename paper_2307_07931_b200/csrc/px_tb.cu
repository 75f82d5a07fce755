// px_tb.cu -- temporal blocking: K Jacobi sweeps per pass over HBM
// (BASELINE config 4; DESIGN.md §6 K7).
//
// Exactly K plain sweeps (bit-identical to them and to the oracle): the
// level-0 iterate streams through shared memory by TMA bulk copies (as in
// k_bulk); each warp advances its 64 loaded columns through K time levels in
// registers, one row behind per level (a wavefront down the chunk):
//     level-0 row q arrives  ->  level 1 row q-1, level 2 row q-2, ...,
//     level K row q-K  ->  HBM
// W/E neighbours at every level come from the adjacent lane (__shfl); a
// warp's two outermost columns have no neighbour, so the valid region
// shrinks by one column per level and each warp writes its inner 64-2K
// columns (redundant halo compute, no inter-warp synchronisation).  Rows of a
// chunk are extended by K above and below (redundant, re-read from L2/HBM).
// Ghost cells inside the loaded halo are advanced like interior cells
// (periodic images and inter-rank copies compute the same values), except
// FIXED_GHOSTS domain faces, which keep their level-0 values.  ρ must carry
// valid ghosts to depth K.  HBM traffic: 24/K bytes per cell-update
// (+ 2K/chunk rows + 2K/(64-2K)... halo, measured in profiles/).
//
// Arithmetic per cell is the oracle's tree; when scale and λ are powers of
// two (h = 2^-p, λ = h²·2^-j, every BASELINE config) the products
// scale·L, λ·r and 4·C are exact, so the fused multiply-adds
// fma(scale, L, -ρ), fma(λ, r, φ), fma(-4, C, t) round exactly like the
// separate operations -- bit-identical, fewer FP64 instructions (P2=1).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "px_device.cuh"
#include "px_internal.h"
#include "px_ptx.cuh"

namespace px {

namespace tb {

constexpr int R = 3;               // rows per stage = rows per unrolled body (the S/C/N cycle)
constexpr int NST = 4;             // ring stages (consumers hold the current and previous one)
constexpr int CHUNK_ROWS = 255;    // nominal rows per work item (multiple of R)

// NW consumer warps + 1 producer warp per CTA.  Blocks are 8 or 16 warps so
// that each SM sub-partition (16K registers) holds 4 warps of 128 registers:
// NW = 7 runs 2 CTAs per SM, NW = 15 one CTA per SM.
template <int K, int NW>
struct Geom {
  static constexpr int THREADS = NW * 32 + 32;
  static constexpr int CPS = NW == 7 ? 2 : 1;
  static constexpr int WO = 64 - 2 * K;          // output columns per warp
  static constexpr int CO = NW * WO;             // output columns per CTA strip
  static constexpr int CL = CO + 2 * K;          // loaded columns per CTA strip
  static constexpr int CLS = (CL + 15) / 16 * 16; // smem row stride (doubles)
  static constexpr int STAGE = R * 2 * CLS;      // φ rows + ρ rows
  static constexpr size_t SMEM = (size_t)NST * STAGE * sizeof(double) + 2 * NST * sizeof(uint64_t);
};

using namespace ptx;

struct P2d {
  double a, b;  // the lane's two cells of a row
};

__device__ __forceinline__ int m3(int v) { return ((v % 3) + 3) % 3; }

}  // namespace tb

using namespace tb;

// One level-t update of a lane's two cells from level t-1 rows S, C, N.
template <int ST, int P2>
__device__ __forceinline__ void lvl_update(const P2d& S, const P2d& C, const P2d& N, double2 f,
                                           double scale, double lambda, double& o0, double& o1,
                                           double& r0, double& r1) {
  const double w = __shfl_up_sync(FULL_MASK, C.b, 1);    // lane 0: invalid column anyway
  const double e = __shfl_down_sync(FULL_MASK, C.a, 1);  // lane 31: invalid column anyway
  double L0, L1;
  if (ST == 0) {
    if (P2) {
      L0 = fma(-4.0, C.a, __dadd_rn(__dadd_rn(__dadd_rn(w, C.b), S.a), N.a));
      L1 = fma(-4.0, C.b, __dadd_rn(__dadd_rn(__dadd_rn(C.a, e), S.b), N.b));
    } else {
      L0 = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(w, C.b), S.a), N.a), __dmul_rn(-4.0, C.a));
      L1 = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(C.a, e), S.b), N.b), __dmul_rn(-4.0, C.b));
    }
  } else {
    const double sw = __shfl_up_sync(FULL_MASK, S.b, 1), se = __shfl_down_sync(FULL_MASK, S.a, 1);
    const double nw = __shfl_up_sync(FULL_MASK, N.b, 1), ne = __shfl_down_sync(FULL_MASK, N.a, 1);
    double q;
    q = __dmul_rn(4.0, w);
    q = __dadd_rn(q, __dmul_rn(4.0, C.b));
    q = __dadd_rn(q, __dmul_rn(4.0, S.a));
    q = __dadd_rn(q, __dmul_rn(4.0, N.a));
    q = __dadd_rn(q, sw);
    q = __dadd_rn(q, S.b);
    q = __dadd_rn(q, nw);
    q = __dadd_rn(q, N.b);
    L0 = __dadd_rn(q, __dmul_rn(-20.0, C.a));
    q = __dmul_rn(4.0, C.a);
    q = __dadd_rn(q, __dmul_rn(4.0, e));
    q = __dadd_rn(q, __dmul_rn(4.0, S.b));
    q = __dadd_rn(q, __dmul_rn(4.0, N.b));
    q = __dadd_rn(q, S.a);
    q = __dadd_rn(q, se);
    q = __dadd_rn(q, N.a);
    q = __dadd_rn(q, ne);
    L1 = __dadd_rn(q, __dmul_rn(-20.0, C.b));
  }
  if (P2) {
    r0 = fma(scale, L0, -f.x);
    r1 = fma(scale, L1, -f.y);
    o0 = fma(lambda, r0, C.a);
    o1 = fma(lambda, r1, C.b);
  } else {
    r0 = __dsub_rn(__dmul_rn(scale, L0), f.x);
    r1 = __dsub_rn(__dmul_rn(scale, L1), f.y);
    o0 = __dadd_rn(C.a, __dmul_rn(lambda, r0));
    o1 = __dadd_rn(C.b, __dmul_rn(lambda, r1));
  }
}

// Per-item consumer state shared by the stage bodies.
struct TbCtx {
  int qbase;        // first level-0 row of the item (y0 - K)
  int y0, y1;       // output rows
  int nrows;        // level-0 rows streamed: y1 - y0 + 2K
  int xg;           // column (rel. region) of the lane's pair
  bool own0, own1;  // lane writes / counts these cells
  bool fx0, fx1;    // FIXED ghost columns (keep level-0 values)
  bool xface;       // a written cell is within g of an x face (ghost images)
  bool img;         // some written cell of this item may have ghost images
};

// Which time levels record residual norms in this launch: NM = 0 none,
// 1 level 0 only (a norm every E >= K sweeps, passes aligned to E), 2 any
// (runtime mask).  Compile-time for 0 / 1 so the steady body carries no
// per-level tests.
template <int NM>
__device__ __forceinline__ bool lvl_act(const bool (&act)[4], int t) {
  return NM == 2 ? act[t] : (NM == 1 && t == 0);
}

// Process the R rows of one stage.  CHECK: warm-up / drain stage (row-range
// conditions evaluated); otherwise every level is computable and every row
// is an output row (steady state, no per-row conditions).
template <int ST, int K, int NW, int P2, int FIX, int NM, bool CHECK>
__device__ __forceinline__ void tb_stage(const StreamLaunch& a, const TbLaunch& x, const TbCtx& c,
                                         int s, const double* sp, const double* pp, int cl,
                                         P2d (&st)[K][3], unsigned long long (&mx)[K], double (&ss)[K],
                                         const bool (&act)[4]) {
  using G = Geom<K, NW>;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = s * R + j;                  // level-0 row index within the item
    if (CHECK && r >= c.nrows) break;
    const double2 v = *reinterpret_cast<const double2*>(sp + j * G::CLS + cl);
    st[0][j] = P2d{v.x, v.y};                 // r ≡ j (mod 3)
#pragma unroll
    for (int t = 1; t <= K; ++t) {
      if (CHECK && r < 2 * t) break;          // level t not yet computable
      const int p = c.qbase + r - t;          // row computed at level t
      // ρ(p) was loaded with level-0 row r-t+1 (this stage or the previous one)
      constexpr int dummy = 0;
      (void)dummy;
      const int e = j - t + 1;
      const double* rp = (e >= 0) ? (sp + (R + e) * G::CLS) : (pp + (R + R + e) * G::CLS);
      const double2 f = *reinterpret_cast<const double2*>(rp + cl);
      double o0, o1, r0, r1;
      lvl_update<ST, P2>(st[t - 1][m3(j - t - 1)], st[t - 1][m3(j - t)], st[t - 1][m3(j - t + 1)], f,
                         a.scale, a.lambda, o0, o1, r0, r1);
      if (FIX) {
        const bool fy = (p < 0 && x.fix[1][0]) || (p >= a.ny && x.fix[1][1]);
        if (fy || c.fx0) o0 = st[t - 1][m3(j - t)].a;
        if (fy || c.fx1) o1 = st[t - 1][m3(j - t)].b;
      }
      const bool prow = !CHECK || (p >= c.y0 && p < c.y1);
      if (lvl_act<NM>(act, t - 1)) {
        // branch-free: a cell the lane does not own contributes r = 0
        // (umax with +0 bits and fma(0, 0, Σ) leave both unchanged)
        const double q0 = (c.own0 && prow) ? r0 : 0.0;
        const double q1 = (c.own1 && prow) ? r1 : 0.0;
        mx[t - 1] = umax64(mx[t - 1], (unsigned long long)__double_as_longlong(fabs(q0)));
        ss[t - 1] = fma(q0, q0, ss[t - 1]);
        mx[t - 1] = umax64(mx[t - 1], (unsigned long long)__double_as_longlong(fabs(q1)));
        ss[t - 1] = fma(q1, q1, ss[t - 1]);
      }
      if (t == K) {
        if (prow) {
          double* dp = a.dst + (int64_t)p * a.ld_dst + c.xg;
          if (c.own0 && c.own1) {
            *reinterpret_cast<double2*>(dp) = make_double2(o0, o1);
          } else {
            if (c.own0) dp[0] = o0;
            if (c.own1) dp[1] = o1;
          }
          if (c.img) {
            const int Y = p + a.gs.o[1];
            if (c.xface || Y < a.gs.g || Y >= a.gs.n[1] - a.gs.g) {
              if (c.own0) images(a, c.xg, p, o0);
              if (c.own1) images(a, c.xg + 1, p, o1);
            }
          }
        }
      } else {
        st[t][m3(j - t)] = P2d{o0, o1};
      }
    }
  }
}

template <int ST, int K, int NW, int P2, int FIX, int NM>
__global__ void __launch_bounds__(NW * 32 + 32, (NW == 7 ? 2 : 1))
    k_tb(const StreamLaunch a, const TbLaunch x, int nstrips, int nitems, int crows) {
  using G = Geom<K, NW>;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * G::STAGE);
  uint64_t* empty = full + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  unsigned long long mx[K];
  double ss[K];
  bool act[4];
#pragma unroll
  for (int t = 0; t < K; ++t) {
    mx[t] = 0ull;
    ss[t] = 0.0;
    act[t] = x.lvl[t].out_max != nullptr;
  }

  if (warp == NW) {
    // ------------- producer: level-0 rows of φ and the rows of ρ -------------
    if (lane == 0) {
      uint64_t pol;
      pol = evict_first_policy();
      int slot = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int sidx = it % nstrips, k = it / nstrips;
        const int cload = sidx * G::CO - K;
        const int wcopy = min(G::CL, a.nx + K - cload);  // even (cload, nx, K even)
        const uint32_t rb = (uint32_t)wcopy * 8u;
        const int y0 = k * crows, y1 = min(a.ny, y0 + crows);
        const int qbase = y0 - K, nrows = y1 - y0 + 2 * K;
        const int nst = (nrows + R - 1) / R;
        for (int s = 0; s < nst; ++s) {
          mbar_wait(&empty[slot], phase ^ 1u);
          double* sp = smem + (size_t)slot * G::STAGE;
          int n = 0;
          for (int j = 0; j < R; ++j) {
            const int r = s * R + j;
            if (r < nrows) n += (r >= 2) ? 2 : 1;
          }
          mbar_arrive_expect_tx(&full[slot], rb * (uint32_t)n);
          for (int j = 0; j < R; ++j) {
            const int r = s * R + j;
            if (r >= nrows) break;
            const int q = qbase + r;
            bulk_g2s(sp + j * G::CLS, a.src + (int64_t)q * a.ld_src + cload, rb, &full[slot], pol);
            if (r >= 2)  // ρ row q-1: rows y0-K+1 .. y1+K-2 are the ones the levels use
              bulk_g2s(sp + (R + j) * G::CLS, a.rhs + (int64_t)(q - 1) * a.ld_rhs + cload, rb, &full[slot], pol);
          }
          if (++slot == NST) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    // ---------------------------- consumers ----------------------------
    const int cl = warp * G::WO + 2 * lane;
    const bool own = (2 * lane >= K) && (2 * lane + 1 < 64 - K);
    int slot = 0, prev = -1;
    uint32_t phase = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int sidx = it % nstrips, k = it / nstrips;
      TbCtx c;
      const int cload = sidx * G::CO - K;
      c.xg = cload + cl;
      c.own0 = own && c.xg >= 0 && c.xg < a.nx;
      c.own1 = own && c.xg + 1 >= 0 && c.xg + 1 < a.nx;
      c.fx0 = FIX && ((c.xg < 0 && x.fix[0][0]) || (c.xg >= a.nx && x.fix[0][1]));
      c.fx1 = FIX && ((c.xg + 1 < 0 && x.fix[0][0]) || (c.xg + 1 >= a.nx && x.fix[0][1]));
      {
        const int X0 = c.xg + a.gs.o[0];
        c.xface = (X0 < a.gs.g + 1) || (X0 + 1 >= a.gs.n[0] - a.gs.g - 1);
      }
      c.y0 = k * crows;
      c.y1 = min(a.ny, c.y0 + crows);
      c.img = a.gs.g > 0 && (c.xface || c.y0 + a.gs.o[1] < a.gs.g || c.y1 - 1 + a.gs.o[1] >= a.gs.n[1] - a.gs.g);
      c.qbase = c.y0 - K;
      c.nrows = c.y1 - c.y0 + 2 * K;
      const int nst = (c.nrows + R - 1) / R;
      P2d st[K][3];
#pragma unroll
      for (int t = 0; t < K; ++t)
#pragma unroll
        for (int u = 0; u < 3; ++u) st[t][u] = P2d{0.0, 0.0};
      const double* pp = smem;  // previous stage (valid from s = 1)
      for (int s = 0; s < nst; ++s) {
        mbar_wait(&full[slot], phase);
        const double* sp = smem + (size_t)slot * G::STAGE;
        const bool steady = (s * R >= 2 * K) && (s * R + R - 1 < c.nrows - K);
        if (steady)
          tb_stage<ST, K, NW, P2, FIX, NM, false>(a, x, c, s, sp, pp, cl, st, mx, ss, act);
        else
          tb_stage<ST, K, NW, P2, FIX, NM, true>(a, x, c, s, sp, pp, cl, st, mx, ss, act);
        __syncwarp();
        if (prev >= 0 && lane == 0) mbar_arrive(&empty[prev]);  // stage s-1 no longer needed
        prev = slot;
        pp = sp;
        if (++slot == NST) {
          slot = 0;
          phase ^= 1u;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[prev]);  // the item's last stage
      prev = -1;
    }
  }
#pragma unroll
  for (int t = 0; t < K; ++t) {
    if (lvl_act<NM>(act, t)) {
      reduce_norms(x.lvl[t], mx[t], ss[t]);
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ wide variant
// k_tbw: the same wavefront, but each lane owns FOUR adjacent columns (a warp
// 128 loaded, 128-2K written).  Per cell this halves the W/E shuffles and the
// redundant halo columns (2K/128 instead of 2K/64) and doubles the independent
// work per lane and level; the level rows (3 x K x 4 doubles) need the full
// register file, so a CTA is 7 consumer warps + 1 producer warp, one per SM.
// Residual max via fmax (NaN recovered from Σr² at the end: any NaN r makes
// Σr² NaN).  DIR: DIRICHLET_CC faces -- after every level t < K the first
// ghost column / row is re-derived from the level's own interior by odd
// reflection (corners by the product rule), so a pass of K levels is exactly
// K plain sweeps with the ghost fill in between (oracle R5).
#ifndef PX_TBW_IDLE_SKIP
#define PX_TBW_IDLE_SKIP 1  // A/B: 0 = idle warps of a narrow strip compute like the others
#endif
#ifndef PX_TBW_SWZ
#define PX_TBW_SWZ 0
#endif
namespace tbw {
constexpr int NW = 7;
constexpr int NST = 5;
template <int K>
struct Geom {
  static constexpr int THREADS = NW * 32 + 32;
  static constexpr int WL = 128;                  // loaded columns per warp
  static constexpr int WO = WL - 2 * K;           // written columns per warp
  static constexpr int CO = NW * WO;              // written columns per CTA strip
  static constexpr int CL = CO + 2 * K;           // loaded columns per CTA strip
  static constexpr int CLS = (CL + 15) / 16 * 16; // smem row stride (doubles)
  static constexpr int STAGE = R * 2 * CLS;       // φ rows + ρ rows
  static constexpr size_t SMEM = (size_t)NST * STAGE * sizeof(double) + 2 * NST * sizeof(uint64_t);
};
struct Q4 {
  double v[4];
};
struct Ctx {
  int qbase, y0, y1, nrows;
  int xg;            // column (rel. region) of the lane's first cell
  bool own01, own23; // the lane writes / counts cells 0,1 / 2,3 (owned in pairs)
  bool fx[4];        // FIXED ghost columns
  bool xface, img;   // images of written cells
  bool xref;         // DIR: the warp holds column -1 or column nx
  int xl, xh;        // DIR: position of column -1 / column nx in this lane (-1: none)
  bool ylo, yhi;     // DIR: reflecting y faces of the region
};
// A lane's four doubles sit 32 B after its left neighbour's, so two plain
// 16-B loads put lanes k and k+4 on the same banks (8 wavefronts per load
// instead of 4).  Lanes with bit 2 set fetch their upper half first: the
// eight lanes of each quarter-warp then cover all eight 16-B bank groups.
__device__ __forceinline__ Q4 lds4(const double* p) {
#if PX_TBW_SWZ
  const int sw = (threadIdx.x >> 1) & 2;  // 2 for lanes with bit 2 set
  const double2 u = *reinterpret_cast<const double2*>(p + sw);
  const double2 w = *reinterpret_cast<const double2*>(p + (2 - sw));
  return sw ? Q4{{w.x, w.y, u.x, u.y}} : Q4{{u.x, u.y, w.x, w.y}};
#else
  const double2 u = *reinterpret_cast<const double2*>(p);
  const double2 w = *reinterpret_cast<const double2*>(p + 2);
  return Q4{{u.x, u.y, w.x, w.y}};
#endif
}
}  // namespace tbw

template <int P2>
__device__ __forceinline__ void upd5(double w, double e, double s, double n, double c, double f, double scale,
                                     double lambda, double& o, double& r) {
  double L;
  if (P2) {
    L = fma(-4.0, c, __dadd_rn(__dadd_rn(__dadd_rn(w, e), s), n));
    r = fma(scale, L, -f);
    o = fma(lambda, r, c);
  } else {
    L = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(w, e), s), n), __dmul_rn(-4.0, c));
    r = __dsub_rn(__dmul_rn(scale, L), f);
    o = __dadd_rn(c, __dmul_rn(lambda, r));
  }
}

__device__ __forceinline__ void upd9(double w, double e, double s, double n, double sw, double se, double nw,
                                     double ne, double c, double f, double scale, double lambda, double& o,
                                     double& r) {
  double q = __dmul_rn(4.0, w);
  q = __dadd_rn(q, __dmul_rn(4.0, e));
  q = __dadd_rn(q, __dmul_rn(4.0, s));
  q = __dadd_rn(q, __dmul_rn(4.0, n));
  q = __dadd_rn(q, sw);
  q = __dadd_rn(q, se);
  q = __dadd_rn(q, nw);
  q = __dadd_rn(q, ne);
  const double L = __dadd_rn(q, __dmul_rn(-20.0, c));
  r = __dsub_rn(__dmul_rn(scale, L), f);
  o = __dadd_rn(c, __dmul_rn(lambda, r));
}

// Neighbour values of a lane's four cells held by the adjacent lanes.
struct Halo4 {
  double w, e, sw, se, nw, ne;
};
template <int ST>
__device__ __forceinline__ Halo4 halo4(const tbw::Q4& S, const tbw::Q4& C, const tbw::Q4& N) {
  Halo4 h;
  h.w = __shfl_up_sync(FULL_MASK, C.v[3], 1);    // lane 0: invalid column anyway
  h.e = __shfl_down_sync(FULL_MASK, C.v[0], 1);  // lane 31: invalid column anyway
  if (ST == 1) {
    h.sw = __shfl_up_sync(FULL_MASK, S.v[3], 1);
    h.se = __shfl_down_sync(FULL_MASK, S.v[0], 1);
    h.nw = __shfl_up_sync(FULL_MASK, N.v[3], 1);
    h.ne = __shfl_down_sync(FULL_MASK, N.v[0], 1);
  }
  return h;
}

// One level-t update of a lane's four cells from level t-1 rows S, C, N.
template <int ST, int P2>
__device__ __forceinline__ void lvl4(const tbw::Q4& S, const tbw::Q4& C, const tbw::Q4& N, const Halo4& h,
                                     const tbw::Q4& f, double scale, double lambda, tbw::Q4& o, double (&r)[4]) {
  if (ST == 0) {
    upd5<P2>(h.w, C.v[1], S.v[0], N.v[0], C.v[0], f.v[0], scale, lambda, o.v[0], r[0]);
    upd5<P2>(C.v[0], C.v[2], S.v[1], N.v[1], C.v[1], f.v[1], scale, lambda, o.v[1], r[1]);
    upd5<P2>(C.v[1], C.v[3], S.v[2], N.v[2], C.v[2], f.v[2], scale, lambda, o.v[2], r[2]);
    upd5<P2>(C.v[2], h.e, S.v[3], N.v[3], C.v[3], f.v[3], scale, lambda, o.v[3], r[3]);
  } else {
    upd9(h.w, C.v[1], S.v[0], N.v[0], h.sw, S.v[1], h.nw, N.v[1], C.v[0], f.v[0], scale, lambda, o.v[0], r[0]);
    upd9(C.v[0], C.v[2], S.v[1], N.v[1], S.v[0], S.v[2], N.v[0], N.v[2], C.v[1], f.v[1], scale, lambda, o.v[1],
         r[1]);
    upd9(C.v[1], C.v[3], S.v[2], N.v[2], S.v[1], S.v[3], N.v[1], N.v[3], C.v[2], f.v[2], scale, lambda, o.v[2],
         r[2]);
    upd9(C.v[2], h.e, S.v[3], N.v[3], S.v[2], h.se, N.v[2], h.ne, C.v[3], f.v[3], scale, lambda, o.v[3], r[3]);
  }
}

// Process the R rows of one stage of the skewed wavefront: at level-0 row r
// (relative to the item's first loaded row) level t computes relative row
// r - (2t - 1).  Level 1 uses the row loaded in this iteration; every other
// level's three inputs were produced in earlier iterations, so the K levels
// of an iteration are independent (K x 4 chains per lane).  Levels run from K
// down to 1 so that level t reads the slot level t-1 overwrites in the same
// iteration before it is overwritten; the level-0 row goes straight into the
// slot of row r-3, which no level reads any more.  ρ of relative row p
// arrives with level-0 row p + 1, i.e. in this stage or one of the two before
// it (sp, p1, p2).
// CHECK: warm-up / drain stage (row-range conditions evaluated).
template <int ST, int K, int P2, int FIX, int DIR, int NM, bool CHECK>
__device__ __forceinline__ void tbw_stage(const StreamLaunch& a, const TbLaunch& x, const tbw::Ctx& c, int s,
                                          const double* sp, const double* p1, const double* p2, int cl,
                                          tbw::Q4 (&st)[K][3], double (&mx)[K], double (&ss)[K],
                                          double (&ia)[4], const bool (&act)[4]) {
  using G = tbw::Geom<K>;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = s * R + j;  // level-0 row index within the item
    if (CHECK && r >= c.nrows + K - 1) break;
    if (!CHECK || r < c.nrows) st[0][j] = tbw::lds4(sp + j * G::CLS + cl);  // r ≡ j (mod 3)
    // gather (5-point): every level's neighbour-lane values first (all
    // independent), so the shuffle latencies overlap; the 9-point stencil
    // needs three times as many and shuffles per level (register budget)
    Halo4 hl[K + 1];
#pragma unroll
    for (int t = K; t >= 1; --t) {
      const int pr = r - 2 * t + 1;
      if (ST == 1 || (CHECK && (pr < t || pr >= c.nrows - t))) continue;
      hl[t] = halo4<ST>(st[t - 1][m3(j - 2 * t)], st[t - 1][m3(j - 2 * t + 1)], st[t - 1][m3(j - 2 * t + 2)]);
    }
#pragma unroll
    for (int t = K; t >= 1; --t) {
      const int pr = r - 2 * t + 1;                   // relative row computed at level t
      if (CHECK && (pr < t || pr >= c.nrows - t)) continue;  // outside level t's valid rows
      const int p = c.qbase + pr;                     // region row
      const int e = j - 2 * t + 2;                    // ρ(p) came with level-0 row pr + 1
      const double* rp = e >= 0 ? sp + (R + e) * G::CLS
                                : (e >= -R ? p1 + (R + e + R) * G::CLS : p2 + (R + e + 2 * R) * G::CLS);
      const tbw::Q4 f = tbw::lds4(rp + cl);
      tbw::Q4 o;
      double rr[4];
      const tbw::Q4& C = st[t - 1][m3(j - 2 * t + 1)];
      if (ST == 1)
        hl[t] = halo4<ST>(st[t - 1][m3(j - 2 * t)], C, st[t - 1][m3(j - 2 * t + 2)]);
      lvl4<ST, P2>(st[t - 1][m3(j - 2 * t)], C, st[t - 1][m3(j - 2 * t + 2)], hl[t], f, a.scale, a.lambda, o, rr);
      if (FIX) {
        const bool fy = (p < 0 && x.fix[1][0]) || (p >= a.ny && x.fix[1][1]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (fy || c.fx[i]) o.v[i] = C.v[i];
      }
      if (DIR && t < K) {
        if (c.xref) {  // warp-uniform
          const double dn = __shfl_down_sync(FULL_MASK, o.v[0], 1);
          const double up = __shfl_up_sync(FULL_MASK, o.v[3], 1);
          if (c.xl == 1) o.v[1] = -o.v[2];
          if (c.xl == 3) o.v[3] = -dn;
          if (c.xh == 0) o.v[0] = -up;
          if (c.xh == 2) o.v[2] = -o.v[1];
        }
        if (CHECK && c.yhi && p == a.ny) {
          const tbw::Q4& B = st[t][m3(j - 2 * t)];  // level t, row ny-1 (previous iteration)
#pragma unroll
          for (int i = 0; i < 4; ++i) o.v[i] = -B.v[i];
        }
      }
      const bool prow = !CHECK || (p >= c.y0 && p < c.y1);
      if (lvl_act<NM>(act, t - 1)) {
        // a NaN r fails the compare but makes Σr² NaN (recovered at the end)
        if (NM == 1 && !CHECK) {
          // steady rows, level-0 norms only: accumulate unconditionally per
          // column pair into the item's accumulators (merged by ownership at
          // the end of the item) -- no per-cell predicates
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double ar = fabs(rr[i]);
            double& m = ia[i < 2 ? 0 : 2];
            m = ar > m ? ar : m;
            ia[i < 2 ? 1 : 3] = fma(rr[i], rr[i], ia[i < 2 ? 1 : 3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double ar = fabs(rr[i]);
            if ((i < 2 ? c.own01 : c.own23) && prow) {
              if (ar > mx[t - 1]) mx[t - 1] = ar;
              ss[t - 1] = fma(rr[i], rr[i], ss[t - 1]);
            }
          }
        }
      }
      if (t == K) {
        if (prow) {
          // columns are owned in aligned pairs (K, the strip origin and nx are even)
          double* dp = a.dst + (int64_t)p * a.ld_dst + c.xg;
          if (c.own01) *reinterpret_cast<double2*>(dp) = make_double2(o.v[0], o.v[1]);
          if (c.own23) *reinterpret_cast<double2*>(dp + 2) = make_double2(o.v[2], o.v[3]);
          if (c.img) {  // warp-uniform
            const int Y = p + a.gs.o[1];
            if (c.xface || Y < a.gs.g || Y >= a.gs.n[1] - a.gs.g) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (i < 2 ? c.own01 : c.own23) images(a, c.xg + i, p, o.v[i]);
            }
          }
        }
      } else {
        st[t][m3(j - 2 * t + 1)] = o;
        if (DIR && CHECK && c.ylo && p == 0) {
          tbw::Q4& B = st[t][m3(j - 2 * t)];  // level t, row -1
#pragma unroll
          for (int i = 0; i < 4; ++i) B.v[i] = -o.v[i];
        }
      }
    }
  }
}

template <int ST, int K, int P2, int FIX, int DIR, int NM>
__global__ void __launch_bounds__(tbw::NW * 32 + 32, 1)
    k_tbw(const StreamLaunch a, const TbLaunch x, int nstrips, int nitems, int crows) {
  using G = tbw::Geom<K>;
  constexpr int NW = tbw::NW, NSTG = tbw::NST;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NSTG * G::STAGE);
  uint64_t* empty = full + NSTG;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double mx[K];
  double ss[K];
  bool act[4];
#pragma unroll
  for (int t = 0; t < K; ++t) {
    mx[t] = 0.0;
    ss[t] = 0.0;
    act[t] = x.lvl[t].out_max != nullptr;
  }

  if (warp == NW) {
    // ------------- producer: level-0 rows of φ and the rows of ρ -------------
    if (lane == 0) {
      uint64_t pol;
      pol = evict_first_policy();
      int slot = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int sidx = it % nstrips, k = it / nstrips;
        const int cload = sidx * G::CO - K;
        const int wcopy = min(G::CL, a.nx + K - cload);  // even (cload, nx, K even)
        const uint32_t rb = (uint32_t)wcopy * 8u;
        const int y0 = k * crows, y1 = min(a.ny, y0 + crows);
        const int qbase = y0 - K, nrows = y1 - y0 + 2 * K;
        const int nst = (nrows + K - 1 + R - 1) / R;  // K-1 drain rows: the output lags 2K-1 rows
        for (int s = 0; s < nst; ++s) {
          mbar_wait_sleep(&empty[slot], phase ^ 1u);
          double* sp = smem + (size_t)slot * G::STAGE;
          uint32_t n = 0;
          for (int j = 0; j < R; ++j) {
            const int r = s * R + j;
            n += (r < nrows ? 1u : 0u) + (r >= 2 && r < nrows ? 1u : 0u);
          }
          mbar_arrive_expect_tx(&full[slot], rb * n);
          for (int j = 0; j < R; ++j) {
            const int r = s * R + j;
            const int q = qbase + r;
            if (r < nrows) bulk_g2s(sp + j * G::CLS, a.src + (int64_t)q * a.ld_src + cload, rb, &full[slot], pol);
            if (r >= 2 && r < nrows)  // ρ of relative row r-1
              bulk_g2s(sp + (R + j) * G::CLS, a.rhs + (int64_t)(q - 1) * a.ld_rhs + cload, rb, &full[slot], pol);
          }
          if (++slot == NSTG) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    // ---------------------------- consumers ----------------------------
    const int cl = warp * G::WO + 4 * lane;
    int slot = 0, prev1 = -1, prev2 = -1;
    uint32_t phase = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const int sidx = it % nstrips, k = it / nstrips;
      tbw::Ctx c;
      const int cload = sidx * G::CO - K;
      c.xg = cload + cl;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int xc = c.xg + i;
        c.fx[i] = FIX && ((xc < 0 && x.fix[0][0]) || (xc >= a.nx && x.fix[0][1]));
      }
      c.own01 = 4 * lane >= K && 4 * lane + 1 < G::WL - K && c.xg >= 0 && c.xg + 1 < a.nx;
      c.own23 = 4 * lane + 2 >= K && 4 * lane + 3 < G::WL - K && c.xg + 2 >= 0 && c.xg + 3 < a.nx;
      {
        const int X0 = c.xg + a.gs.o[0];
        c.xface = (X0 < a.gs.g + 1) || (X0 + 3 >= a.gs.n[0] - a.gs.g - 1);
      }
      c.xl = c.xh = -1;
      c.ylo = c.yhi = false;
      c.xref = false;
      if (DIR) {
        if (x.refl[0][0] && c.xg <= -1 && c.xg + 3 >= -1) c.xl = -1 - c.xg;
        if (x.refl[0][1] && c.xg <= a.nx && c.xg + 3 >= a.nx) c.xh = a.nx - c.xg;
        c.xref = __any_sync(FULL_MASK, c.xl >= 0 || c.xh >= 0);
        c.ylo = x.refl[1][0] != 0;
        c.yhi = x.refl[1][1] != 0;
      }
      c.y0 = k * crows;
      c.y1 = min(a.ny, c.y0 + crows);
      c.img = __any_sync(FULL_MASK, a.gs.g > 0 && (c.xface || c.y0 + a.gs.o[1] < a.gs.g ||
                                                   c.y1 - 1 + a.gs.o[1] >= a.gs.n[1] - a.gs.g));
      c.qbase = c.y0 - K;
      c.nrows = c.y1 - c.y0 + 2 * K;
      tbw::Q4 st[K][3];
#pragma unroll
      for (int t = 0; t < K; ++t)
#pragma unroll
        for (int u = 0; u < 3; ++u) st[t][u] = tbw::Q4{{0.0, 0.0, 0.0, 0.0}};
      double ia[4] = {0.0, 0.0, 0.0, 0.0};  // item accumulators (max, Σ) of pairs 01, 23
      const double* pp1 = smem;  // previous stages (ρ rows; valid from s = 1, 2)
      const double* pp2 = smem;
      const int nst = (c.nrows + K - 1 + R - 1) / R;
      const int s_steady0 = (3 * K - 1 + R - 1) / R;  // first stage with every level valid
      // a warp with no column to write in this strip (the last, narrow strip
      // of a row of strips) only keeps the stage protocol: its levels would be
      // discarded, and under the board's power cap the saved energy is time
      const bool widle = PX_TBW_IDLE_SKIP && cload + warp * G::WO + K >= a.nx;
      for (int s = 0; s < nst; ++s) {
        mbar_wait(&full[slot], phase);
        const double* sp = smem + (size_t)slot * G::STAGE;
        const bool steady = s >= s_steady0 && (s * R + R - 1 < c.nrows - K);
        if (widle) {
        } else if (steady)
          tbw_stage<ST, K, P2, FIX, DIR, NM, false>(a, x, c, s, sp, pp1, pp2, cl, st, mx, ss, ia, act);
        else
          tbw_stage<ST, K, P2, FIX, DIR, NM, true>(a, x, c, s, sp, pp1, pp2, cl, st, mx, ss, ia, act);
        __syncwarp();
        if (prev2 >= 0 && lane == 0) mbar_arrive(&empty[prev2]);  // stage s-2 no longer needed
        prev2 = prev1;
        prev1 = slot;
        pp2 = pp1;
        pp1 = sp;
        if (++slot == NSTG) {
          slot = 0;
          phase ^= 1u;
        }
      }
      __syncwarp();
      if (lane == 0) {  // the item's last two stages
        if (prev2 >= 0) mbar_arrive(&empty[prev2]);
        if (prev1 >= 0) mbar_arrive(&empty[prev1]);
      }
      prev1 = prev2 = -1;
      if (NM == 1) {
        if (c.own01) {
          mx[0] = ia[0] > mx[0] ? ia[0] : mx[0];
          ss[0] = ss[0] + ia[1];
        }
        if (c.own23) {
          mx[0] = ia[2] > mx[0] ? ia[2] : mx[0];
          ss[0] = ss[0] + ia[3];
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < K; ++t) {
    if (lvl_act<NM>(act, t)) {
      // a NaN residual makes Σr² NaN (fmax alone would drop it): report NaN
      const unsigned long long bits = isnan(ss[t]) ? 0x7ff8000000000000ull
                                                   : (unsigned long long)__double_as_longlong(mx[t]);
      reduce_norms(x.lvl[t], bits, ss[t]);
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ host
static int tb_nsm() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct TbPlan {
  int nstrips, nitems, crows, grid;
};

static int tb_nw() {
  static int nw = 0;
  if (!nw) {
    // A/B knob: 7 (2 CTAs/SM) or 15 (1 CTA/SM, default: 734 vs 726 Gcell/s at
    // 16384², k=4, norm every 4 sweeps -- profiles/round1_tb.json)
    const char* e = getenv("PROTOX_TB_NW");
    nw = (e && atoi(e) == 7) ? 7 : 15;
  }
  return nw;
}

// Which kernel runs the passes: the wide kernel (4 columns per lane, default)
// or the narrow one (2 columns per lane; PROTOX_TB_IMPL=narrow, A/B only --
// it has no per-level Dirichlet reflection).
static bool tb_wide() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("PROTOX_TB_IMPL");
    w = (e && e[0] == 'n') ? 0 : 1;
  }
  return w == 1;
}

// co: written columns per CTA strip; cps: CTAs per SM
static TbPlan tb_plan_g(int K, int nx, int ny, int co, int cps) {
  TbPlan g;
  g.nstrips = (nx + co - 1) / co;
  const int gmax = cps * tb_nsm() < BULK_MAX_GRID ? cps * tb_nsm() : BULK_MAX_GRID;
  const int c0 = (ny + CHUNK_ROWS - 1) / CHUNK_ROWS;
  double best = 1e30;
  int bestc = c0;
  const int cmax = 2 * c0 > (gmax + g.nstrips - 1) / g.nstrips ? 2 * c0 : (gmax + g.nstrips - 1) / g.nstrips;
  for (int c = c0; c <= cmax && c <= ny; ++c) {
    int rows = (ny + c - 1) / c;
    rows = (rows + 2) / 3 * 3;  // whole stages of R = 3 rows
    const int cc = (ny + rows - 1) / rows;
    const int items = g.nstrips * cc;
    const int waves = (items + gmax - 1) / gmax;
    const double cost = (double)waves * (rows + 2 * K);
    if (cost < best - 1e-9) {
      best = cost;
      bestc = cc;
    }
  }
  g.crows = (ny + bestc - 1) / bestc;
  g.crows = (g.crows + 2) / 3 * 3;
  const int nch = (ny + g.crows - 1) / g.crows;
  g.nitems = g.nstrips * nch;
  g.grid = g.nitems < gmax ? g.nitems : gmax;
  return g;
}

static TbPlan tb_plan(int K, int nx, int ny) {
  if (tb_wide()) return tb_plan_g(K, nx, ny, tbw::NW * (128 - 2 * K), 1);
  const int NW = tb_nw();
  return tb_plan_g(K, nx, ny, NW * (64 - 2 * K), NW == 7 ? 2 : 1);
}

int32_t tb_blocks(int K, const StreamLaunch& a) { return tb_plan(K, a.nx, a.ny).grid; }

static bool pow2(double v) {
  if (!(v > 0.0) || !std::isfinite(v)) return false;
  int e;
  return std::frexp(v, &e) == 0.5;
}

template <int ST, int K, int NW, int P2, int FIX, int NM>
static cudaError_t tb_launch_nm(const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  using G = Geom<K, NW>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_tb<ST, K, NW, P2, FIX, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const TbPlan g = tb_plan(K, a.nx, a.ny);
  k_tb<ST, K, NW, P2, FIX, NM><<<g.grid, G::THREADS, G::SMEM, s>>>(a, x, g.nstrips, g.nitems, g.crows);
  return cudaGetLastError();
}

template <int ST, int K, int NW, int P2, int FIX>
static cudaError_t tb_launch_nw(const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  unsigned mask = 0;
  for (int t = 0; t < K; ++t)
    if (x.lvl[t].out_max) mask |= 1u << t;
  if (mask == 0) return tb_launch_nm<ST, K, NW, P2, FIX, 0>(a, x, s);
  if (mask == 1) return tb_launch_nm<ST, K, NW, P2, FIX, 1>(a, x, s);
  return tb_launch_nm<ST, K, NW, P2, FIX, 2>(a, x, s);
}

template <int ST, int K, int P2, int FIX>
static cudaError_t tb_launch_t(const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  return tb_nw() == 7 ? tb_launch_nw<ST, K, 7, P2, FIX>(a, x, s) : tb_launch_nw<ST, K, 15, P2, FIX>(a, x, s);
}

template <int ST, int K, int P2, int FIX, int DIR, int NM>
static cudaError_t tbw_launch_nm(const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  using G = tbw::Geom<K>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_tbw<ST, K, P2, FIX, DIR, NM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const TbPlan g = tb_plan(K, a.nx, a.ny);
  k_tbw<ST, K, P2, FIX, DIR, NM><<<g.grid, G::THREADS, G::SMEM, s>>>(a, x, g.nstrips, g.nitems, g.crows);
  return cudaGetLastError();
}

template <int ST, int K, int P2, int FIX, int DIR>
static cudaError_t tbw_launch_bc(const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  unsigned mask = 0;
  for (int t = 0; t < K; ++t)
    if (x.lvl[t].out_max) mask |= 1u << t;
  if (mask == 0) return tbw_launch_nm<ST, K, P2, FIX, DIR, 0>(a, x, s);
  if (mask == 1) return tbw_launch_nm<ST, K, P2, FIX, DIR, 1>(a, x, s);
  return tbw_launch_nm<ST, K, P2, FIX, DIR, 2>(a, x, s);
}

template <int ST, int K, int P2>
static cudaError_t tb_fix(const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  const bool fix = x.fix[0][0] || x.fix[0][1] || x.fix[1][0] || x.fix[1][1];
  const bool dir = x.refl[0][0] || x.refl[0][1] || x.refl[1][0] || x.refl[1][1];
  if (tb_wide()) {
    if (dir) return tbw_launch_bc<ST, K, P2, 0, 1>(a, x, s);
    return fix ? tbw_launch_bc<ST, K, P2, 1, 0>(a, x, s) : tbw_launch_bc<ST, K, P2, 0, 0>(a, x, s);
  }
  return fix ? tb_launch_t<ST, K, P2, 1>(a, x, s) : tb_launch_t<ST, K, P2, 0>(a, x, s);
}

px_status launch_tb(int stencil, int K, const StreamLaunch& a, const TbLaunch& x, cudaStream_t s) {
  if (a.phase != 0 || (a.nx & 1)) return fail(PX_ERR_ALIGN, "temporal blocking needs an aligned, even-width slab");
  const bool dir = x.refl[0][0] || x.refl[0][1] || x.refl[1][0] || x.refl[1][1];
  if (dir && !tb_wide())
    return fail(PX_ERR_UNSUPPORTED, "DIRICHLET_CC temporal blocking needs the wide kernel (PROTOX_TB_IMPL)");
  const bool p2 = stencil == 0 && pow2(a.scale) && pow2(a.lambda);
  cudaError_t e;
  const int key = (stencil * 8 + K) * 2 + (p2 ? 1 : 0);
  switch (key) {
    case (0 * 8 + 2) * 2 + 0: e = tb_fix<0, 2, 0>(a, x, s); break;
    case (0 * 8 + 2) * 2 + 1: e = tb_fix<0, 2, 1>(a, x, s); break;
    case (0 * 8 + 4) * 2 + 0: e = tb_fix<0, 4, 0>(a, x, s); break;
    case (0 * 8 + 4) * 2 + 1: e = tb_fix<0, 4, 1>(a, x, s); break;
    case (1 * 8 + 2) * 2 + 0: e = tb_fix<1, 2, 0>(a, x, s); break;
    case (1 * 8 + 4) * 2 + 0: e = tb_fix<1, 4, 0>(a, x, s); break;
    default: return fail(PX_ERR_UNSUPPORTED, "temporal_k=%d not built (2 or 4)", K);
  }
  note_kernel(tb_wide() ? "k_tbw" : "k_tb");
  count_launches(1);
  return cuda_check(e, "temporal-blocking kernel launch");
}

}  // namespace px
