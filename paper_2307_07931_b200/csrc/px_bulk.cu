// px_bulk.cu -- the TMA-staged fused relax sweep (kernel K1b).
//
// Same arithmetic as k_stream (px_kernels.cu) -- per cell the oracle's
// expression tree, every * and + rounded separately -- but the HBM streams
// are moved by the Tensor Memory Accelerator: a producer warp issues
// cp.async.bulk (TMA bulk copies, SASS UBLKCP) of whole row segments of φ and
// of the right-hand side into a ring of shared-memory stages, each guarded by
// an mbarrier with a transaction count; eight consumer warps read a stage,
// keep the rows S, C, N of their column pair in registers, write φ' with
// 16-byte stores and release the stage.  The bytes in flight per SM are set
// by the ring depth (up to NST-1 stages of 32 KB), not by registers, so one
// 288-thread CTA per SM saturates HBM.  Persistent grid: one CTA per SM walks
// (strip of 512 columns) x (chunk of rows) work items.
//
// Halo: the W neighbour of a strip's first column and the E neighbour of its
// last column come from the adjacent strips; the two edge threads load them
// with plain 8-byte loads one stage ahead (into registers).  The row above
// a chunk is re-read once per chunk (2 rows per CHUNK_ROWS).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "px_internal.h"
#include "px_device.cuh"
#include "px_ptx.cuh"

namespace px {

namespace bulk {

// NC consumer warps (a strip of W = 64*NC columns, one column pair per
// thread) + 1 producer warp.
constexpr int CHUNK_ROWS = 1024;         // nominal rows per work item
// ring of NST stages of R rows of φ and of the rhs (R * 8 KB per stage)
template <int NST, int R, int NC>
constexpr size_t smem_bytes() {
  return (size_t)NST * (R * 2 * 64 * NC) * sizeof(double) + 2 * NST * sizeof(uint64_t);
}

using namespace ptx;

// ---- fused halo push over peer memory (PushSpec, px_internal.h) ----
// spin until own arrival counter `side` reaches base + wcount (acquire, system
// scope; bounded: px_spin_until)
__device__ __forceinline__ void ps_wait(const PushSpec& ps, int side) {
  px_spin_until(ps.wflag[side], *ps.epoch + ps.wcount, ps.err);
}
// The pair (x, x+1) of a row pushed into the neighbour's ghost row rp, with
// the x images of the pair's cells at the domain's x faces (corners).  Rare
// (2g rows per sweep): out of line, scalar arguments only, so the kernel's
// inner loop keeps its registers.
static __device__ __noinline__ void ps_push(double* rp, int x, double v0, double v1, int X0, int g, int n0,
                                            int m0, int m1) {
  *reinterpret_cast<double2*>(rp + x) = make_double2(v0, v1);
  for (int q = 0; q < 2; ++q) {
    const int X = X0 + q;
    const double v = q ? v1 : v0;
    const int o = x + q - X;  // region-relative column of global column 0
    if (X < g && m0 != GH_NONE) rp[(m0 == GH_WRAP ? X + n0 : -X - 1) + o] = m0 == GH_REFLECT ? -v : v;
    if (X >= n0 - g && m1 != GH_NONE) rp[(m1 == GH_WRAP ? X - n0 : 2 * n0 - 1 - X) + o] = m1 == GH_REFLECT ? -v : v;
  }
}
// End of a boundary item: push its rows [0,g) (lo side) and/or [ny-g,ny) (hi
// side) of φ' -- read back from this thread's own stores -- into the
// neighbours' ghost rows (plain stores; their arrival is counted by the next
// kernel, see k_bulk).  Outside the per-stage loop, out of line: the sweep's
// inner loop is untouched.
static __device__ __noinline__ void push_rows(const double* dst, int64_t ld, double* rlo, double* rhi, int ny,
                                              int g, int x, bool live, bool xface, int X0, int gg, int n0, int m0,
                                              int m1) {
  if (!live) return;
  for (int side = 0; side < 2; ++side) {
    double* rd = side ? rhi : rlo;
    if (!rd) continue;
    const int p0 = side ? ny - g : 0;
    for (int r = 0; r < g; ++r) {
      const double2 v = *reinterpret_cast<const double2*>(dst + (int64_t)(p0 + r) * ld + x);
      double* rp = rd + (int64_t)r * ld;
      if (xface)
        ps_push(rp, x, v.x, v.y, X0, gg, n0, m0, m1);
      else
        *reinterpret_cast<double2*>(rp + x) = v;
    }
  }
}

struct Item {
  int c;       // first column of the strip (relative to region.lo)
  int w;       // strip width (even)
  int y0, y1;  // rows computed: [y0, y1)
};

template <int W, int PUSH>
__device__ __forceinline__ Item item_of(const StreamLaunch& a, int it, int nstrips, int crows) {
  Item t;
  const int s = it % nstrips;
  int k = it / nstrips;
  if (PUSH && k > 0) {
    // push mode: the first and the last row chunk (the ones that push rows to
    // and read ghost rows from the neighbours) are the first two chunks run
    const int nchunks = (a.ny + crows - 1) / crows;
    k = (k == 1) ? nchunks - 1 : k - 1;
  }
  t.c = s * W;
  t.w = min(W, a.nx - t.c);
  t.y0 = k * crows;
  t.y1 = min(a.ny, t.y0 + crows);
  return t;
}
// φ rows streamed for an item: y0-1 .. y1 (inclusive) -> y1-y0+2 rows
template <int R>
__device__ __forceinline__ int item_stages(const Item& t) { return (t.y1 - t.y0 + 2 + R - 1) / R; }

}  // namespace bulk

using namespace bulk;


// NST stages of R rows per CTA, CPS CTAs per SM.
// PW bit 0: scale is a power of two, bit 1: λ is a power of two (exact
// products, so fused multiply-adds are bit-identical to the separate ops).
// PUSH: fused peer-memory halo push (PushSpec; px_solve P2P mode)
template <int MODE, int ST, int NST, int R, int CPS, int NC, int PW, int PUSH>
__global__ void __launch_bounds__(NC * 32 + 32, CPS) k_bulk(const StreamLaunch a, int nstrips, int nitems,
                                                            int crows) {
  constexpr int W = 64 * NC, NCW = NC;
  constexpr bool P2 = (PW & 1) != 0, PL = (PW & 2) != 0;
  static_assert(R % 3 == 0, "rows live in slots indexed by row mod 3");
  constexpr int STAGE_DOUBLES = R * 2 * W;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * STAGE_DOUBLES);
  uint64_t* empty = full + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Programmatic dependent launch (a.pdl: the sweep loop of px_solve): the
  // next sweep's grid may be launched now -- its CTAs take SM slots as this
  // grid's CTAs exit and run their prologue -- and this grid waits here
  // until the previous sweep's grid has completed and its stores are
  // visible (no-op without the launch attribute).  Every global access of
  // the kernel (including the norm workspace) comes after the wait.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (PUSH && tid == 0) {
    if (blockIdx.x == 0 && a.ps.rel) {
      // the previous sweep's pushes into the neighbours' ghost rows are
      // complete: that kernel has finished (stream order; a finished grid's
      // stores, peer stores included, are performed), so one relaxed count
      // per side publishes them -- no system-scope fence in the sweep
      for (int side = 0; side < 2; ++side)
        if (a.ps.rflag[side])
          asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(a.ps.rflag[side]), "l"(1ull) : "memory");
    }
    if (blockIdx.x < nitems) {
      // push mode: the boundary items (first and last row chunk) are every
      // CTA's FIRST item (they are scheduled first and the grid covers them,
      // bulk_geom), so the ghost rows the neighbours push are awaited once,
      // here, before any thread of the CTA touches them: the acquire plus the
      // CTA barrier below order every consumer load after the neighbours'
      // stores, and the proxy fence orders the producer's TMA reads.
      const Item t = item_of<W, PUSH>(a, blockIdx.x, nstrips, crows);
      if (t.y0 == 0 && a.ps.wflag[0]) ps_wait(a.ps, 0);
      if (t.y1 == a.ny && a.ps.wflag[1]) ps_wait(a.ps, 1);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
  __syncthreads();

  // max|r| as a double through fmax (one DMNMX per cell instead of a 64-bit
  // integer compare-and-select): fmax returns one of its operands, so the
  // max is exact; it drops NaN, but a NaN r makes Σr² NaN, which restores it
  // below (R7)
  double mxd = 0.0;
  double ss = 0.0;

  if (warp == NCW) {
    // ================= producer (one elected lane) =================
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int slot = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item t = item_of<W, PUSH>(a, it, nstrips, crows);
        const int nst = item_stages<R>(t);
        const uint32_t rowbytes = (uint32_t)t.w * 8u;
        for (int st = 0; st < nst; ++st) {
          mbar_wait(&empty[slot], phase ^ 1u);
          double* sp = smem + (size_t)slot * STAGE_DOUBLES;
          uint32_t bytes = 0;
          int nphi = 0, nrhs = 0;
          for (int i = 0; i < R; ++i) {
            const int yf = t.y0 - 1 + st * R + i;  // φ row of entry i
            if (yf <= t.y1) ++nphi;
            const int yr = yf - 1;                 // rhs row of entry i
            if (yr >= t.y0 && yr < t.y1) ++nrhs;
          }
          bytes = rowbytes * (uint32_t)(nphi + ((MODE == MODE_RELAX || MODE == MODE_RESID) ? nrhs : 0));
          mbar_arrive_expect_tx(&full[slot], bytes);
          for (int i = 0; i < R; ++i) {
            const int yf = t.y0 - 1 + st * R + i;
            const int yw = a.wrap ? (yf < 0 ? yf + a.ny : (yf >= a.ny ? yf - a.ny : yf)) : yf;  // periodic image
            if (yf <= t.y1)
              bulk_g2s(sp + i * W, a.src + (int64_t)yw * a.ld_src + t.c, rowbytes, &full[slot], pol);
            const int yr = yf - 1;
            if ((MODE == MODE_RELAX || MODE == MODE_RESID) && yr >= t.y0 && yr < t.y1)
              bulk_g2s(sp + (R + i) * W, a.rhs + (int64_t)yr * a.ld_rhs + t.c, rowbytes, &full[slot], pol);
          }
          if (++slot == NST) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    // ================= consumers =================
    const int j = tid;                     // pair index within the strip
    const int c0 = 2 * j;                  // strip-relative first column of the pair
    int slot = 0;
    uint32_t phase = 0;
    // W / E halo of the strip for the rows of the NEXT stage (loaded one
    // stage ahead by the two edge threads; 0 elsewhere)
    double hw_next[R], he_next[R];
    auto load_halo = [&](const Item& t, int st) {
      const bool L = (j == 0), Rt = (c0 + 2 == t.w);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int yf = t.y0 - 1 + st * R + i;
        hw_next[i] = 0.0;
        he_next[i] = 0.0;
        if (yf <= t.y1) {
          if (a.wrap) {  // periodic images of row and column
            const int yw = yf < 0 ? yf + a.ny : (yf >= a.ny ? yf - a.ny : yf);
            const double* row = a.src + (int64_t)yw * a.ld_src;
            if (L) hw_next[i] = row[t.c == 0 ? a.nx - 1 : t.c - 1];
            if (Rt) he_next[i] = row[t.c + t.w == a.nx ? 0 : t.c + t.w];
          } else {
            const double* row = a.src + (int64_t)yf * a.ld_src;
            if (L && t.c - 1 >= a.src_x0) hw_next[i] = row[t.c - 1];
            if (Rt && t.c + t.w <= a.src_x1) he_next[i] = row[t.c + t.w];
          }
        }
      }
    };
    int it = blockIdx.x;
    Item t;
    if (it < nitems) {
      t = item_of<W, PUSH>(a, it, nstrips, crows);
      load_halo(t, 0);
    }
    for (; it < nitems; it += gridDim.x) {
      const int nst = item_stages<R>(t);
      const bool live = c0 < t.w;
      const bool left = (j == 0);
      const bool edge_r = (c0 + 2 == t.w);        // this pair ends the strip
      // the pair's cells lie within g of an x face (ghost images)
      const int X0 = t.c + c0 + a.gs.o[0];
      const bool xface = a.gs.g > 0 && ((X0 < a.gs.g) || (X0 + 1 >= a.gs.n[0] - a.gs.g));
      // rows in three register slots indexed by (row - (y0-1)) mod 3: R is a
      // multiple of 3, so the S/C/N roles are compile-time and nothing moves
      double rw[3] = {0, 0, 0}, ra[3] = {0, 0, 0}, rb[3] = {0, 0, 0}, re[3] = {0, 0, 0};
      for (int st = 0; st < nst; ++st) {
        double hw[R], he[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          hw[i] = hw_next[i];
          he[i] = he_next[i];
        }
        // prefetch the halos of the next stage (this item's or the next item's)
        if (st + 1 < nst) {
          load_halo(t, st + 1);
        } else if (it + (int)gridDim.x < nitems) {
          load_halo(item_of<W, PUSH>(a, it + gridDim.x, nstrips, crows), 0);
        }
        mbar_wait(&full[slot], phase);
        const double* sp = smem + (size_t)slot * STAGE_DOUBLES;
        const bool full_stage = (t.y0 - 1 + st * R + R - 1 <= t.y1) && (t.y0 - 1 + st * R - 1 >= t.y0);
        // ghost images from this stage: the pair is at an x face, or a row of
        // the stage lies within g of a y face (decided once per stage, so the
        // per-row test below is skipped in the bulk of the domain)
        bool stage_img = false;
        if (MODE == MODE_RELAX && a.gs.g > 0) {
          const int Ylo = t.y0 - 2 + st * R + a.gs.o[1], Yhi = Ylo + R - 1;
          stage_img = xface || Ylo < a.gs.g || Yhi >= a.gs.n[1] - a.gs.g;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
          constexpr int dummy = 0;
          (void)dummy;
          const int n_ = i % 3, c_ = (i + 2) % 3, s_ = (i + 1) % 3;  // N, C, S slots
          const int yf = t.y0 - 1 + st * R + i;
          if (!full_stage && yf > t.y1) break;
          // row N = φ row yf, from shared memory
          if (live) {
            const double2 pr = *reinterpret_cast<const double2*>(sp + i * W + c0);
            ra[n_] = pr.x;
            rb[n_] = pr.y;
            rw[n_] = left ? hw[i] : sp[i * W + c0 - 1];
            re[n_] = edge_r ? he[i] : sp[i * W + c0 + 2];
          }
          const int r = yf - 1;  // the row computed now
          if (live && (full_stage || r >= t.y0)) {
            const double w_c = rw[c_], a_c = ra[c_], b_c = rb[c_], e_c = re[c_];
            const double w_s = rw[s_], a_s = ra[s_], b_s = rb[s_], e_s = re[s_];
            const double w_n = rw[n_], a_n = ra[n_], b_n = rb[n_], e_n = re[n_];
            double L0, L1;
            if (ST == 0) {
              // -4·C is exact, so the fused multiply-add rounds like the separate ops
              L0 = fma(-4.0, a_c, __dadd_rn(__dadd_rn(__dadd_rn(w_c, b_c), a_s), a_n));
              L1 = fma(-4.0, b_c, __dadd_rn(__dadd_rn(__dadd_rn(a_c, e_c), b_s), b_n));
              (void)w_s;
              (void)e_s;
              (void)w_n;
              (void)e_n;
            } else {
              double q;
              q = __dmul_rn(4.0, w_c);
              q = fma(4.0, b_c, q);  // 4·x exact: fma == separate ops
              q = fma(4.0, a_s, q);
              q = fma(4.0, a_n, q);
              q = __dadd_rn(q, w_s);
              q = __dadd_rn(q, b_s);
              q = __dadd_rn(q, w_n);
              q = __dadd_rn(q, b_n);
              L0 = __dadd_rn(q, __dmul_rn(-20.0, a_c));
              q = __dmul_rn(4.0, a_c);
              q = fma(4.0, e_c, q);
              q = fma(4.0, b_s, q);
              q = fma(4.0, b_n, q);
              q = __dadd_rn(q, a_s);
              q = __dadd_rn(q, e_s);
              q = __dadd_rn(q, a_n);
              q = __dadd_rn(q, e_n);
              L1 = __dadd_rn(q, __dmul_rn(-20.0, b_c));
            }
            const double2 f = *reinterpret_cast<const double2*>(sp + (R + i) * W + c0);
            // scale, λ powers of two (P2): the products are exact, fma rounds like the separate ops
            const double e0 = P2 ? fma(a.scale, L0, -f.x) : __dsub_rn(__dmul_rn(a.scale, L0), f.x);
            const double e1 = P2 ? fma(a.scale, L1, -f.y) : __dsub_rn(__dmul_rn(a.scale, L1), f.y);
            mxd = fmax(mxd, fabs(e0));
            mxd = fmax(mxd, fabs(e1));
            ss = fma(e0, e0, ss);
            ss = fma(e1, e1, ss);
            if (MODE == MODE_RELAX) {
              const double o0 = PL ? fma(a.lambda, e0, a_c) : __dadd_rn(a_c, __dmul_rn(a.lambda, e0));
              const double o1 = PL ? fma(a.lambda, e1, b_c) : __dadd_rn(b_c, __dmul_rn(a.lambda, e1));
              const int x = t.c + c0;
              double* dp = a.dst + (int64_t)r * a.ld_dst + x;
              *reinterpret_cast<double2*>(dp) = make_double2(o0, o1);
              if (stage_img) {
                const int Y = r + a.gs.o[1];
                if (xface || Y < a.gs.g || Y >= a.gs.n[1] - a.gs.g) {
                  images(a, x, r, o0);
                  images(a, x + 1, r, o1);
                }
              }
            }
          }
        }
        // order this warp's shared-memory reads of the stage before the
        // producer's next TMA write into it (generic -> async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == NST) {
          slot = 0;
          phase ^= 1u;
        }
      }
      if (PUSH && ((t.y0 == 0 && a.ps.rdst[0]) || (t.y1 == a.ny && a.ps.rdst[1])))
        push_rows(a.dst, a.ld_dst, t.y0 == 0 ? a.ps.rdst[0] : nullptr, t.y1 == a.ny ? a.ps.rdst[1] : nullptr, a.ny,
                  a.ps.g, t.c + c0, live, a.ps.xg > 0 && (X0 < a.ps.xg || X0 + 1 >= a.ps.xn0 - a.ps.xg), X0,
                  a.ps.xg, a.ps.xn0, a.ps.xm0, a.ps.xm1);
      if (it + (int)gridDim.x < nitems) t = item_of<W, PUSH>(a, it + gridDim.x, nstrips, crows);
    }
  }
  if (a.norms.out_max) {
    const unsigned long long mx =
        isnan(ss) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(mxd);
    reduce_norms(a.norms, mx, ss);
  }
}

// PROTOX_PDL=0 (read once) launches the sweep kernels without programmatic
// dependent launch (A/B)
static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PROTOX_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int g_nsm = 0;
static int num_sms() {
  if (!g_nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsm <= 0) g_nsm = 148;
  }
  return g_nsm;
}

// Ring configurations built (stages x rows per stage x CTAs per SM); the
// default is the measured best at 16384² (profiles/).
// PROTOX_BULK_CFG=<index> selects another for A/B, PROTOX_BULK_CHUNK the
// nominal rows per work item.
struct BulkCfg {
  int nst, r, cps, nc;
};
// {stages, rows per stage, CTAs per SM, consumer warps}; measured at 16384²
// (GB/s, profiles/round1_bulk_configs.json).  Rows live in 3 register slots
// (row mod 3), so R is a multiple of 3: {3,3,2,8} 6244, {4,3,2,8} 6208,
// {4,3,1,15} 6202, {3,3,3,7} 5769 (spills at 80 registers).  Earlier R = 2
// variants with register moves: {3,2,3,7} 6171-6195, {3,2,3,8} 6118-6132,
// {3,4,2,8} 5917, {5,4,1,8} 5433.
static const BulkCfg kCfgs[] = {{3, 3, 2, 8}, {4, 3, 2, 8}, {4, 3, 1, 15}, {3, 3, 3, 7}, {5, 3, 1, 8}};
static const BulkCfg& bulk_cfg() {
  static int idx = -1;
  if (idx < 0) {
    idx = 0;
    if (const char* e = getenv("PROTOX_BULK_CFG")) {
      const int v = atoi(e);
      if (v >= 0 && v < (int)(sizeof(kCfgs) / sizeof(kCfgs[0]))) idx = v;
    }
  }
  return kCfgs[idx];
}
// the fused push always runs the default configuration (its arrival count
// depends on the strip width)
static const BulkCfg& cfg_for(const StreamLaunch& a) { return a.ps.on ? kCfgs[0] : bulk_cfg(); }
static int bulk_chunk() {
  static int c = 0;
  if (!c) {
    c = CHUNK_ROWS;
    if (const char* e = getenv("PROTOX_BULK_CHUNK")) {
      const int v = atoi(e);
      if (v >= 8 && v <= 65536) c = v;
    }
  }
  return c;
}

bool bulk_eligible(int mode, const StreamLaunch& a) {
  static int disabled = -1;
  if (disabled < 0) {
    const char* e = getenv("PROTOX_KERNEL");
    disabled = (e && e[0] == 'l') ? 1 : 0;  // PROTOX_KERNEL=ldg forces the LDG kernel (A/B)
  }
  if (disabled) return false;
  if (mode != MODE_RELAX && mode != MODE_RESID) return false;
  if (a.phase != 0 || (a.nx & 1) || a.nx <= 0 || a.ny <= 0) return false;
  // small (L2-resident, launch-bound) problems cannot fill a persistent grid;
  // the fused peer-memory push runs in this kernel at any size
  if (!a.ps.on && (int64_t)a.nx * a.ny < (int64_t)4 * 1024 * 1024) return false;
  if (a.ps.on && (mode != MODE_RELAX || a.ps.g < 1 || a.ny < a.ps.g)) return false;
  if ((a.ld_src & 1) || (mode == MODE_RELAX && (a.ld_dst & 1)) || (a.ld_rhs & 1)) return false;
  // bulk copies need 16-byte aligned row starts
  if (((uintptr_t)a.src & 15) || ((uintptr_t)a.rhs & 15)) return false;
  return true;
}

// Work decomposition: strips of W columns x chunks of rows.  The chunk
// count is chosen (from the nominal CHUNK_ROWS up to twice as many chunks)
// so that the item count divides evenly over the persistent grid.
struct BulkGeom {
  int nstrips, nchunks, crows, nitems, grid;
};
static BulkGeom bulk_geom(const StreamLaunch& a) {
  BulkGeom g;
  const BulkCfg& cfg = cfg_for(a);
  g.nstrips = (a.nx + 64 * cfg.nc - 1) / (64 * cfg.nc);
  const int per_sm = cfg.cps;
  int gmax = num_sms() * per_sm < BULK_MAX_GRID ? num_sms() * per_sm : BULK_MAX_GRID;
  const int c0 = (a.ny + bulk_chunk() - 1) / bulk_chunk();
  double best = 1e30;
  g.nchunks = a.ps.on ? 1 : c0;
  // up to twice the nominal chunk count, or enough chunks to give every CTA an item
  const int cmax = 2 * c0 > (gmax + g.nstrips - 1) / g.nstrips ? 2 * c0 : (gmax + g.nstrips - 1) / g.nstrips;
  for (int c = c0; c <= cmax && c <= a.ny; ++c) {
    const int rows = (a.ny + c - 1) / c;
    const int cc = (a.ny + rows - 1) / rows;       // chunks actually produced
    // push mode: each pushed block of g boundary rows lies within one chunk
    if (a.ps.on && (rows < a.ps.g || a.ny - (cc - 1) * rows < a.ps.g)) continue;
    const int items = g.nstrips * cc;
    const int waves = (items + gmax - 1) / gmax;
    // time ~ waves * (rows + 2): balance and per-chunk halo overhead
    const double cost = (double)waves * (rows + 2);
    if (cost < best - 1e-9) {
      best = cost;
      g.nchunks = cc;
    }
  }
  g.crows = (a.ny + g.nchunks - 1) / g.nchunks;
  g.nchunks = (a.ny + g.crows - 1) / g.crows;
  g.nitems = g.nstrips * g.nchunks;
  g.grid = g.nitems < gmax ? g.nitems : gmax;
  return g;
}

int32_t bulk_blocks(const StreamLaunch& a) { return bulk_geom(a).grid; }

int32_t bulk_push_arrivals(const StreamLaunch& a) {
  if (!a.ps.on || !bulk_eligible(MODE_RELAX, a)) return 0;
  const BulkGeom g = bulk_geom(a);
  // every boundary item must be some CTA's first item (the kernel-start wait)
  if ((g.nchunks > 1 ? 2 : 1) * g.nstrips > g.grid) return 0;
  return 1;  // one count per side per sweep (CTA 0 of the next kernel)
}

template <int MODE, int ST, int NST, int R, int CPS, int NC, int PW, int PUSH = 0>
static cudaError_t launch_b(const StreamLaunch& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_bulk<MODE, ST, NST, R, CPS, NC, PW, PUSH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes<NST, R, NC>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const BulkGeom g = bulk_geom(a);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(NC * 32 + 32);
  cfg.dynamicSmemBytes = smem_bytes<NST, R, NC>();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (a.pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_bulk<MODE, ST, NST, R, CPS, NC, PW, PUSH>, a, g.nstrips, g.nitems, g.crows);
}

static bool is_pow2(double v) {
  if (!(v > 0.0) || !std::isfinite(v)) return false;
  int e;
  return std::frexp(v, &e) == 0.5;
}

template <int MODE, int ST, int PW>
static cudaError_t launch_pw(const StreamLaunch& a, cudaStream_t s) {
  if constexpr (MODE == MODE_RELAX) {
    if (a.ps.on) return launch_b<MODE, ST, 3, 3, 2, 8, PW, 1>(a, s);  // = kCfgs[0]
  }
  const BulkCfg& c = bulk_cfg();
  if (c.nc == 8 && c.nst == 4) return launch_b<MODE, ST, 4, 3, 2, 8, PW>(a, s);
  if (c.nc == 15) return launch_b<MODE, ST, 4, 3, 1, 15, PW>(a, s);
  if (c.nc == 7) return launch_b<MODE, ST, 3, 3, 3, 7, PW>(a, s);
  if (c.nst == 5) return launch_b<MODE, ST, 5, 3, 1, 8, PW>(a, s);
  return launch_b<MODE, ST, 3, 3, 2, 8, PW>(a, s);
}

template <int MODE, int ST>
static cudaError_t launch_cfg(const StreamLaunch& a, cudaStream_t s) {
  const int pw = (is_pow2(a.scale) ? 1 : 0) | (is_pow2(a.lambda) ? 2 : 0);
  switch (pw) {
    case 3: return launch_pw<MODE, ST, 3>(a, s);
    case 2: return launch_pw<MODE, ST, 2>(a, s);
    case 1: return launch_pw<MODE, ST, 1>(a, s);
    default: return launch_pw<MODE, ST, 0>(a, s);
  }
}

px_status launch_bulk(int mode, int stencil, const StreamLaunch& a, cudaStream_t s) {
  cudaError_t e;
  switch (mode * 2 + stencil) {
    case MODE_RELAX * 2 + 0: e = launch_cfg<MODE_RELAX, 0>(a, s); break;
    case MODE_RELAX * 2 + 1: e = launch_cfg<MODE_RELAX, 1>(a, s); break;
    case MODE_RESID * 2 + 0: e = launch_cfg<MODE_RESID, 0>(a, s); break;
    case MODE_RESID * 2 + 1: e = launch_cfg<MODE_RESID, 1>(a, s); break;
    default: return fail(PX_ERR_ARG, "bulk kernel: bad mode");
  }
  if (mode == MODE_RELAX) note_kernel("k_bulk");
  count_launches(1);
  return cuda_check(e, "bulk relax kernel launch");
}

}  // namespace px
