// px3d.cu -- the 3D relaxation: the fused 7-point
// point-Jacobi sweep of the 3D Poisson equation on one device.
//
// The paper's Point and Box are dimension-generic (Z^D) and
// its step size is λ = h²/(4D); the 7-point Laplacian is the
// D = 3 form of Eq.1.  Per cell, in the oracle's expression
// tree (R-3D1, oracle/protox_oracle3d.cpp):
//     L = (((((W + E) + S) + N) + B) + T) + (-6·C)
//     r = scale·L − ρ,   φ' = φ + λ·r       (every * and + rounded once)
// plus the residual norms max|r| (u64 bit max, NaN-propagating) and Σr².
//
// k3_relax: a persistent grid (one 288-thread CTA per SM: 8 consumer warps +
// 1 producer warp).  A work item is a 64 x 32 (x, y) tile and a range of z
// planes; the CTA marches the tile up in z.  Per plane the producer's elected
// lane issues two TMA TENSOR copies (cp.async.bulk.tensor.3d, SASS UTMALDG)
// into a 4-stage shared-memory ring guarded by full/empty mbarriers: the φ
// plane with its x/y halo (68 x 34 doubles) and the ρ tile of the previous
// plane (ρ lags φ by one plane).  Consumer thread (warp w, lane l) owns the
// cell pair x0+2l, x0+2l+1 in rows y0+4w .. y0+4w+3: W/E and S/N come from
// the plane's halo box in shared memory, T from the next plane's box, B from
// registers (the pair's values of the previous plane).  HBM traffic: φ read
// once (+ halo re-reads served by L2), ρ read once, φ' written once: 24 B per
// cell-update algorithmic.  Ghost cells are filled by k3_ghost (separate
// launches, 6/n of the traffic) -- periodic wrap / odd reflection per face,
// phased x, y, z so edges and corners follow the product rule.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "px_device.cuh"
#include "px_internal.h"
#include "px_ptx.cuh"

namespace px {
namespace k3 {

constexpr int TX = 64, TY = 32;             // tile (x, y)
constexpr int BXW = TX + 4, BYH = TY + 2;   // φ box: columns x0-2 .. x0+TX+1, rows y0-1 .. y0+TY
constexpr int NWC = 8;                      // consumer warps, warp w: tile rows 4w .. 4w+3
constexpr int RPW = TY / NWC;               // rows per warp (4)
constexpr int THREADS = NWC * 32 + 32;
constexpr int PHI_PAD = (BXW * BYH + 15) / 16 * 16;  // 128-byte aligned ρ tile
constexpr int STAGE = PHI_PAD + TX * TY;             // doubles
constexpr uint32_t PHI_BYTES = BXW * BYH * 8u;
constexpr uint32_t RHO_BYTES = TX * TY * 8u;
template <int NST>
constexpr size_t smem_bytes() { return (size_t)NST * STAGE * sizeof(double) + 2 * NST * sizeof(uint64_t); }
constexpr int MAX_GRID = 512;

using namespace ptx;

}  // namespace k3

// Launch geometry and scalars of one 3D sweep (or residual pass).
struct Relax3 {
  double* dst;            // cell (0,0,0) of φ' (RELAX); null for RESID
  int64_t ld, plane;      // pitches of dst (elements)
  int32_t n[3];
  int32_t ntx, nty, nzc, zlen;  // tiles in x, y; z chunks of zlen planes
  int32_t nitems;
  double scale, lambda;
  NormSlot norms;
  int32_t policy;         // L2 policies (A/B knob PROTOX_K3_POLICY): 0 ρ evict_first + φ evict_last
};

// r = scale·L − ρ, φ' = φ + λr for the pair, store, accumulate the norms
template <int MODE>
__device__ __forceinline__ void k3_finish(const Relax3& a, const double* tp, int brow, int lane, int cx, int y0,
                                          int z, bool ox0, bool ox1, double2 C, double L0, double L1,
                                          unsigned long long& mx, double& ss) {
  using namespace k3;
  const double2 f = *reinterpret_cast<const double2*>(tp + PHI_PAD + (brow - 1) * TX + 2 * lane);
  const double r0 = __dsub_rn(__dmul_rn(a.scale, L0), f.x);
  const double r1 = __dsub_rn(__dmul_rn(a.scale, L1), f.y);
  const int y = y0 + brow - 1;
  const bool oy = y < a.n[1];
  const bool w0 = ox0 && oy, w1 = ox1 && oy;
  if (MODE == MODE_RELAX) {
    const double o0 = __dadd_rn(C.x, __dmul_rn(a.lambda, r0));
    const double o1 = __dadd_rn(C.y, __dmul_rn(a.lambda, r1));
    double* dp = a.dst + cx + (int64_t)y * a.ld + (int64_t)z * a.plane;
    if (w0 && w1)
      *reinterpret_cast<double2*>(dp) = make_double2(o0, o1);
    else if (w0)
      dp[0] = o0;
  }
  const double q0 = w0 ? r0 : 0.0, q1 = w1 ? r1 : 0.0;
  mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(q0)));
  ss = fma(q0, q0, ss);
  mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(q1)));
  ss = fma(q1, q1, ss);
}

// Undivided 27-point Mehrstellen sum (R-3D4) of one cell, v(q, dy, dx) the
// value at plane z+q-1: the oracle's tap order, every product and sum rounded.
template <class V>
__device__ __forceinline__ double m27(const V& v) {
  double acc = __dmul_rn(14.0, v(1, 0, -1));  // faces W, E, S, N, B, T
  acc = __dadd_rn(acc, __dmul_rn(14.0, v(1, 0, 1)));
  acc = __dadd_rn(acc, __dmul_rn(14.0, v(1, -1, 0)));
  acc = __dadd_rn(acc, __dmul_rn(14.0, v(1, 1, 0)));
  acc = __dadd_rn(acc, __dmul_rn(14.0, v(0, 0, 0)));
  acc = __dadd_rn(acc, __dmul_rn(14.0, v(2, 0, 0)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(1, -1, -1)));  // edges xy
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(1, -1, 1)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(1, 1, -1)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(1, 1, 1)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(0, 0, -1)));  // edges xz
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(0, 0, 1)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(2, 0, -1)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(2, 0, 1)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(0, -1, 0)));  // edges yz
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(0, 1, 0)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(2, -1, 0)));
  acc = __dadd_rn(acc, __dmul_rn(3.0, v(2, 1, 0)));
  acc = __dadd_rn(acc, v(0, -1, -1));  // corners, z-major
  acc = __dadd_rn(acc, v(0, -1, 1));
  acc = __dadd_rn(acc, v(0, 1, -1));
  acc = __dadd_rn(acc, v(0, 1, 1));
  acc = __dadd_rn(acc, v(2, -1, -1));
  acc = __dadd_rn(acc, v(2, -1, 1));
  acc = __dadd_rn(acc, v(2, 1, -1));
  acc = __dadd_rn(acc, v(2, 1, 1));
  return __dadd_rn(acc, __dmul_rn(-128.0, v(1, 0, 0)));
}

// The map's origin is cell (-2, -g, -g) of the patch, so tensor coordinate
// (c0, c1, c2) is cell (c0 - 2, c1 - g, c2 - g).
template <int MODE, int NST, int ST>
__global__ void __maxnreg__(ST == 1 ? 168 : 112)  // 9 warps: 3 share a sub-partition (16K regs)
    k3_relax(const __grid_constant__ CUtensorMap mphi, const __grid_constant__ CUtensorMap mrho, const Relax3 a,
             int g) {
  using namespace k3;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * STAGE);
  uint64_t* empty = full + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long mx = 0ull;
  double ss = 0.0;
  if (warp == NWC) {
    // ------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mphi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mrho)) : "memory");
      uint64_t pol, pol_halo;  // ρ: read once; φ planes: their halo rows are re-read by the neighbouring tiles
      if (a.policy == 0) {
        pol = evict_first_policy();
        pol_halo = evict_last_policy();
      } else if (a.policy == 1) {
        pol = evict_normal_policy();
        pol_halo = pol;
      } else {
        pol = evict_first_policy();
        pol_halo = evict_normal_policy();
      }
      int slot = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
        const int tx = it % a.ntx, rest = it / a.ntx, ty = rest % a.nty, zc = rest / a.nty;
        const int x0 = tx * TX, y0 = ty * TY, z0 = zc * a.zlen, z1 = min(a.n[2], z0 + a.zlen);
        const int nstg = z1 - z0 + 2;
        for (int s = 0; s < nstg; ++s) {
          mbar_wait(&empty[slot], phase ^ 1u);
          double* sp = smem + (size_t)slot * STAGE;
          const bool rho = s >= 2;
          mbar_arrive_expect_tx(&full[slot], PHI_BYTES + (rho ? RHO_BYTES : 0u));
          // φ plane z0-1+s with its halo: cells (x0-2.., y0-1.., z)
          tma3(sp, &mphi, x0, y0 - 1 + g, z0 - 1 + s + g, &full[slot], pol_halo);
          if (rho) tma3(sp + PHI_PAD, &mrho, x0 + 2, y0 + g, z0 - 2 + s + g, &full[slot], pol);
          if (++slot == NST) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------ consumers
    int slot = 0;
    uint32_t phase = 0;
    const int bc = 2 * lane + 2;  // box column of the pair
    for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
      const int tx = it % a.ntx, rest = it / a.ntx, ty = rest % a.nty, zc = rest / a.nty;
      const int x0 = tx * TX, y0 = ty * TY, z0 = zc * a.zlen, z1 = min(a.n[2], z0 + a.zlen);
      const int cx = x0 + 2 * lane;
      const bool ox0 = cx < a.n[0], ox1 = cx + 1 < a.n[0];
      double2 Bv[RPW];
      // stage 0: plane z0-1 -> B (7-point: its pair values in registers, the
      // stage released at once; 27-point: the whole box is held as the B plane)
      mbar_wait(&full[slot], phase);
      int bslot = slot;
      if (ST == 0) {
        const double* sp = smem + (size_t)slot * STAGE;
#pragma unroll
        for (int i = 0; i < RPW; ++i)
          Bv[i] = *reinterpret_cast<const double2*>(sp + (RPW * warp + i + 1) * BXW + bc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
      if (++slot == NST) {
        slot = 0;
        phase ^= 1u;
      }
      // stage 1: plane z0 (held: the C plane of the first step)
      mbar_wait(&full[slot], phase);
      int cslot = slot;
      if (++slot == NST) {
        slot = 0;
        phase ^= 1u;
      }
      for (int z = z0; z < z1; ++z) {
        mbar_wait(&full[slot], phase);  // plane z+1 and ρ(z)
        const double* cp = smem + (size_t)cslot * STAGE;
        const double* tp = smem + (size_t)slot * STAGE;
        if (ST == 0) {
          double2 r[RPW + 2];
#pragma unroll
          for (int i = 0; i < RPW + 2; ++i) r[i] = *reinterpret_cast<const double2*>(cp + (RPW * warp + i) * BXW + bc);
#pragma unroll
          for (int i = 0; i < RPW; ++i) {
            const int brow = RPW * warp + i + 1;
            const double2 C = r[i + 1], S = r[i], N = r[i + 2];
            const double W = cp[brow * BXW + bc - 1], E = cp[brow * BXW + bc + 2];
            const double2 T = *reinterpret_cast<const double2*>(tp + brow * BXW + bc);
            const double2 B = Bv[i];
            double L0 = __dadd_rn(W, C.y);
            L0 = __dadd_rn(L0, S.x);
            L0 = __dadd_rn(L0, N.x);
            L0 = __dadd_rn(L0, B.x);
            L0 = __dadd_rn(L0, T.x);
            L0 = __dadd_rn(L0, __dmul_rn(-6.0, C.x));
            double L1 = __dadd_rn(C.x, E);
            L1 = __dadd_rn(L1, S.y);
            L1 = __dadd_rn(L1, N.y);
            L1 = __dadd_rn(L1, B.y);
            L1 = __dadd_rn(L1, T.y);
            L1 = __dadd_rn(L1, __dmul_rn(-6.0, C.y));
            k3_finish<MODE>(a, tp, brow, lane, cx, y0, z, ox0, ox1, C, L0, L1, mx, ss);
            Bv[i] = C;
          }
        } else {
          // 27-point: rows 4w .. 4w+5 of the B, C, T plane boxes (pairs and the
          // W / E neighbours), then the taps in the oracle's order (R-3D4)
          const double* bp = smem + (size_t)bslot * STAGE;
          // rolling window of three rows per plane (slot = row mod 3)
          double2 P[3][3];
          double Wv[3][3], Ev[3][3];
          auto load_row = [&](int k) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const double* rp = (q == 0 ? bp : (q == 1 ? cp : tp)) + (RPW * warp + k) * BXW + bc;
              P[q][k % 3] = *reinterpret_cast<const double2*>(rp);
              Wv[q][k % 3] = rp[-1];
              Ev[q][k % 3] = rp[2];
            }
          };
          load_row(0);
          load_row(1);
#pragma unroll
          for (int i = 0; i < RPW; ++i) {
            load_row(i + 2);
            const int brow = RPW * warp + i + 1;
            // value of (plane q = dz+1, dy, dx) for the pair's cell 0 / cell 1
            auto v0 = [&](int q, int dy, int dx) {
              const int k = (i + 1 + dy) % 3;
              return dx < 0 ? Wv[q][k] : (dx == 0 ? P[q][k].x : P[q][k].y);
            };
            auto v1 = [&](int q, int dy, int dx) {
              const int k = (i + 1 + dy) % 3;
              return dx < 0 ? P[q][k].x : (dx == 0 ? P[q][k].y : Ev[q][k]);
            };
            const double L0 = m27(v0), L1 = m27(v1);
            k3_finish<MODE>(a, tp, brow, lane, cx, y0, z, ox0, ox1, P[1][(i + 1) % 3], L0, L1, mx, ss);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[bslot]);  // plane z-1 no longer needed
          bslot = cslot;
        }
        if (ST == 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[cslot]);  // plane z no longer needed
        }
        cslot = slot;
        if (++slot == NST) {
          slot = 0;
          phase ^= 1u;
        }
      }
      if (ST == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[bslot]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cslot]);  // the item's last plane
    }
  }
  if (a.norms.out_max) reduce_norms(a.norms, mx, ss);
}

// Ghost layer of one dimension D: periodic wrap (mode 1) or odd reflection
// (mode 2) of the owned cells; dimensions before D cover their ghosts too
// (phased x, y, z: edges and corners by the product rule).
template <int D>
__global__ void k3_ghost(double* o, int64_t ld, int64_t plane, int n0, int n1, int n2, int g, int mode,
                         int sides) {
  const int n[3] = {n0, n1, n2};
  // extents of the face set: dims < D padded, D ghost-only (2g), dims > D interior
  int e[3];
  for (int d = 0; d < 3; ++d) e[d] = d < D ? n[d] + 2 * g : (d == D ? 2 * g : n[d]);
  const int64_t total = (int64_t)e[0] * e[1] * e[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    int64_t t = i;
    for (int d = 0; d < 3; ++d) {
      c[d] = (int)(t % e[d]);
      t /= e[d];
    }
    for (int d = 0; d < 3; ++d) {
      if (d < D) c[d] -= g;
      if (d == D) c[d] = c[d] < g ? c[d] - g : n[d] + (c[d] - g);
    }
    int s[3] = {c[0], c[1], c[2]};
    double sign = 1.0;
    const int cd = c[D];
    if (!(sides & (cd < 0 ? 1 : 2))) continue;  // bit 0: lower face, bit 1: upper face
    if (mode == GH_WRAP) {
      s[D] = cd < 0 ? cd + n[D] : cd - n[D];
    } else {
      s[D] = cd < 0 ? -cd - 1 : 2 * n[D] - 1 - cd;
      sign = -1.0;
    }
    const double v = o[s[0] + (int64_t)s[1] * ld + (int64_t)s[2] * plane];
    o[c[0] + (int64_t)c[1] * ld + (int64_t)c[2] * plane] = sign * v;
  }
}

// f = ρ + c12·S7(ρ) over the owned cells (27-point right-hand side, R-3D4);
// ρ's ghosts must be filled.  S7 in the canonical order W,E,S,N,B,T, −6C.
__global__ void k3_mrhs(const double* rho, double* f, int64_t ld, int64_t plane, int n0, int n1, int n2,
                        double c12) {
  const int64_t total = (int64_t)n0 * n1 * n2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % n0);
    const int64_t r = i / n0;
    const int y = (int)(r % n1), z = (int)(r / n1);
    const double* c = rho + x + (int64_t)y * ld + (int64_t)z * plane;
    double L = __dadd_rn(c[-1], c[1]);
    L = __dadd_rn(L, c[-ld]);
    L = __dadd_rn(L, c[ld]);
    L = __dadd_rn(L, c[-plane]);
    L = __dadd_rn(L, c[plane]);
    L = __dadd_rn(L, __dmul_rn(-6.0, c[0]));
    f[x + (int64_t)y * ld + (int64_t)z * plane] = __dadd_rn(c[0], __dmul_rn(c12, L));
  }
}

__device__ __forceinline__ uint64_t splitmix64_3(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// synthetic fields: kind 0 zero, 1 counter hash of the global cell index
// x + n0 (y + n1 (z + z0)) (the 2D recipe in 3D; z0 = the slab's first
// global plane), owned cells only
__global__ void k3_init(double* o, int64_t ld, int64_t plane, int n0, int n1, int n2, int kind, uint64_t seed,
                        int z0) {
  const int64_t total = (int64_t)n0 * n1 * n2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % n0);
    const int64_t r = i / n0;
    const int y = (int)(r % n1), z = (int)(r / n1);
    double v = 0.0;
    if (kind == 1) {
      const uint64_t u = splitmix64_3(seed ^ (uint64_t)(i + (int64_t)z0 * n0 * n1));
      v = ((double)(u >> 11) * 0x1p-53) * 2.0 - 1.0;
    }
    o[x + (int64_t)y * ld + (int64_t)z * plane] = v;
  }
}

// ------------------------------------------------------------------- host
static int k3_nsm() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Tensor map over cells (-2 .. n0+1, -g .. n1+g-1, -g .. n2+g-1) of a patch.
static px_status make_map(const px_patch3& p, uint32_t bx, uint32_t by, CUtensorMap* m) {
  auto fn = encode_fn();
  if (!fn) return fail(PX_ERR_CUDA, "cuTensorMapEncodeTiled not available from the driver");
  const int g = p.ghost;
  double* base = p.data - 2 - (int64_t)g * p.ld - (int64_t)g * p.plane;
  cuuint64_t dims[3] = {(cuuint64_t)p.n[0] + 4, (cuuint64_t)p.n[1] + 2 * g, (cuuint64_t)p.n[2] + 2 * g};
  cuuint64_t strides[2] = {(cuuint64_t)p.ld * 8, (cuuint64_t)p.plane * 8};
  cuuint32_t box[3] = {bx, by, 1};
  cuuint32_t es[3] = {1, 1, 1};
  static int promo = -1;  // A/B knob PROTOX_K3_PROMO: 0 none, 1 64B, 2 128B (default), 3 256B
  if (promo < 0) {
    const char* ev = getenv("PROTOX_K3_PROMO");
    promo = ev ? atoi(ev) : 2;
    if (promo < 0 || promo > 3) promo = 2;
  }
  const CUtensorMapL2promotion pr[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, pr[promo], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PX_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PX_OK;
}

// z chunks: items = tiles x chunks; minimise waves x (planes per chunk + 2)
// ring stages and CTAs per SM: 4 stages x 1 CTA (default) or 3 stages x 2 CTAs
// (PROTOX_K3_NST=3 selects the latter; 6 = six stages x 1 CTA), A/B knob
static int k3_nst() {
  static int nst = -1;
  if (nst < 0) {
    const char* ev = getenv("PROTOX_K3_NST");
    nst = ev ? atoi(ev) : 4;
    if (nst != 3 && nst != 6) nst = 4;
  }
  return nst;
}

static void plan3(const int32_t n[3], Relax3& a, int* grid, int stencil = PX_LAPLACE_7PT_3D) {
  a.ntx = (n[0] + k3::TX - 1) / k3::TX;
  a.nty = (n[1] + k3::TY - 1) / k3::TY;
  const int tiles = a.ntx * a.nty;
  const int cps = (k3_nst() == 3 && stencil == PX_LAPLACE_7PT_3D) ? 2 : 1;
  const int gmax = cps * k3_nsm() < k3::MAX_GRID ? cps * k3_nsm() : k3::MAX_GRID;
  double best = 1e30;
  int bc = 1;
  for (int c = 1; c <= n[2] && c <= 64; ++c) {
    const int zl = (n[2] + c - 1) / c;
    const int cc = (n[2] + zl - 1) / zl;
    const int items = tiles * cc;
    const int waves = (items + gmax - 1) / gmax;
    const double cost = (double)waves * (zl + 2);
    if (cost < best - 1e-9) {
      best = cost;
      bc = cc;
    }
  }
  a.zlen = (n[2] + bc - 1) / bc;
  a.nzc = (n[2] + a.zlen - 1) / a.zlen;
  a.nitems = tiles * a.nzc;
  *grid = a.nitems < gmax ? a.nitems : gmax;
}

int32_t relax3_blocks(const int32_t n[3], int stencil) {
  Relax3 a;
  int grid = 0;
  plan3(n, a, &grid, stencil);
  return grid;
}

static px_status check3(const px_patch3* p, const char* name) {
  if (!p || !p->data) return fail(PX_ERR_ARG, "%s: null patch", name);
  for (int d = 0; d < 3; ++d)
    if (p->n[d] < 1) return fail(PX_ERR_SHAPE, "%s: extent %d must be >= 1", name, d);
  if (p->ghost < 1 || p->ghost > 16) return fail(PX_ERR_SHAPE, "%s: ghost width must be in [1, 16]", name);
  if (p->ld < p->n[0] + 4 || p->plane < p->ld * (p->n[1] + 2 * p->ghost))
    return fail(PX_ERR_SHAPE, "%s: pitches too small (ld >= n0 + 4, plane >= ld * (n1 + 2g))", name);
  if ((reinterpret_cast<uintptr_t>(p->data) & 15) || (p->ld & 1) || (p->plane & 1))
    return fail(PX_ERR_ALIGN, "%s: cell (0,0,0) must be 16-byte aligned and ld, plane even", name);
  return PX_OK;
}

static px_status same_shape3(const px_patch3& a, const px_patch3& b, const char* name) {
  if (a.n[0] != b.n[0] || a.n[1] != b.n[1] || a.n[2] != b.n[2] || a.ghost != b.ghost)
    return fail(PX_ERR_SHAPE, "%s: extents / ghost width differ from phi", name);
  return PX_OK;
}

static bool positive_finite(double h) { return h > 0.0 && std::isfinite(h); }

template <int MODE, int NST, int ST>
static cudaError_t k3_go(const CUtensorMap& mphi, const CUtensorMap& mrho, const Relax3& a, int g, int grid,
                         cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k3_relax<MODE, NST, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)k3::smem_bytes<NST>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k3_relax<MODE, NST, ST><<<grid, k3::THREADS, k3::smem_bytes<NST>(), s>>>(mphi, mrho, a, g);
  return cudaSuccess;
}

static px_status launch_relax3(int mode, const px_relax_params& prm, const px_patch3& in, const px_patch3* out,
                               const px_patch3& rhs, const NormSlot& ns, cudaStream_t s) {
  CUtensorMap mphi, mrho;
  PX_TRY(make_map(in, k3::BXW, k3::BYH, &mphi));
  PX_TRY(make_map(rhs, k3::TX, k3::TY, &mrho));
  Relax3 a;
  std::memset(&a, 0, sizeof a);
  for (int d = 0; d < 3; ++d) a.n[d] = in.n[d];
  int grid = 0;
  plan3(a.n, a, &grid, prm.stencil);
  a.dst = out ? out->data : nullptr;
  a.ld = out ? out->ld : 0;
  a.plane = out ? out->plane : 0;
  a.scale = prm.stencil == PX_MEHRSTELLEN_27PT_3D ? 1.0 / (30.0 * prm.h * prm.h) : 1.0 / (prm.h * prm.h);
  a.lambda = prm.lambda;
  a.norms = ns;
  static int policy = -1;
  if (policy < 0) {
    const char* ev = getenv("PROTOX_K3_POLICY");
    policy = ev ? atoi(ev) : 0;
  }
  a.policy = policy;
  const int nst = k3_nst();
  cudaError_t e = cudaSuccess;
  if (prm.stencil == PX_MEHRSTELLEN_27PT_3D) {  // three planes held: 5 stages
    e = mode == MODE_RELAX ? k3_go<MODE_RELAX, 5, 1>(mphi, mrho, a, in.ghost, grid, s)
                           : k3_go<MODE_RESID, 5, 1>(mphi, mrho, a, in.ghost, grid, s);
  } else if (mode == MODE_RELAX) {
    if (nst == 3) e = k3_go<MODE_RELAX, 3, 0>(mphi, mrho, a, in.ghost, grid, s);
    else if (nst == 6) e = k3_go<MODE_RELAX, 6, 0>(mphi, mrho, a, in.ghost, grid, s);
    else e = k3_go<MODE_RELAX, 4, 0>(mphi, mrho, a, in.ghost, grid, s);
  } else {
    e = k3_go<MODE_RESID, 4, 0>(mphi, mrho, a, in.ghost, grid, s);
  }
  if (e != cudaSuccess) return cuda_check(e, "3D relax attribute");
  count_launches(1);
  return cuda_check(cudaGetLastError(), "3D relax launch");
}

// ghost layers: dimensions x, y (both sides) and z on the `zsides` faces
// (bit 0 lower, bit 1 upper): the slab solve fills the inter-rank z faces by
// exchange
static px_status launch_ghost3(px_bc bc, const px_patch3& p, cudaStream_t s, int zsides = 3) {
  if (bc == PX_BC_FIXED_GHOSTS) return PX_OK;
  const int mode = bc == PX_BC_PERIODIC ? GH_WRAP : GH_REFLECT;
  const int g = p.ghost;
  if (g > p.n[0] || g > p.n[1] || g > p.n[2])
    return fail(PX_ERR_SHAPE, "ghost width %d exceeds an extent (%d, %d, %d)", g, p.n[0], p.n[1], p.n[2]);
  const int T = 256;
  auto blocks = [&](int64_t cells) {
    int64_t b = (cells + T - 1) / T;
    return (int)(b < 4096 ? (b > 0 ? b : 1) : 4096);
  };
  const int64_t f0 = (int64_t)2 * g * p.n[1] * p.n[2];
  const int64_t f1 = (int64_t)(p.n[0] + 2 * g) * 2 * g * p.n[2];
  const int64_t f2 = (int64_t)(p.n[0] + 2 * g) * (p.n[1] + 2 * g) * 2 * g;
  k3_ghost<0><<<blocks(f0), T, 0, s>>>(p.data, p.ld, p.plane, p.n[0], p.n[1], p.n[2], g, mode, 3);
  k3_ghost<1><<<blocks(f1), T, 0, s>>>(p.data, p.ld, p.plane, p.n[0], p.n[1], p.n[2], g, mode, 3);
  count_launches(2);
  if (zsides) {
    k3_ghost<2><<<blocks(f2), T, 0, s>>>(p.data, p.ld, p.plane, p.n[0], p.n[1], p.n[2], g, mode, zsides);
    count_launches(1);
  }
  return cuda_check(cudaGetLastError(), "3D ghost fill launch");
}

static px_status check_params3(const px_relax_params* p) {
  if (!p) return fail(PX_ERR_ARG, "null params");
  if (p->stencil != PX_LAPLACE_7PT_3D && p->stencil != PX_MEHRSTELLEN_27PT_3D)
    return fail(PX_ERR_UNSUPPORTED, "3D calls take stencil PX_LAPLACE_7PT_3D or PX_MEHRSTELLEN_27PT_3D");
  if (!positive_finite(p->h)) return fail(PX_ERR_ARG, "h must be positive and finite");
  return PX_OK;
}

// norm slot over a caller buffer laid out as px_norm_buffer3_len describes
static NormSlot slot_from(double* d, int32_t expected) {
  NormSlot ns;
  std::memset(&ns, 0, sizeof ns);
  if (!d) return ns;
  ns.out_max = d;
  ns.out_sum = d + 1;
  ns.counter = reinterpret_cast<unsigned int*>(d + 2);
  ns.partials = d + 4;
  ns.offset = 0;
  ns.expected = expected;
  return ns;
}

// Elements spanned by cells (-2 .. n0+1, -g .. n1+g-1, -g .. n2+g-1), starting at cell (-2, -g, -g):
// the memory a 3D patch must provide (the TMA boxes read columns -2 and n0+1).
static int64_t span3(const px_patch3& p) {
  return (int64_t)(p.n[2] + 2 * p.ghost - 1) * p.plane + (int64_t)(p.n[1] + 2 * p.ghost - 1) * p.ld + p.n[0] + 4;
}
static double* start3(const px_patch3& p) { return p.data - 2 - (int64_t)p.ghost * (p.ld + p.plane); }

// ------------------------------------------------------------ solve plan
struct Plan3 {
  // key
  px_comm* comm = nullptr;
  px_bc bc;
  px_relax_params prm;
  px_solve_opts opts;
  px_patch3 a, b, r;
  cudaStream_t s;
  // resources
  double* d_ring = nullptr;  // 2 per entry
  double* d_ws = nullptr;    // counter (2) + partials (2 per block)
  int n_entries = 0;
  int64_t launches_per_run = 0;
  cudaGraphExec_t exec = nullptr;
  ~Plan3() {
    if (exec) cudaGraphExecDestroy(exec);
    if (d_ring) cudaFree(d_ring);
    if (d_ws) cudaFree(d_ws);
  }
};
static std::unique_ptr<Plan3> g_plan3;

static bool same_key(const Plan3& p, px_comm* comm, px_bc bc, const px_relax_params& prm, const px_solve_opts& o,
                     const px_patch3& a, const px_patch3& b, const px_patch3& r, cudaStream_t s) {
  return p.comm == comm && p.bc == bc && std::memcmp(&p.prm, &prm, sizeof prm) == 0 && std::memcmp(&p.opts, &o, sizeof o) == 0 &&
         std::memcmp(&p.a, &a, sizeof a) == 0 && std::memcmp(&p.b, &b, sizeof b) == 0 &&
         std::memcmp(&p.r, &r, sizeof r) == 0 && p.s == s;
}

static px_status nccl3(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PX_OK;
  return fail(PX_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

// z-slab neighbours of this rank (-1: a domain face handled locally)
static void slab_nbrs(const Plan3& P, int* lo, int* hi) {
  *lo = *hi = -1;
  if (!P.comm) return;
  const int np = comm_nranks(P.comm), r = comm_rank(P.comm);
  const bool per = P.bc == PX_BC_PERIODIC;
  if (np == 1) {
    if (per && comm_self_exchange(P.comm)) *lo = *hi = 0;  // test mode: the rank is its own neighbour
    return;
  }
  *lo = r > 0 ? r - 1 : (per ? np - 1 : -1);
  *hi = r < np - 1 ? r + 1 : (per ? 0 : -1);
}

// ghost fill of one iterate: x, y locally; z planes from the slab neighbours
// (one NCCL group, posted send-up, send-down, recv-down, recv-up -- NCCL
// matches a peer pair's sends and receives in posting order, so two ranks on
// a periodic ring pair the right planes) or locally at a domain face.
static px_status exchange3(const Plan3& P, const px_patch3& p) {
  int lo, hi;
  slab_nbrs(P, &lo, &hi);
  const int zs = (lo < 0 ? 1 : 0) | (hi < 0 ? 2 : 0);
  if (!P.comm) return launch_ghost3(P.bc, p, P.s, 3);
  PX_TRY(launch_ghost3(P.bc, p, P.s, zs));
  if (lo < 0 && hi < 0) return PX_OK;
  // a full plane, cells (-2 .. n0+1, -g .. n1+g-1) of plane z
  const int g = p.ghost, nz = p.n[2];
  const size_t cnt = (size_t)(p.n[1] + 2 * g - 1) * p.ld + p.n[0] + 4;
  auto plane_at = [&](int z) { return p.data + (int64_t)z * p.plane - (int64_t)g * p.ld - 2; };
  ncclComm_t nc = (ncclComm_t)comm_nccl(P.comm);
  PX_TRY(nccl3(ncclGroupStart(), "ncclGroupStart"));
  if (hi >= 0) PX_TRY(nccl3(ncclSend(plane_at(nz - 1), cnt, ncclDouble, hi, nc, P.s), "ncclSend up"));
  if (lo >= 0) PX_TRY(nccl3(ncclSend(plane_at(0), cnt, ncclDouble, lo, nc, P.s), "ncclSend down"));
  if (lo >= 0) PX_TRY(nccl3(ncclRecv(plane_at(-1), cnt, ncclDouble, lo, nc, P.s), "ncclRecv down"));
  if (hi >= 0) PX_TRY(nccl3(ncclRecv(plane_at(nz), cnt, ncclDouble, hi, nc, P.s), "ncclRecv up"));
  return nccl3(ncclGroupEnd(), "ncclGroupEnd");
}

static px_status enqueue_solve3(Plan3& P) {
  const int N = P.opts.nsweeps, E = P.opts.norm_every;
  const int32_t blocks = relax3_blocks(P.a.n, P.prm.stencil);
  const px_patch3* cur = &P.a;
  const px_patch3* nxt = &P.b;
  int entry = 0;
  auto slot = [&](int e) {
    NormSlot ns;
    std::memset(&ns, 0, sizeof ns);
    ns.out_max = P.d_ring + e;  // ring: max[ne] then sum[ne] (all-reduced as two arrays)
    ns.out_sum = P.d_ring + (P.n_entries > 0 ? P.n_entries : 1) + e;
    ns.counter = reinterpret_cast<unsigned int*>(P.d_ws);
    ns.partials = P.d_ws + 2;
    ns.offset = 0;
    ns.expected = blocks;
    return ns;
  };
  for (int it = 0; it < N; ++it) {
    PX_TRY(exchange3(P, *cur));
    NormSlot ns;
    std::memset(&ns, 0, sizeof ns);
    if (E > 0 && it % E == 0) ns = slot(entry++);
    PX_TRY(launch_relax3(MODE_RELAX, P.prm, *cur, nxt, P.r, ns, P.s));
    std::swap(cur, nxt);
  }
  PX_TRY(exchange3(P, *cur));
  if (E >= 0) PX_TRY(launch_relax3(MODE_RESID, P.prm, *cur, nullptr, P.r, slot(entry++), P.s));
  if (P.comm && E >= 0) {  // the residual norms over all ranks, once per solve (R14)
    const int ne = P.n_entries;
    ncclComm_t nc = (ncclComm_t)comm_nccl(P.comm);
    PX_TRY(nccl3(ncclGroupStart(), "ncclGroupStart"));
    // max|r| as u64 bit patterns (non-negative doubles: exact, NaN-propagating, R7)
    PX_TRY(nccl3(ncclAllReduce(P.d_ring, P.d_ring, ne, ncclUint64, ncclMax, nc, P.s), "ncclAllReduce max"));
    PX_TRY(nccl3(ncclAllReduce(P.d_ring + ne, P.d_ring + ne, ne, ncclDouble, ncclSum, nc, P.s), "ncclAllReduce sum"));
    PX_TRY(nccl3(ncclGroupEnd(), "ncclGroupEnd"));
  }
  return PX_OK;
}

}  // namespace px

using namespace px;

extern "C" {

px_status px3_layout(const int32_t n[3], int32_t ghost, int64_t* ld, int64_t* plane, int64_t* origin,
                     int64_t* alloc_elems) {
  clear_error();
  if (!n || !ld || !plane || !origin || !alloc_elems) return fail(PX_ERR_ARG, "null argument");
  for (int d = 0; d < 3; ++d)
    if (n[d] < 1) return fail(PX_ERR_SHAPE, "extent %d must be >= 1", d);
  if (ghost < 1 || ghost > 16) return fail(PX_ERR_SHAPE, "ghost width must be in [1, 16]");
  *ld = ((int64_t)n[0] + 32 + 15) / 16 * 16;
  *plane = *ld * (n[1] + 2 * ghost);
  *origin = 16 + (int64_t)ghost * *ld + (int64_t)ghost * *plane;
  *alloc_elems = *plane * (n[2] + 2 * ghost);
  return PX_OK;
}

int64_t px3_norm_buffer_len(void) { return 4 + 2 * (int64_t)k3::MAX_GRID; }

px_status px3_init_field(px_patch3* p, int32_t kind, uint64_t seed, int32_t z0, void* stream) {
  clear_error();
  PX_TRY(check3(p, "field"));
  if (kind != 0 && kind != 1) return fail(PX_ERR_ARG, "kind must be 0 (zero) or 1 (hash)");
  if (z0 < 0) return fail(PX_ERR_ARG, "z0 must be >= 0");
  k3_init<<<1024, 256, 0, (cudaStream_t)stream>>>(p->data, p->ld, p->plane, p->n[0], p->n[1], p->n[2], kind, seed,
                                                  z0);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "3D init launch");
}

px_status px3_mehrstellen_rhs(const px_patch3* rho, px_patch3* f, void* stream) {
  clear_error();
  PX_TRY(check3(rho, "rho"));
  PX_TRY(check3(f, "f"));
  PX_TRY(same_shape3(*rho, *f, "f"));
  if (rho->ld != f->ld || rho->plane != f->plane) return fail(PX_ERR_SHAPE, "rho and f must share ld and plane");
  if (rho->data == f->data) return fail(PX_ERR_ARG, "rho and f must differ");
  k3_mrhs<<<2048, 256, 0, (cudaStream_t)stream>>>(rho->data, f->data, rho->ld, rho->plane, rho->n[0], rho->n[1],
                                                  rho->n[2], 1.0 / 12.0);
  count_launches(1);
  return cuda_check(cudaGetLastError(), "3D Mehrstellen rhs launch");
}

px_status px3_fill_ghosts(px_bc bc, px_patch3* p, void* stream) {
  clear_error();
  PX_TRY(check3(p, "phi"));
  if (bc != PX_BC_PERIODIC && bc != PX_BC_DIRICHLET_CC && bc != PX_BC_FIXED_GHOSTS)
    return fail(PX_ERR_ARG, "unknown boundary condition %d", (int)bc);
  return launch_ghost3(bc, *p, (cudaStream_t)stream);
}

px_status px3_relax_step(const px_relax_params* p, const px_patch3* phi_in, px_patch3* phi_out,
                         const px_patch3* rhs, double* d_norms, void* stream) {
  clear_error();
  PX_TRY(check_params3(p));
  PX_TRY(check3(phi_in, "phi_in"));
  PX_TRY(check3(phi_out, "phi_out"));
  PX_TRY(check3(rhs, "rhs"));
  PX_TRY(same_shape3(*phi_in, *phi_out, "phi_out"));
  PX_TRY(same_shape3(*phi_in, *rhs, "rhs"));
  if (phi_in->data == phi_out->data) return fail(PX_ERR_ARG, "phi_in and phi_out must not overlap");
  return launch_relax3(MODE_RELAX, *p, *phi_in, phi_out, *rhs, slot_from(d_norms, relax3_blocks(phi_in->n, p->stencil)),
                       (cudaStream_t)stream);
}

px_status px3_residual_norm(const px_relax_params* p, const px_patch3* phi, const px_patch3* rhs, double* d_norms,
                            void* stream) {
  clear_error();
  PX_TRY(check_params3(p));
  PX_TRY(check3(phi, "phi"));
  PX_TRY(check3(rhs, "rhs"));
  PX_TRY(same_shape3(*phi, *rhs, "rhs"));
  if (!d_norms) return fail(PX_ERR_ARG, "d_norms is required");
  return launch_relax3(MODE_RESID, *p, *phi, nullptr, *rhs, slot_from(d_norms, relax3_blocks(phi->n, p->stencil)),
                       (cudaStream_t)stream);
}

}  // extern "C"

namespace px {
static px_status solve3_impl(px_comm* comm, px_bc bc, const px_relax_params* p, const px_solve_opts* o,
                             px_patch3* phi, px_patch3* phi_scratch, const px_patch3* rhs, double* h_norms,
                             int32_t cap, int32_t* n_written, int32_t* in_scratch, void* stream) {
  PX_TRY(check_params3(p));
  if (!o) return fail(PX_ERR_ARG, "null options");
  if (o->nsweeps < 0) return fail(PX_ERR_ARG, "nsweeps must be >= 0");
  if (o->temporal_k > 1) return fail(PX_ERR_UNSUPPORTED, "3D temporal blocking not built");
  if (bc != PX_BC_PERIODIC && bc != PX_BC_DIRICHLET_CC && bc != PX_BC_FIXED_GHOSTS)
    return fail(PX_ERR_ARG, "unknown boundary condition %d", (int)bc);
  PX_TRY(check3(phi, "phi"));
  PX_TRY(check3(phi_scratch, "phi_scratch"));
  PX_TRY(check3(rhs, "rhs"));
  PX_TRY(same_shape3(*phi, *phi_scratch, "phi_scratch"));
  PX_TRY(same_shape3(*phi, *rhs, "rhs"));
  if (phi->data == phi_scratch->data) return fail(PX_ERR_ARG, "phi and phi_scratch must differ");
  cudaStream_t s = (cudaStream_t)stream;
  const int E = o->norm_every, N = o->nsweeps;
  const int n_entries = E < 0 ? 0 : (E > 0 ? (N + E - 1) / E : 0) + 1;
  if (n_entries > 0 && (!h_norms || cap < 1)) return fail(PX_ERR_ARG, "h_norms / cap required for norm entries");
  if (bc == PX_BC_FIXED_GHOSTS) {  // the caller's ghost ring belongs to every iterate
    PX_TRY(cuda_check(cudaMemcpyAsync(start3(*phi_scratch), start3(*phi), sizeof(double) * span3(*phi),
                                      cudaMemcpyDeviceToDevice, s),
                      "fixed ghost copy"));
  }
  if (!g_plan3 || !same_key(*g_plan3, comm, bc, *p, *o, *phi, *phi_scratch, *rhs, s)) {
    g_plan3.reset(new Plan3());
    Plan3& P = *g_plan3;
    P.comm = comm;
    P.bc = bc;
    P.prm = *p;
    P.opts = *o;
    P.a = *phi;
    P.b = *phi_scratch;
    P.r = *rhs;
    P.s = s;
    P.n_entries = n_entries;
    PX_TRY(cuda_check(cudaMalloc(&P.d_ring, sizeof(double) * 2 * (n_entries > 0 ? n_entries : 1)), "norm ring"));
    PX_TRY(cuda_check(cudaMalloc(&P.d_ws, sizeof(double) * (2 + 2 * k3::MAX_GRID)), "norm workspace"));
    PX_TRY(cuda_check(cudaMemset(P.d_ws, 0, sizeof(double) * (2 + 2 * k3::MAX_GRID)), "norm workspace"));
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fills before any user-stream work
    if (o->use_graph) {
      cudaGraph_t graph;
      const int64_t before = px_kernel_launch_count();
      PX_TRY(cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture"));
      px_status st = enqueue_solve3(P);
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      P.launches_per_run = px_kernel_launch_count() - before;
      count_launches(-P.launches_per_run);  // captured, not launched
      if (st != PX_OK) return st;
      PX_TRY(cuda_check(ce, "end capture"));
      ce = cudaGraphInstantiate(&P.exec, graph, 0);
      cudaGraphDestroy(graph);
      PX_TRY(cuda_check(ce, "graph instantiate"));
    }
  }
  Plan3& P = *g_plan3;
  if (P.exec) {
    PX_TRY(cuda_check(cudaGraphLaunch(P.exec, s), "graph launch"));
    count_launches(P.launches_per_run);
  } else {
    PX_TRY(enqueue_solve3(P));
  }
  std::vector<double> ring(2 * (size_t)(n_entries > 0 ? n_entries : 1));
  if (n_entries > 0)
    PX_TRY(cuda_check(cudaMemcpyAsync(ring.data(), P.d_ring, sizeof(double) * 2 * n_entries, cudaMemcpyDeviceToHost, s),
                      "norms D2H"));
  PX_TRY(cuda_check(cudaStreamSynchronize(s), "solve sync"));
  const int nw = n_entries < cap ? n_entries : cap;
  for (int j = 0; j < nw; ++j) {  // ring: max[n_entries] then sum[n_entries]
    h_norms[2 * j] = ring[j];
    h_norms[2 * j + 1] = ring[n_entries + j];
  }
  if (n_written) *n_written = nw;
  const bool odd = (N & 1) != 0;
  if (in_scratch) {
    *in_scratch = odd ? 1 : 0;
  } else if (odd) {
    PX_TRY(cuda_check(cudaMemcpyAsync(start3(*phi), start3(*phi_scratch), sizeof(double) * span3(*phi),
                                      cudaMemcpyDeviceToDevice, s),
                      "result copy"));
    PX_TRY(cuda_check(cudaStreamSynchronize(s), "solve sync"));
  }
  return PX_OK;
}

}  // namespace px

extern "C" {

px_status px3_solve(px_bc bc, const px_relax_params* p, const px_solve_opts* o, px_patch3* phi,
                    px_patch3* phi_scratch, const px_patch3* rhs, double* h_norms, int32_t cap,
                    int32_t* n_written, int32_t* in_scratch, void* stream) {
  clear_error();
  return solve3_impl(nullptr, bc, p, o, phi, phi_scratch, rhs, h_norms, cap, n_written, in_scratch, stream);
}

px_status px3_slab(int32_t n2, int32_t nranks, int32_t rank, int32_t* z0, int32_t* z1) {
  clear_error();
  if (!z0 || !z1) return fail(PX_ERR_ARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PX_ERR_ARG, "bad rank %d of %d", rank, nranks);
  if (n2 < nranks) return fail(PX_ERR_SHAPE, "n2 = %d planes for %d ranks", n2, nranks);
  *z0 = (int32_t)((int64_t)rank * n2 / nranks);
  *z1 = (int32_t)((int64_t)(rank + 1) * n2 / nranks);
  return PX_OK;
}

px_status px3_solve_comm(px_comm* c, px_bc bc, const px_relax_params* p, const px_solve_opts* o, px_patch3* phi,
                         px_patch3* phi_scratch, const px_patch3* rhs, double* h_norms, int32_t cap,
                         int32_t* n_written, int32_t* in_scratch, void* stream) {
  clear_error();
  if (!c) return fail(PX_ERR_ARG, "null communicator");
  if (!comm_nccl(c)) return fail(PX_ERR_UNSUPPORTED, "px3_solve_comm needs an NCCL communicator (px_comm_create)");
  return solve3_impl(c, bc, p, o, phi, phi_scratch, rhs, h_norms, cap, n_written, in_scratch, stream);
}

// ---------------------------------------------------------------- host batch
// Three device buffer sets, each with its own cached plan (and graph): problem
// i's H2D (s_in) and problem i-1's D2H (s_out) overlap problem i's solve.
namespace {
struct Batch3 {
  static constexpr int NSET = 3;
  int32_t n[3] = {0, 0, 0};
  int32_t ghost = 0;
  int64_t ld = 0, plane = 0, origin = 0, alloc = 0;
  double* d[NSET][3] = {};
  double* h_ring[NSET] = {};
  int ne = 0;
  std::unique_ptr<Plan3> plan[NSET];
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in[NSET] = {}, ev_done[NSET] = {}, ev_free[NSET] = {};
  void release_fields() {
    for (auto& pl : plan) pl.reset();
    for (auto& set : d)
      for (auto& q : set) {
        if (q) cudaFree(q);
        q = nullptr;
      }
    for (auto& h : h_ring) {
      if (h) cudaFreeHost(h);
      h = nullptr;
    }
    alloc = 0;
    ne = 0;
  }
  void release() {
    release_fields();
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    s_in = s_out = nullptr;
    auto destroy = [](cudaEvent_t& e) {
      if (e) cudaEventDestroy(e);
      e = nullptr;
    };
    destroy(ev_start);
    for (int b = 0; b < NSET; ++b) {
      destroy(ev_in[b]);
      destroy(ev_done[b]);
      destroy(ev_free[b]);
    }
  }
  px_patch3 patch(int b, int k) const {
    px_patch3 q;
    q.data = d[b][k] + origin;
    for (int i = 0; i < 3; ++i) q.n[i] = n[i];
    q.ghost = ghost;
    q.ld = ld;
    q.plane = plane;
    return q;
  }
};
Batch3 g_batch3;

// dense host (n2, n1, n0) <-> the owned cells of a padded device field
cudaMemcpy3DParms copy3(const Batch3& B, double* dev_origin, double* host, bool h2d) {
  cudaMemcpy3DParms c;
  std::memset(&c, 0, sizeof c);
  cudaPitchedPtr hp = make_cudaPitchedPtr(host, B.n[0] * sizeof(double), B.n[0] * sizeof(double), B.n[1]);
  cudaPitchedPtr dp = make_cudaPitchedPtr(dev_origin, B.ld * sizeof(double), B.n[0] * sizeof(double),
                                          B.n[1] + 2 * B.ghost);
  c.srcPtr = h2d ? hp : dp;
  c.dstPtr = h2d ? dp : hp;
  c.extent = make_cudaExtent(B.n[0] * sizeof(double), B.n[1], B.n[2]);
  c.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  return c;
}
}  // namespace

px_status px3_solve_host_batch(px_bc bc, const px_relax_params* p, const px_solve_opts* o, const int32_t n[3],
                               int32_t ghost, int32_t nprob, const double* const* h_phi0,
                               const double* const* h_rho, double* const* h_phi_out, double* h_norms, int32_t cap,
                               int32_t* n_written, void* stream) {
  clear_error();
  if (!p || !o || !n || !h_rho || !h_phi_out) return fail(PX_ERR_ARG, "null argument");
  PX_TRY(check_params3(p));
  if (nprob < 0) return fail(PX_ERR_ARG, "nprob must be >= 0");
  if (o->nsweeps < 0) return fail(PX_ERR_ARG, "nsweeps must be >= 0");
  if (o->temporal_k > 1) return fail(PX_ERR_UNSUPPORTED, "3D temporal blocking not built");
  if (bc != PX_BC_PERIODIC && bc != PX_BC_DIRICHLET_CC)
    return fail(PX_ERR_UNSUPPORTED, "px3_solve_host_batch takes PERIODIC or DIRICHLET_CC (host arrays carry no ghosts)");
  if (!stream) return fail(PX_ERR_ARG, "px3_solve_host_batch needs a non-default compute stream");
  const int E = o->norm_every, N = o->nsweeps;
  const int ne = E < 0 ? 0 : (E > 0 ? (N + E - 1) / E : 0) + 1;
  if (ne > 0 && (!h_norms || cap < 1)) return fail(PX_ERR_ARG, "h_norms / cap required for norm entries");
  for (int32_t i = 0; i < nprob; ++i)
    if (!h_rho[i] || !h_phi_out[i]) return fail(PX_ERR_ARG, "null host buffer for problem %d", i);
  int64_t ld, plane, origin, alloc;
  PX_TRY(px3_layout(n, ghost, &ld, &plane, &origin, &alloc));
  if (nprob == 0) return PX_OK;
  Batch3& B = g_batch3;
  cudaStream_t s = (cudaStream_t)stream;
  if (!B.s_in) {
    PX_TRY(cuda_check(cudaStreamCreateWithFlags(&B.s_in, cudaStreamNonBlocking), "stream"));
    PX_TRY(cuda_check(cudaStreamCreateWithFlags(&B.s_out, cudaStreamNonBlocking), "stream"));
    PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_start, cudaEventDisableTiming), "event"));
    for (int b = 0; b < Batch3::NSET; ++b) {
      PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_in[b], cudaEventDisableTiming), "event"));
      PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_done[b], cudaEventDisableTiming), "event"));
      PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_free[b], cudaEventDisableTiming), "event"));
    }
  }
  if (B.alloc != alloc || B.ld != ld || B.ghost != ghost || std::memcmp(B.n, n, sizeof B.n) != 0 || B.ne < ne) {
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "sync before realloc"));
    B.release_fields();
    for (auto& set : B.d)
      for (auto& q : set) {
        PX_TRY(cuda_check(cudaMalloc(&q, alloc * sizeof(double)), "cudaMalloc"));
        PX_TRY(cuda_check(cudaMemset(q, 0, alloc * sizeof(double)), "memset"));
      }
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fills before any user-stream work
    B.ne = ne > 0 ? ne : 1;
    for (auto& h : B.h_ring) PX_TRY(cuda_check(cudaMallocHost(&h, 2 * (size_t)B.ne * sizeof(double)), "cudaMallocHost"));
    std::memcpy(B.n, n, sizeof B.n);
    B.ghost = ghost;
    B.ld = ld;
    B.plane = plane;
    B.origin = origin;
    B.alloc = alloc;
  }
  // one plan (norm ring, workspace, graph) per buffer set
  for (int b = 0; b < Batch3::NSET; ++b) {
    const px_patch3 a = B.patch(b, 0), c = B.patch(b, 1), r = B.patch(b, 2);
    if (B.plan[b] && same_key(*B.plan[b], nullptr, bc, *p, *o, a, c, r, s)) continue;
    B.plan[b].reset(new Plan3());
    Plan3& P = *B.plan[b];
    P.bc = bc;
    P.prm = *p;
    P.opts = *o;
    P.a = a;
    P.b = c;
    P.r = r;
    P.s = s;
    P.n_entries = ne;
    PX_TRY(cuda_check(cudaMalloc(&P.d_ring, sizeof(double) * 2 * (ne > 0 ? ne : 1)), "norm ring"));
    PX_TRY(cuda_check(cudaMalloc(&P.d_ws, sizeof(double) * (2 + 2 * k3::MAX_GRID)), "norm workspace"));
    PX_TRY(cuda_check(cudaMemset(P.d_ws, 0, sizeof(double) * (2 + 2 * k3::MAX_GRID)), "norm workspace"));
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fills before any user-stream work
    if (o->use_graph) {
      cudaGraph_t graph;
      const int64_t before = px_kernel_launch_count();
      PX_TRY(cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture"));
      px_status st = enqueue_solve3(P);
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      P.launches_per_run = px_kernel_launch_count() - before;
      count_launches(-P.launches_per_run);
      if (st != PX_OK) return st;
      PX_TRY(cuda_check(ce, "end capture"));
      ce = cudaGraphInstantiate(&P.exec, graph, 0);
      cudaGraphDestroy(graph);
      PX_TRY(cuda_check(ce, "graph instantiate"));
    }
  }
  PX_TRY(cuda_check(cudaEventRecord(B.ev_start, s), "event"));
  PX_TRY(cuda_check(cudaStreamWaitEvent(B.s_in, B.ev_start, 0), "wait"));
  PX_TRY(cuda_check(cudaStreamWaitEvent(B.s_out, B.ev_start, 0), "wait"));
  bool pending[Batch3::NSET] = {};
  int32_t pend_i[Batch3::NSET] = {};
  auto harvest = [&](int b) -> px_status {
    if (!pending[b]) return PX_OK;
    PX_TRY(cuda_check(cudaEventSynchronize(B.ev_free[b]), "batch D2H"));
    const int32_t i = pend_i[b];
    const int32_t nw = ne < cap ? ne : cap;
    for (int32_t j = 0; j < nw; ++j) {  // ring: max[ne] then sum[ne]
      h_norms[(size_t)i * 2 * cap + 2 * j] = B.h_ring[b][j];
      h_norms[(size_t)i * 2 * cap + 2 * j + 1] = B.h_ring[b][ne + j];
    }
    if (n_written) n_written[i] = nw;
    pending[b] = false;
    return PX_OK;
  };
  const bool odd = (N & 1) != 0;
  for (int32_t i = 0; i < nprob; ++i) {
    const int b = i % Batch3::NSET;
    PX_TRY(harvest(b));  // problem i-NSET has left set b
    Plan3& P = *B.plan[b];
    // ---- copy in (s_in)
    if (h_phi0 && h_phi0[i]) {
      cudaMemcpy3DParms c = copy3(B, P.a.data, const_cast<double*>(h_phi0[i]), true);
      PX_TRY(cuda_check(cudaMemcpy3DAsync(&c, B.s_in), "H2D phi"));
    } else {
      PX_TRY(cuda_check(cudaMemsetAsync(B.d[b][0], 0, alloc * sizeof(double), B.s_in), "zero phi"));
    }
    cudaMemcpy3DParms cr = copy3(B, P.r.data, const_cast<double*>(h_rho[i]), true);
    PX_TRY(cuda_check(cudaMemcpy3DAsync(&cr, B.s_in), "H2D rho"));
    PX_TRY(cuda_check(cudaEventRecord(B.ev_in[b], B.s_in), "event"));
    // ---- solve (compute stream)
    PX_TRY(cuda_check(cudaStreamWaitEvent(s, B.ev_in[b], 0), "wait"));
    if (P.exec) {
      PX_TRY(cuda_check(cudaGraphLaunch(P.exec, s), "graph launch"));
      count_launches(P.launches_per_run);
    } else {
      PX_TRY(enqueue_solve3(P));
    }
    PX_TRY(cuda_check(cudaEventRecord(B.ev_done[b], s), "event"));
    // ---- copy out (s_out)
    PX_TRY(cuda_check(cudaStreamWaitEvent(B.s_out, B.ev_done[b], 0), "wait"));
    cudaMemcpy3DParms co = copy3(B, odd ? P.b.data : P.a.data, h_phi_out[i], false);
    PX_TRY(cuda_check(cudaMemcpy3DAsync(&co, B.s_out), "D2H phi"));
    if (ne > 0)
      PX_TRY(cuda_check(cudaMemcpyAsync(B.h_ring[b], P.d_ring, 2 * ne * sizeof(double), cudaMemcpyDeviceToHost,
                                        B.s_out), "D2H norms"));
    PX_TRY(cuda_check(cudaEventRecord(B.ev_free[b], B.s_out), "event"));
    pending[b] = true;
    pend_i[b] = i;
  }
  for (int b = 0; b < Batch3::NSET; ++b)
    if (pending[b]) PX_TRY(cuda_check(cudaStreamWaitEvent(s, B.ev_free[b], 0), "wait"));
  for (int b = 0; b < Batch3::NSET; ++b) PX_TRY(harvest(b));
  return cuda_check(cudaStreamSynchronize(s), "px3_solve_host_batch");
}

void px3_release(void) {
  g_plan3.reset();
  g_batch3.release();
}

}  // extern "C"

namespace px {
// drop the cached 3D plan of a communicator being destroyed (px_comm_destroy)
void release3_for_comm(const px_comm* c) {
  if (g_plan3 && g_plan3->comm == c) g_plan3.reset();
}
}  // namespace px

extern "C" {

}  // extern "C"
