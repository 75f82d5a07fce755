// px_cluster.cu -- a whole small single-box solve on a THREAD-BLOCK CLUSTER
// (BASELINE config 1: one 64x64 box, 100 sweeps).
//
// k_smallbox runs such a solve in one CTA: 4096 cells per sweep on one SM,
// latency-bound.  Here a cluster of CL = 8 CTAs (8 SMs) shares it: CTA c
// keeps rows [c·ny/CL, (c+1)·ny/CL) of φ (two copies) and of the right-hand
// side in its shared memory, plus one halo row above and below.  Per sweep
// every CTA updates its rows (the oracle's expression tree, every operation
// rounded -- bit-identical) with their x ghost columns, pushes its first and
// last new rows straight into its two neighbours' halo rows (distributed
// shared memory stores through mapped addresses) and release-arrives on
// their mbarriers (mbarrier.arrive.release.cluster on a mapa address); it
// then waits only for its own two neighbours -- no cluster-wide barrier per
// sweep.  Domain faces: periodic = the ring of CTAs; Dirichlet: odd
// reflection; fixed: kept.  No global-memory
// traffic inside the sweep loop.  Residual norms: per CTA in fixed order per
// recorded sweep, kept in shared memory; at the end CTA 0 reduces every entry
// over the CTAs in rank order through DSMEM.
//
// Buffer reuse: a neighbour pushes its sweep-s rows into our buffer (s+1)&1
// after it received our sweep-(s-1) push, i.e. after we finished reading
// that buffer in sweep s-1; the halo it fills is read in sweep s+1.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "px_device.cuh"
#include "px_internal.h"

namespace cg = cooperative_groups;

namespace px {

constexpr int CB_CL = 8;         // CTAs per cluster (portable maximum)
constexpr int CB_THREADS = 256;

template <int ST>
__device__ __forceinline__ double cb_taps(const double* p, int P, int i) {
  if (ST == 0)
    return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(p[i - 1], p[i + 1]), p[i - P]), p[i + P]), __dmul_rn(-4.0, p[i]));
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

// x ghost columns of padded row `row` (P = nx + 2) by the boundary rule
__device__ __forceinline__ void cb_xghost(double* row, int nx, int bc) {
  if (bc == PX_BC_PERIODIC) {
    row[0] = row[nx];
    row[nx + 1] = row[1];
  } else if (bc == PX_BC_DIRICHLET_CC) {
    row[0] = -row[1];
    row[nx + 1] = -row[nx];
  }
}

// release-arrive on the mbarrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mb_arrive_remote(uint64_t* bar, int rank) {
  uint32_t local = (uint32_t)__cvta_generic_to_shared(bar), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// wait (acquire at cluster scope) for the phase with parity `par` to complete
__device__ __forceinline__ void mb_wait_cluster(uint64_t* bar, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(par)
      : "memory");
}

template <int ST>
__global__ void __cluster_dims__(CB_CL, 1, 1) __launch_bounds__(CB_THREADS, 1) k_cluster_box(const SmallBox b,
                                                                                          int n_entries) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int c = (int)cluster.block_rank(), tid = threadIdx.x, nt = blockDim.x;
  const int nx = b.nx, ny = b.ny, P = nx + 2;
  const int y0 = c * ny / CB_CL, y1 = (c + 1) * ny / CB_CL, R = y1 - y0;
  const int rmax = (ny + CB_CL - 1) / CB_CL;
  double* bufs[2] = {sm, sm + (size_t)(rmax + 2) * P};
  double* F = sm + (size_t)2 * (rmax + 2) * P;
  constexpr int NWP = CB_THREADS / 32;
  // per-warp partials of every recorded entry: reduced (warps in order, then
  // CTAs in rank order) once at the end, off the sweep's critical path
  unsigned long long* pm = reinterpret_cast<unsigned long long*>(F + (size_t)rmax * nx);  // [entry][warp]
  double* ps = reinterpret_cast<double*>(pm + (size_t)n_entries * NWP);                 // [entry][warp]
  const int lane = tid & 31, wid = tid >> 5;
  auto warp_partial = [&](unsigned long long mx, double ss, int e) {
    for (int o = 16; o > 0; o >>= 1) {
      mx = umax64(mx, __shfl_xor_sync(FULL_MASK, mx, o));
      ss = ss + __shfl_xor_sync(FULL_MASK, ss, o);
    }
    if (lane == 0) {
      pm[(size_t)e * NWP + wid] = mx;
      ps[(size_t)e * NWP + wid] = ss;
    }
  };
  const int up = c > 0 ? c - 1 : CB_CL - 1, dn = c < CB_CL - 1 ? c + 1 : 0;
  const bool top_face = c == 0, bot_face = c == CB_CL - 1;

  // rows y0-1 .. y1 (with their x ghost columns) as given, into both copies
  for (int k = tid; k < (R + 2) * P; k += nt) {
    const int x = k % P - 1, r = k / P;
    const double v = b.phi_in[x + (int64_t)(y0 - 1 + r) * b.ld_in];
    bufs[0][k] = v;
    bufs[1][k] = v;
  }
  for (int k = tid; k < R * nx; k += nt) F[k] = b.rhs[(k % nx) + (int64_t)(y0 + k / nx) * b.ld_rhs];
  __syncthreads();

  // halo rows of buffer D from the neighbours' buffer D (or the face rule);
  // D's own rows and their x ghosts must be final in every CTA
  auto halo = [&](int d) {
    double* D = bufs[d];
    cluster.sync();  // every CTA's rows of D (and their x ghosts) are complete
    const double* Du = cluster.map_shared_rank(bufs[d], up);
    const double* Dd = cluster.map_shared_rank(bufs[d], dn);
    const int Ru = (up + 1) * ny / CB_CL - up * ny / CB_CL;  // rows of the upper neighbour
    for (int x = tid; x < P; x += nt) {
      if (!top_face || b.bc == PX_BC_PERIODIC) D[x] = Du[(size_t)Ru * P + x];
      else if (b.bc == PX_BC_DIRICHLET_CC) D[x] = -D[P + x];
      if (!bot_face || b.bc == PX_BC_PERIODIC) D[(size_t)(R + 1) * P + x] = Dd[P + x];
      else if (b.bc == PX_BC_DIRICHLET_CC) D[(size_t)(R + 1) * P + x] = -D[(size_t)R * P + x];
    }
    __syncthreads();
  };
  // neighbour-to-neighbour halo barrier: one arrival per pushing neighbour
  const bool has_up = !top_face || b.bc == PX_BC_PERIODIC, has_dn = !bot_face || b.bc == PX_BC_PERIODIC;
  const int nexp = (has_up ? 1 : 0) + (has_dn ? 1 : 0);
  // two barriers, alternating by sweep parity: a neighbour may run one sweep
  // ahead (it depends on us, not on our other neighbour), so its next
  // arrival must not count toward the phase we are still waiting for
  __shared__ __align__(8) uint64_t hbar[2];
  if (tid == 0 && nexp) {
    for (int k = 0; k < 2; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&hbar[k])),
                   "r"(nexp)
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the given ghost ring may be stale for periodic / Dirichlet: re-derive it
  for (int r = 1 + tid; r <= R; r += nt) cb_xghost(bufs[0] + (size_t)r * P, nx, b.bc);
  __syncthreads();
  halo(0);
  if (tid < 2) cb_xghost(bufs[0] + (size_t)(tid == 0 ? 0 : R + 1) * P, nx, b.bc);
  __syncthreads();

  const double scale = b.scale, lambda = b.lambda;
  const int ncell = R * nx;
  // thread -> cells k = tid, tid + nt, ... without a division per cell
  const int cx0 = tid % nx, cr0 = tid / nx, sx = nt % nx, sr = nt / nx;
  int cur = 0, entry = 0;
  for (int s = 0; s < b.nsweeps; ++s) {
    const double* A = bufs[cur];
    double* B = bufs[cur ^ 1];
    const bool rec = b.every > 0 && s % b.every == 0;
    unsigned long long mx = 0ull;
    double ss = 0.0;
    for (int k = tid, x = cx0, r = cr0; k < ncell; k += nt) {
      const int i = (x + 1) + (r + 1) * P;
      const double L = cb_taps<ST>(A, P, i);
      const double rr = __dsub_rn(__dmul_rn(scale, L), F[k]);
      const double o = __dadd_rn(A[i], __dmul_rn(lambda, rr));
      B[i] = o;
      // the row's x ghost images of this cell (wrap / odd reflection)
      if (x == 0) {
        if (b.bc == PX_BC_PERIODIC) B[i + nx] = o;
        else if (b.bc == PX_BC_DIRICHLET_CC) B[i - 1] = -o;
      }
      if (x == nx - 1) {
        if (b.bc == PX_BC_PERIODIC) B[i - nx] = o;
        else if (b.bc == PX_BC_DIRICHLET_CC) B[i + 1] = -o;
      }
      mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(rr)));
      ss = fma(rr, rr, ss);
      x += sx;
      r += sr;
      if (x >= nx) {
        x -= nx;
        ++r;
      }
    }
    __syncthreads();  // the CTA's new rows (and their x ghosts) are complete
    // halo rows, neighbour-to-neighbour: push the first / last new row (with
    // its ghost columns) straight into the neighbours' halo rows of the same
    // buffer (DSMEM stores), then release-arrive on their barriers; at a
    // Dirichlet face the halo row is the negated own row (corners by the
    // product rule); fixed faces keep theirs.  A neighbour is at least at
    // the end of its sweep s-1 compute (it pushed to us before we started
    // sweep s), so its copy of this buffer is no longer being read.
    {
      double* Bu = cluster.map_shared_rank(B, up);  // up's buffer: its last halo row R_up+1
      double* Bd = cluster.map_shared_rank(B, dn);  // dn's buffer: its halo row 0
      const int Ru = (up + 1) * ny / CB_CL - up * ny / CB_CL;
      for (int x = tid; x < P; x += nt) {
        if (has_up) Bu[(size_t)(Ru + 1) * P + x] = B[P + x];
        else if (b.bc == PX_BC_DIRICHLET_CC) B[x] = -B[P + x];
        if (has_dn) Bd[x] = B[(size_t)R * P + x];
        else if (b.bc == PX_BC_DIRICHLET_CC) B[(size_t)(R + 1) * P + x] = -B[(size_t)R * P + x];
      }
      __syncthreads();
      if (tid == 0) {
        if (has_up) mb_arrive_remote(&hbar[s & 1], up);
        if (has_dn) mb_arrive_remote(&hbar[s & 1], dn);
      }
      // the norm's warp reduction overlaps the neighbours' arrival latency
      if (rec) warp_partial(mx, ss, entry++);
      // both neighbours' rows of this sweep have arrived in our halo
      if (nexp) mb_wait_cluster(&hbar[s & 1], (uint32_t)((s >> 1) & 1));
    }
    cur ^= 1;
  }
  if (b.final_norm) {
    const double* A = bufs[cur];
    unsigned long long mx = 0ull;
    double ss = 0.0;
    for (int k = tid; k < ncell; k += nt) {
      const int x = k % nx, r = k / nx;
      const double rr = __dsub_rn(__dmul_rn(scale, cb_taps<ST>(A, P, (x + 1) + (r + 1) * P)), F[k]);
      mx = umax64(mx, (unsigned long long)__double_as_longlong(fabs(rr)));
      ss = fma(rr, rr, ss);
    }
    warp_partial(mx, ss, entry++);
  }
  cluster.sync();  // every CTA's partials are final
  if (c == 0) {
    for (int e = tid; e < entry; e += nt) {
      unsigned long long m = 0ull;
      double t = 0.0;
      for (int q = 0; q < CB_CL; ++q) {  // CTAs in rank order, warps in order
        const unsigned long long* qm = cluster.map_shared_rank(pm, q) + (size_t)e * NWP;
        const double* qs = cluster.map_shared_rank(ps, q) + (size_t)e * NWP;
        unsigned long long mq = qm[0];
        double tq = qs[0];
        for (int w = 1; w < NWP; ++w) {
          mq = umax64(mq, qm[w]);
          tq = tq + qs[w];
        }
        m = umax64(m, mq);
        t = t + tq;
      }
      b.d_max[e] = __longlong_as_double((long long)m);
      b.d_sum[e] = t;
    }
  }
  // φ^N: own rows with their ghost columns; the face CTAs also the ghost rows
  const double* A = bufs[cur];
  const int r0 = top_face ? 0 : 1, r1 = bot_face ? R + 1 : R;
  for (int k = tid; k < (r1 - r0 + 1) * P; k += nt) {
    const int x = k % P - 1, r = r0 + k / P;
    b.phi_out[x + (int64_t)(y0 - 1 + r) * b.ld_out] = A[(size_t)r * P + x + 1];
  }
  cluster.sync();  // no CTA leaves while CTA 0 may still read its partials
}

static int cluster_box_entries(const SmallBox& b) {
  const int n_entries = (b.every > 0 ? (b.nsweeps + b.every - 1) / b.every : 0) + (b.final_norm ? 1 : 0);
  return n_entries > 0 ? n_entries : 1;
}

// dynamic shared memory of k_cluster_box: two row buffers with halo rows, the
// CTA's rhs rows, and the per-warp norm partials of every recorded entry
static size_t cluster_box_smem(int nx, int ny, int ne) {
  const int rmax = (ny + CB_CL - 1) / CB_CL;
  return ((size_t)2 * (rmax + 2) * (nx + 2) + (size_t)rmax * nx) * sizeof(double) +
         (size_t)ne * (CB_THREADS / 32) * (sizeof(unsigned long long) + sizeof(double));
}

bool cluster_box_eligible(const SmallBox& b) {
  static int en = -1;
  if (en < 0) {
    const char* e = getenv("PROTOX_SMALLBOX_CLUSTER");
    en = (e && e[0] == '0') ? 0 : 1;
  }
  if (!en || b.nx < 1 || b.ny < 2 * CB_CL) return false;
  // the norm partials of every recorded entry live in shared memory too: a
  // long solve with many recorded norms falls back to k_smallbox (global ring)
  return cluster_box_smem(b.nx, b.ny, cluster_box_entries(b)) <= 200 * 1024;
}

px_status launch_cluster_box(const SmallBox& b, cudaStream_t s) {
  const int ne = cluster_box_entries(b);
  const size_t smem = cluster_box_smem(b.nx, b.ny, ne);
  if (smem > 200 * 1024) return fail(PX_ERR_UNSUPPORTED, "cluster box too large");
  cudaError_t e;
  if (b.stencil == 0) {
    static bool a0 = false;
    if (!a0) {
      cudaFuncSetAttribute(k_cluster_box<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      a0 = true;
    }
    k_cluster_box<0><<<CB_CL, CB_THREADS, smem, s>>>(b, ne);
  } else {
    static bool a1 = false;
    if (!a1) {
      cudaFuncSetAttribute(k_cluster_box<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      a1 = true;
    }
    k_cluster_box<1><<<CB_CL, CB_THREADS, smem, s>>>(b, ne);
  }
  note_kernel("k_cluster_box");
  e = cudaGetLastError();
  count_launches(1);
  return cuda_check(e, "cluster box kernel launch");
}

}  // namespace px
