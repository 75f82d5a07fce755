// px_mg.cu -- multigrid V-cycle with the fused relax sweep as its smoother
// ("Jacobi as the smoother of a geometric
// multigrid V-cycle"; the paper names multigrid as a Proto use of stencils,
// PAPER.md:25, and as ProtoX future work).  The V-cycle is
// defined by DESIGN.md readings R-MG1..R-MG6 and written out plainly in the
// oracle (oracle/protox_oracle.cpp, orc_mg_solve); this file computes the
// same numbers (bit-identical) on the GPU:
//
//   level 0 = the caller's patch (single rank), level l >= 1 = library-owned
//   (n0 >> l) x (n1 >> l) patches with one ghost layer, h_l = 2^l h,
//   λ_l = 4^l λ, the same stencil and (homogeneous) boundary rule;
//   smoothing sweeps = the hot-path relax kernels (k_bulk / k_stream with
//   fused ghost images), the coarsest level = the single-CTA k_smallbox
//   solve when it fits;
//   k_mg_restrict: the defect d = scale·S(φ) − f at the four children and
//   f_c = −0.25·(((d00 + d10) + d01) + d11), φ_c = 0, in one pass;
//   k_mg_prolong: φ += (((9·e_P + 3·e_X) + 3·e_Y) + e_D)·(1/16), in place.
//
// The whole sequence of all cycles is captured once into a CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "px_device.cuh"
#include "px_internal.h"

namespace px {

template <int ST>
__device__ __forceinline__ double mg_taps(const double* p, int64_t ld) {
  if (ST == 0)
    return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(p[-1], p[1]), p[-ld]), p[ld]), __dmul_rn(-4.0, p[0]));
  double q = __dmul_rn(4.0, p[-1]);
  q = __dadd_rn(q, __dmul_rn(4.0, p[1]));
  q = __dadd_rn(q, __dmul_rn(4.0, p[-ld]));
  q = __dadd_rn(q, __dmul_rn(4.0, p[ld]));
  q = __dadd_rn(q, p[-ld - 1]);
  q = __dadd_rn(q, p[-ld + 1]);
  q = __dadd_rn(q, p[ld - 1]);
  q = __dadd_rn(q, p[ld + 1]);
  return __dadd_rn(q, __dmul_rn(-20.0, p[0]));
}

// One thread per coarse cell: defect at its four children, minus their
// average into the coarse right-hand side, zero into the coarse iterate.
template <int ST>
__global__ void k_mg_restrict(const double* __restrict__ phi, int64_t ldp, const double* __restrict__ f,
                              int64_t ldf, double* __restrict__ fc, int64_t ldfc, double* __restrict__ phic,
                              int64_t ldpc, int ncx, int ncy, double scale) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y;
  if (I >= ncx) return;
  double d[2][2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int x = 2 * I + a, y = 2 * J + b;
      const double L = mg_taps<ST>(phi + x + (int64_t)y * ldp, ldp);
      d[b][a] = __dsub_rn(__dmul_rn(scale, L), f[x + (int64_t)y * ldf]);
    }
  double t = __dadd_rn(d[0][0], d[0][1]);
  t = __dadd_rn(t, d[1][0]);
  t = __dadd_rn(t, d[1][1]);
  fc[I + (int64_t)J * ldfc] = __dmul_rn(-0.25, t);
  phic[I + (int64_t)J * ldpc] = 0.0;
}

// One thread per fine cell: φ += P e (cell-centred bilinear; coarse ghosts valid).
__global__ void k_mg_prolong(const double* __restrict__ e, int64_t lde, double* __restrict__ phi, int64_t ldp,
                             int nx) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= nx) return;
  const int I = x >> 1, J = y >> 1;
  const int xn = (x & 1) ? I + 1 : I - 1, yn = (y & 1) ? J + 1 : J - 1;
  double t = __dmul_rn(9.0, e[I + (int64_t)J * lde]);
  t = __dadd_rn(t, __dmul_rn(3.0, e[xn + (int64_t)J * lde]));
  t = __dadd_rn(t, __dmul_rn(3.0, e[I + (int64_t)yn * lde]));
  t = __dadd_rn(t, e[xn + (int64_t)yn * lde]);
  double* p = phi + x + (int64_t)y * ldp;
  *p = __dadd_rn(*p, __dmul_rn(0.0625, t));
}

namespace {

struct MgLevel {
  int nx = 0, ny = 0;
  double scale = 0.0, lambda = 0.0;
  px_patch buf[2];   // iterate / scratch (swapped by the sweeps)
  px_patch f;
  int cur = 0;       // which of buf holds the current iterate
  double* alloc[3] = {nullptr, nullptr, nullptr};
  px_box owned() const { return mkbox(0, 0, nx - 1, ny - 1); }
};

struct MgKey {
  uint64_t gen;
  int32_t stencil;
  double h, lambda;
  px_mg_opts o;
  const double *phi, *scr, *rhs;
  px_box rbox;       // rhs patch geometry (offsets baked into the captured launches)
  int64_t rld;
  cudaStream_t s;
  bool operator==(const MgKey& k) const {
    return gen == k.gen && stencil == k.stencil && h == k.h && lambda == k.lambda &&
           std::memcmp(&o, &k.o, sizeof o) == 0 && phi == k.phi && scr == k.scr && rhs == k.rhs &&
           std::memcmp(&rbox, &k.rbox, sizeof rbox) == 0 && rld == k.rld && s == k.s;
  }
};

struct MgPlan {
  MgKey key;
  std::vector<MgLevel> lv;
  int mx = GH_NONE, my = GH_NONE;  // boundary rule of every level
  int bc = 0;
  double* d_max = nullptr;
  double* d_sum = nullptr;
  double* d_ws = nullptr;
  int n_entries = 0;
  int final_cur = 0;
  cudaGraphExec_t exec = nullptr;
  int64_t launches_per_run = 0;
  ~MgPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    for (size_t l = 1; l < lv.size(); ++l)
      for (double* a : lv[l].alloc)
        if (a) cudaFree(a);
    if (d_max) cudaFree(d_max);
    if (d_sum) cudaFree(d_sum);
    if (d_ws) cudaFree(d_ws);
  }
};

std::vector<std::unique_ptr<MgPlan>>& mg_plans() {
  static std::vector<std::unique_ptr<MgPlan>> v;
  return v;
}

GhostSpec level_ghosts(const MgPlan& P, const MgLevel& L) {
  GhostSpec g;
  g.mode[0][0] = g.mode[0][1] = P.mx;
  g.mode[1][0] = g.mode[1][1] = P.my;
  g.n[0] = L.nx;
  g.n[1] = L.ny;
  g.o[0] = g.o[1] = 0;
  g.g = 1;
  return g;
}

px_status fill_level_ghosts(const MgPlan& P, MgLevel& L, const px_patch& q, int g, cudaStream_t s) {
  return launch_fill_ghosts_raw(at(q, 0, 0), q.ld, L.nx, L.ny, g, P.mx, P.my, P.my, s);
}

// ν relax sweeps on level L (the current iterate alternates between buffers)
px_status mg_relax(const MgPlan& P, MgLevel& L, int stencil, int nu, cudaStream_t s) {
  if (nu <= 0) return PX_OK;
  const bool small = (int64_t)L.nx * L.ny <= 16384 && smallbox_fits(L.nx, L.ny) && &L != &P.lv[0];
  if (small) {
    // the whole ν sweeps in one CTA, in place (ghost ring refilled per sweep)
    SmallBox b;
    std::memset(&b, 0, sizeof b);
    b.phi_in = at(L.buf[L.cur], 0, 0);
    b.phi_out = at(L.buf[L.cur], 0, 0);
    b.rhs = at(L.f, 0, 0);
    b.ld_in = b.ld_out = L.buf[L.cur].ld;
    b.ld_rhs = L.f.ld;
    b.nx = L.nx;
    b.ny = L.ny;
    b.g = 1;
    b.bc = P.bc;
    b.stencil = stencil;
    b.scale = L.scale;
    b.lambda = L.lambda;
    b.nsweeps = nu;
    b.every = -1;
    b.final_norm = 0;
    return launch_smallbox(b, s);
  }
  for (int k = 0; k < nu; ++k) {
    StreamLaunch a;
    px_patch dst = L.buf[L.cur ^ 1];
    PX_TRY(make_stream_launch(MODE_RELAX, stencil, L.scale, L.lambda, &L.buf[L.cur], &L.f, &dst, L.owned(), &a));
    a.gs = level_ghosts(P, L);
    PX_TRY(launch_stream(MODE_RELAX, stencil, a, s));
    L.cur ^= 1;
  }
  return PX_OK;
}

px_status mg_restrict(MgPlan& P, int l, int stencil, cudaStream_t s) {
  MgLevel& F = P.lv[l];
  MgLevel& C = P.lv[l + 1];
  const px_patch& pf = F.buf[F.cur];
  const px_patch& pc = C.buf[C.cur];
  dim3 grid((C.nx + 127) / 128, C.ny);
  if (stencil)
    k_mg_restrict<1><<<grid, 128, 0, s>>>(at(pf, 0, 0), pf.ld, at(F.f, 0, 0), F.f.ld, at(C.f, 0, 0), C.f.ld,
                                          at(pc, 0, 0), pc.ld, C.nx, C.ny, F.scale);
  else
    k_mg_restrict<0><<<grid, 128, 0, s>>>(at(pf, 0, 0), pf.ld, at(F.f, 0, 0), F.f.ld, at(C.f, 0, 0), C.f.ld,
                                          at(pc, 0, 0), pc.ld, C.nx, C.ny, F.scale);
  count_launches(1);
  PX_TRY(cuda_check(cudaGetLastError(), "restriction kernel launch"));
  return fill_level_ghosts(P, C, pc, 1, s);
}

px_status mg_prolong(MgPlan& P, int l, cudaStream_t s) {
  MgLevel& F = P.lv[l];
  MgLevel& C = P.lv[l + 1];
  const px_patch& pf = F.buf[F.cur];
  const px_patch& pc = C.buf[C.cur];
  dim3 grid((F.nx + 127) / 128, F.ny);
  k_mg_prolong<<<grid, 128, 0, s>>>(at(pc, 0, 0), pc.ld, at(pf, 0, 0), pf.ld, F.nx);
  count_launches(1);
  PX_TRY(cuda_check(cudaGetLastError(), "prolongation kernel launch"));
  return fill_level_ghosts(P, F, pf, 1, s);
}

px_status vcycle(MgPlan& P, int l, int stencil, const px_mg_opts& o, cudaStream_t s) {
  MgLevel& L = P.lv[l];
  if (l + 1 == (int)P.lv.size()) return mg_relax(P, L, stencil, o.nu_coarse, s);
  PX_TRY(mg_relax(P, L, stencil, o.nu1, s));
  PX_TRY(mg_restrict(P, l, stencil, s));
  PX_TRY(vcycle(P, l + 1, stencil, o, s));
  PX_TRY(mg_prolong(P, l, s));
  return mg_relax(P, L, stencil, o.nu2, s);
}

px_status mg_residual(MgPlan& P, int stencil, int entry, cudaStream_t s) {
  MgLevel& L = P.lv[0];
  StreamLaunch a;
  PX_TRY(make_stream_launch(MODE_RESID, stencil, L.scale, 0.0, &L.buf[L.cur], &L.f, nullptr, L.owned(), &a));
  a.norms.out_max = P.d_max + entry;
  a.norms.out_sum = P.d_sum + entry;
  a.norms.counter = reinterpret_cast<unsigned int*>(P.d_ws);
  a.norms.partials = P.d_ws + 2;
  a.norms.offset = 0;
  a.norms.expected = launch_blocks(MODE_RESID, a);
  return launch_stream(MODE_RESID, stencil, a, s);
}

// the whole solve: ghosts of φ^0, norms of φ^0, ncycles V-cycles with norms
px_status mg_enqueue(MgPlan& P, int stencil, const px_mg_opts& o, int ghost, cudaStream_t s) {
  for (MgLevel& L : P.lv) L.cur = 0;
  MgLevel& L0 = P.lv[0];
  PX_TRY(fill_level_ghosts(P, L0, L0.buf[0], ghost, s));
  PX_TRY(mg_residual(P, stencil, 0, s));
  for (int c = 0; c < o.ncycles; ++c) {
    PX_TRY(vcycle(P, 0, stencil, o, s));
    PX_TRY(mg_residual(P, stencil, c + 1, s));
  }
  if (L0.cur == 1) {
    // φ ends in the scratch buffer: copy its interior into phi
    const px_patch& a = L0.buf[1];
    const px_patch& b = L0.buf[0];
    PX_TRY(cuda_check(cudaMemcpy2DAsync(at(b, 0, 0), b.ld * sizeof(double), at(a, 0, 0), a.ld * sizeof(double),
                                        L0.nx * sizeof(double), L0.ny, cudaMemcpyDeviceToDevice, s),
                      "copy result"));
  }
  // the sweeps keep one ghost layer current; the result gets the full ring
  PX_TRY(fill_level_ghosts(P, L0, L0.buf[0], ghost, s));
  P.final_cur = L0.cur;
  return PX_OK;
}

}  // namespace

void mg_drop_layout_plans(uint64_t gen) {
  auto& v = mg_plans();
  auto dead = [gen](const std::unique_ptr<MgPlan>& p) { return p->key.gen == gen; };
  if (std::any_of(v.begin(), v.end(), dead)) {
    cudaDeviceSynchronize();
    v.erase(std::remove_if(v.begin(), v.end(), dead), v.end());
  }
}
}  // namespace px

using namespace px;

extern "C" {

px_status px_mg_solve(const px_layout* l, const px_relax_params* p, const px_mg_opts* o, px_patch* phi,
                      px_patch* phi_scratch, const px_patch* rhs, double* h_norms, int32_t cap,
                      int32_t* n_written, void* stream) {
  if (!l || !p || !o || !phi || !phi_scratch || !rhs) return fail(PX_ERR_ARG, "null argument");
  if (l->nranks != 1) return fail(PX_ERR_UNSUPPORTED, "px_mg_solve needs a single-rank layout");
  if (l->bc == PX_BC_FIXED_GHOSTS)
    return fail(PX_ERR_UNSUPPORTED, "multigrid needs PERIODIC or DIRICHLET_CC boundaries");
  if (p->stencil != PX_LAPLACE_5PT && p->stencil != PX_MEHRSTELLEN_9PT) return fail(PX_ERR_ARG, "bad stencil");
  if (!(p->h > 0.0)) return fail(PX_ERR_ARG, "h must be positive");
  if (o->levels < 1 || o->levels > 30 || o->nu1 < 0 || o->nu2 < 0 || o->nu_coarse < 0 || o->ncycles < 0)
    return fail(PX_ERR_ARG, "bad multigrid options");
  if (cap < 0 || (cap > 0 && !h_norms)) return fail(PX_ERR_ARG, "bad norm output");
  px_local_info li;
  PX_TRY(local_info(l, 0, &li));
  const int n0 = ext(li.owned, 0), n1 = ext(li.owned, 1);
  const int div = 1 << (o->levels - 1);
  if (n0 % div || n1 % div)
    return fail(PX_ERR_SHAPE, "domain %dx%d not divisible by 2^(levels-1) = %d", n0, n1, div);
  const px_patch* in[3] = {phi, phi_scratch, rhs};
  for (const px_patch* q : in) {
    PX_TRY(check_patch(q, "patch"));
    if (!contains(q->box, li.alloc)) return fail(PX_ERR_SHAPE, "patch does not cover the ghosted domain");
  }
  if (((uintptr_t)phi->data / 8) % 2 != ((uintptr_t)phi_scratch->data / 8) % 2)
    return fail(PX_ERR_ALIGN, "phi and phi_scratch have different 16-byte phases");
  cudaStream_t s = (cudaStream_t)stream;
  if (o->use_graph && !s) return fail(PX_ERR_ARG, "use_graph needs a non-default stream");

  MgKey key{layout_generation(l), p->stencil, p->h, p->lambda, *o, phi->data, phi_scratch->data, rhs->data,
            rhs->box, rhs->ld, s};
  MgPlan* P = nullptr;
  for (auto& q : mg_plans())
    if (q->key == key) P = q.get();
  if (!P) {
    std::unique_ptr<MgPlan> np(new MgPlan());
    np->key = key;
    np->bc = l->bc;
    np->mx = np->my = l->bc == PX_BC_PERIODIC ? GH_WRAP : GH_REFLECT;
    np->lv.resize(o->levels);
    for (int k = 0; k < o->levels; ++k) {
      MgLevel& L = np->lv[k];
      L.nx = n0 >> k;
      L.ny = n1 >> k;
      const double hk = p->h * (double)(1 << k);
      L.scale = stencil_scale(p->stencil, hk);
      L.lambda = p->lambda * (double)(1 << k) * (double)(1 << k);
      if (k == 0) {
        // caller's patches, re-based so that cell (0,0) is the domain origin
        L.buf[0] = *phi;
        L.buf[1] = *phi_scratch;
        L.f = *rhs;
        px_patch* mine[3] = {&L.buf[0], &L.buf[1], &L.f};
        for (px_patch* q : mine)
          q->box = mkbox(q->box.lo.c[0] - li.owned.lo.c[0], q->box.lo.c[1] - li.owned.lo.c[1],
                         q->box.hi.c[0] - li.owned.lo.c[0], q->box.hi.c[1] - li.owned.lo.c[1]);
      } else {
        // interior column 0 at a 128-byte boundary, one ghost layer
        const int64_t ld = ((int64_t)L.nx + 32 + 15) / 16 * 16;
        const size_t bytes = (size_t)ld * (L.ny + 2) * sizeof(double);
        for (int b = 0; b < 3; ++b) {
          PX_TRY(cuda_check(cudaMalloc(&L.alloc[b], bytes), "cudaMalloc level"));
          PX_TRY(cuda_check(cudaMemset(L.alloc[b], 0, bytes), "memset level"));
        }
        for (int b = 0; b < 3; ++b) {
          px_patch q;
          q.data = L.alloc[b] + 15;  // cell (-1,-1); cell (0,0) at alloc + 16 + ld
          q.box = mkbox(-1, -1, L.nx, L.ny);
          q.ld = ld;
          (b < 2 ? L.buf[b] : L.f) = q;
        }
      }
    }
    np->n_entries = o->ncycles + 1;
    PX_TRY(cuda_check(cudaMalloc(&np->d_max, np->n_entries * sizeof(double)), "cudaMalloc ring"));
    PX_TRY(cuda_check(cudaMalloc(&np->d_sum, np->n_entries * sizeof(double)), "cudaMalloc ring"));
    const int64_t wsl = std::max<int64_t>(4 + 2 * (int64_t)stream_blocks(n0, n1, 1), 8192);
    PX_TRY(cuda_check(cudaMalloc(&np->d_ws, wsl * sizeof(double)), "cudaMalloc ws"));
    PX_TRY(cuda_check(cudaMemset(np->d_ws, 0, wsl * sizeof(double)), "memset ws"));
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fills before any user-stream work
    P = np.get();
    mg_plans().push_back(std::move(np));
  }
  plan_touch(mg_plans(), P);
  if (o->use_graph) {
    if (!P->exec) {
      const int64_t before = px_kernel_launch_count();
      PX_TRY(cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture"));
      px_status st = mg_enqueue(*P, p->stencil, *o, l->ghost, s);
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      if (st != PX_OK) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return st;
      }
      PX_TRY(cuda_check(ce, "end capture"));
      P->launches_per_run = px_kernel_launch_count() - before;
      count_launches(-P->launches_per_run);
      ce = cudaGraphInstantiate(&P->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) {
        P->exec = nullptr;
        cudaGetLastError();
      }
      PX_TRY(cuda_check(ce, "graph instantiate"));
    }
    PX_TRY(cuda_check(cudaGraphLaunch(P->exec, s), "graph launch"));
    count_launches(P->launches_per_run);
  } else {
    PX_TRY(mg_enqueue(*P, p->stencil, *o, l->ghost, s));
  }
  std::vector<double> hm(P->n_entries), hs(P->n_entries);
  PX_TRY(cuda_check(cudaMemcpyAsync(hm.data(), P->d_max, P->n_entries * sizeof(double), cudaMemcpyDeviceToHost, s),
                    "D2H norms"));
  PX_TRY(cuda_check(cudaMemcpyAsync(hs.data(), P->d_sum, P->n_entries * sizeof(double), cudaMemcpyDeviceToHost, s),
                    "D2H norms"));
  PX_TRY(cuda_check(cudaStreamSynchronize(s), "mg solve"));
  const int32_t nw = std::min<int32_t>(P->n_entries, cap);
  for (int32_t j = 0; j < nw; ++j) {
    h_norms[2 * j] = hm[j];
    h_norms[2 * j + 1] = hs[j];
  }
  if (n_written) *n_written = nw;
  return PX_OK;
}

void px_mg_release(void) { mg_plans().clear(); }

}  // extern "C"
