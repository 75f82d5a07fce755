// px_host.cpp -- status/errors, geometry (Point/Box), the box
// layout / slab partitioner (Proto's box decomposition)
// and the validated single-patch entry points of libprotox.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "px_internal.h"

namespace px {

static thread_local std::string g_last_error;

px_status fail(px_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

void clear_error() { g_last_error.clear(); }

px_status check_patch(const px_patch* p, const char* name) {
  if (!p) return fail(PX_ERR_ARG, "%s: null patch", name);
  if (!p->data) return fail(PX_ERR_ARG, "%s: null data pointer", name);
  if (empty(p->box)) return fail(PX_ERR_SHAPE, "%s: empty patch box", name);
  if (p->ld < ext(p->box, 0))
    return fail(PX_ERR_SHAPE, "%s: ld %lld < box width %d", name, (long long)p->ld, ext(p->box, 0));
  if (((uintptr_t)p->data) % 8)
    return fail(PX_ERR_ALIGN, "%s: data pointer not 8-byte aligned", name);
  if (p->ld % 2) return fail(PX_ERR_ALIGN, "%s: ld %lld is odd (rows must keep 16-byte phase)",
                             name, (long long)p->ld);
  return PX_OK;
}

static int64_t roundup(int64_t a, int64_t m) { return (a + m - 1) / m * m; }

px_status local_info(const px_layout* l, int32_t rank, px_local_info* out) {
  if (!l) return fail(PX_ERR_ARG, "null layout");
  if (!out) return fail(PX_ERR_ARG, "null output");
  if (rank < 0 || rank >= l->nranks)
    return fail(PX_ERR_ARG, "rank %d out of range [0,%d)", rank, l->nranks);
  const int32_t by0 = l->row_lo[rank], by1 = l->row_lo[rank + 1];
  px_box owned = mkbox(l->domain.lo.c[0], l->domain.lo.c[1] + by0 * l->box_size.c[1],
                       l->domain.hi.c[0], l->domain.lo.c[1] + by1 * l->box_size.c[1] - 1);
  out->owned = owned;
  out->alloc = grow(owned, l->ghost);
  out->ld = l->ld;
  out->patch_offset = 16 - l->ghost;
  out->alloc_elems = l->ld * (int64_t)ext(out->alloc, 1);
  const bool periodic = l->bc == PX_BC_PERIODIC;
  out->nbr_lo = rank > 0 ? rank - 1 : (periodic ? l->nranks - 1 : -1);
  out->nbr_hi = rank < l->nranks - 1 ? rank + 1 : (periodic ? 0 : -1);
  return PX_OK;
}

}  // namespace px

using namespace px;

extern "C" {

const char* px_status_str(px_status s) {
  switch (s) {
    case PX_OK: return "PX_OK";
    case PX_ERR_ARG: return "PX_ERR_ARG";
    case PX_ERR_SHAPE: return "PX_ERR_SHAPE";
    case PX_ERR_DOMAIN: return "PX_ERR_DOMAIN";
    case PX_ERR_ALIGN: return "PX_ERR_ALIGN";
    case PX_ERR_UNSUPPORTED: return "PX_ERR_UNSUPPORTED";
    case PX_ERR_CUDA: return "PX_ERR_CUDA";
    case PX_ERR_NCCL: return "PX_ERR_NCCL";
    case PX_ERR_STATE: return "PX_ERR_STATE";
  }
  return "PX_UNKNOWN_STATUS";
}

const char* px_last_error(void) { return g_last_error.c_str(); }
int32_t px_api_version(void) { return PX_API_VERSION; }

// ------------------------------------------------------------- geometry
int64_t px_box_size(px_box b) { return empty(b) ? 0 : (int64_t)ext(b, 0) * ext(b, 1); }
int32_t px_box_is_empty(px_box b) { return empty(b) ? 1 : 0; }
px_box px_box_grow(px_box b, int32_t r) { return grow(b, r); }
px_box px_box_intersect(px_box a, px_box b) {
  return mkbox(std::max(a.lo.c[0], b.lo.c[0]), std::max(a.lo.c[1], b.lo.c[1]),
               std::min(a.hi.c[0], b.hi.c[0]), std::min(a.hi.c[1], b.hi.c[1]));
}
px_status px_box_ordinal(px_box b, px_point p, int64_t* out) {
  if (!out) return fail(PX_ERR_ARG, "null output");
  if (empty(b) || p.c[0] < b.lo.c[0] || p.c[0] > b.hi.c[0] || p.c[1] < b.lo.c[1] ||
      p.c[1] > b.hi.c[1])
    return fail(PX_ERR_DOMAIN, "point (%d,%d) outside box [(%d,%d),(%d,%d)]", p.c[0], p.c[1],
                b.lo.c[0], b.lo.c[1], b.hi.c[0], b.hi.c[1]);
  *out = (int64_t)(p.c[0] - b.lo.c[0]) + (int64_t)(p.c[1] - b.lo.c[1]) * ext(b, 0);
  return PX_OK;
}

// --------------------------------------------------------------- layout
px_status px_layout_create(px_box domain, px_point box_size, int32_t ghost, px_bc bc,
                           int32_t nranks, px_partition part, px_layout** out) {
  if (!out) return fail(PX_ERR_ARG, "null output");
  *out = nullptr;
  if (empty(domain)) return fail(PX_ERR_SHAPE, "empty domain");
  if (box_size.c[0] < 1 || box_size.c[1] < 1)
    return fail(PX_ERR_ARG, "box size must be positive");
  const int32_t n0 = ext(domain, 0), n1 = ext(domain, 1);
  if (n0 % box_size.c[0] || n1 % box_size.c[1])
    return fail(PX_ERR_SHAPE, "box size (%d,%d) does not divide the domain (%d,%d)",
                box_size.c[0], box_size.c[1], n0, n1);
  if (ghost < 1 || ghost > 16) return fail(PX_ERR_ARG, "ghost width %d not in [1,16]", ghost);
  if (ghost > box_size.c[0] || ghost > box_size.c[1])
    return fail(PX_ERR_SHAPE, "ghost width %d exceeds the box size", ghost);
  if (bc != PX_BC_PERIODIC && bc != PX_BC_DIRICHLET_CC && bc != PX_BC_FIXED_GHOSTS)
    return fail(PX_ERR_ARG, "bad boundary condition %d", (int)bc);
  if (part != PX_PART_SLABS) return fail(PX_ERR_UNSUPPORTED, "only slab partitions are built");
  const int32_t nby = n1 / box_size.c[1];
  if (nranks < 1 || nranks > nby)
    return fail(PX_ERR_ARG, "nranks %d not in [1, %d box-rows]", nranks, nby);
  if ((int64_t)n0 + 2 * ghost + 16 > INT32_MAX / 2) return fail(PX_ERR_SHAPE, "domain too wide");
  px_layout* l = new (std::nothrow) px_layout();
  if (!l) return fail(PX_ERR_ARG, "out of host memory");
  l->domain = domain;
  l->box_size = box_size;
  l->ghost = ghost;
  l->bc = bc;
  l->nranks = nranks;
  l->nbx = n0 / box_size.c[0];
  l->nby = nby;
  l->row_lo.resize(nranks + 1);
  // contiguous blocks of box-rows, sizes differing by at most one
  for (int32_t r = 0; r <= nranks; ++r) l->row_lo[r] = (int32_t)((int64_t)nby * r / nranks);
  // 16 columns of padding on both sides: interior column 0 at element 16
  // (128-byte aligned rows), and every column in [-16, n0+16) addressable.
  l->ld = roundup((int64_t)n0 + 32, 16);
  static uint64_t next_gen = 1;
  l->gen = next_gen++;
  *out = l;
  return PX_OK;
}

void px_layout_destroy(px_layout* l) {
  if (!l) return;
  px::drop_layout_plans(l->gen);  // cached solve plans built for this layout
  delete l;
}

px_status px_layout_num_boxes(const px_layout* l, int32_t* n) {
  if (!l || !n) return fail(PX_ERR_ARG, "null argument");
  *n = l->nbx * l->nby;
  return PX_OK;
}

px_status px_layout_box(const px_layout* l, int32_t ibox, px_box* box, int32_t* owner) {
  if (!l || !box) return fail(PX_ERR_ARG, "null argument");
  if (ibox < 0 || ibox >= l->nbx * l->nby)
    return fail(PX_ERR_ARG, "box index %d out of range", ibox);
  const int32_t bx = ibox % l->nbx, by = ibox / l->nbx;
  *box = mkbox(l->domain.lo.c[0] + bx * l->box_size.c[0], l->domain.lo.c[1] + by * l->box_size.c[1],
               l->domain.lo.c[0] + (bx + 1) * l->box_size.c[0] - 1,
               l->domain.lo.c[1] + (by + 1) * l->box_size.c[1] - 1);
  if (owner) {
    int32_t r = 0;
    while (r + 1 < l->nranks && by >= l->row_lo[r + 1]) ++r;
    *owner = r;
  }
  return PX_OK;
}

px_status px_layout_local(const px_layout* l, int32_t rank, px_local_info* out) {
  return local_info(l, rank, out);
}

px_status px_layout_patch(const px_layout* l, int32_t rank, double* alloc_base, px_patch* out) {
  if (!out || !alloc_base) return fail(PX_ERR_ARG, "null argument");
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  out->data = alloc_base + li.patch_offset;
  out->box = li.alloc;
  out->ld = li.ld;
  return PX_OK;
}

px_status px_layout_halo_plan(const px_layout* l, int32_t rank, px_halo_op ops[4], int32_t* nops) {
  return halo_plan(l, rank, ops, nops, false);
}

}  // extern "C"

namespace px {
// allow_self: a one-rank periodic layout exchanges with itself (used by the
// NCCL self-exchange test mode, px_comm_create with PROTOX_NCCL_SELF_EXCHANGE=1)
px_status halo_plan(const px_layout* l, int32_t rank, px_halo_op ops[4], int32_t* nops, bool allow_self) {
  if (!ops || !nops) return fail(PX_ERR_ARG, "null argument");
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  *nops = 0;
  if (l->nranks == 1 && !(allow_self && l->bc == PX_BC_PERIODIC)) return PX_OK;
  const int32_t g = l->ghost;
  const int64_t count = (int64_t)(g - 1) * li.ld + ext(li.alloc, 0);
  auto off = [&](int32_t y) { return (int64_t)(y - li.alloc.lo.c[1]) * li.ld; };
  auto add = [&](int32_t peer, int32_t recv, int32_t row) {
    px_halo_op& o = ops[(*nops)++];
    o.peer = peer;
    o.is_recv = recv;
    o.row = row;
    o.nrows = g;
    o.offset = off(row);
    o.count = count;
  };
  if (li.nbr_hi >= 0) add(li.nbr_hi, 0, li.owned.hi.c[1] - g + 1);
  if (li.nbr_lo >= 0) add(li.nbr_lo, 0, li.owned.lo.c[1]);
  if (li.nbr_lo >= 0) add(li.nbr_lo, 1, li.owned.lo.c[1] - g);
  if (li.nbr_hi >= 0) add(li.nbr_hi, 1, li.owned.hi.c[1] + 1);
  return PX_OK;
}
}  // namespace px

extern "C" {

int64_t px_norm_buffer_len(px_box region) {
  // results (2) + counter slot (2) + 2 partials per block, for any phase
  int32_t nb = stream_blocks(ext(region, 0), ext(region, 1), 1);
  return 4 + 2 * (int64_t)nb;
}

}  // extern "C"

// ----------------------------------------------------- single-patch calls
namespace px {

// First violating (cell, tap) in the oracle's scan order (y-major, x
// fastest, taps in canonical order) when grow(region,1) is not inside src.
static px_status domain_violation(int stencil, const px_patch& src, const px_box& region) {
  static const int t5[5][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {0, 0}};
  static const int t9[9][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-1, -1},
                               {1, -1}, {-1, 1}, {1, 1}, {0, 0}};
  const int nt = stencil ? 9 : 5;
  const int(*t)[2] = stencil ? t9 : t5;
  int32_t xs[3] = {region.lo.c[0], std::min(region.lo.c[0] + 1, region.hi.c[0]), region.hi.c[0]};
  int32_t ys[2] = {region.lo.c[1], region.hi.c[1]};
  for (int iy = 0; iy < 2; ++iy)
    for (int ix = 0; ix < 3; ++ix)
      for (int k = 0; k < nt; ++k) {
        int32_t qx = xs[ix] + t[k][0], qy = ys[iy] + t[k][1];
        if (qx < src.box.lo.c[0] || qx > src.box.hi.c[0] || qy < src.box.lo.c[1] ||
            qy > src.box.hi.c[1])
          return fail(PX_ERR_DOMAIN, "stencil domain violation at i=(%d,%d) tap=(%d,%d)", xs[ix],
                      ys[iy], t[k][0], t[k][1]);
      }
  return PX_OK;
}

static int phase_of(const double* p) { return (int)(((uintptr_t)p >> 3) & 1); }

// Validate and describe a stream-kernel launch over `region`.
px_status make_stream_launch(int mode, int stencil, double scale, double lambda,
                             const px_patch* src, const px_patch* rhs, px_patch* dst,
                             px_box region, StreamLaunch* a) {
  if (stencil != PX_LAPLACE_5PT && stencil != PX_MEHRSTELLEN_9PT)
    return fail(PX_ERR_ARG, "bad stencil %d", stencil);
  PX_TRY(check_patch(src, "src"));
  if (dst) PX_TRY(check_patch(dst, "dst"));
  if (rhs) PX_TRY(check_patch(rhs, "rhs"));
  std::memset(a, 0, sizeof *a);
  if (empty(region)) return PX_OK;
  if (!contains(src->box, grow(region, 1))) return domain_violation(stencil, *src, region);
  if (dst && !contains(dst->box, region))
    return fail(PX_ERR_DOMAIN, "region [(%d,%d),(%d,%d)] not inside the output patch",
                region.lo.c[0], region.lo.c[1], region.hi.c[0], region.hi.c[1]);
  if (rhs && !contains(rhs->box, region))
    return fail(PX_ERR_DOMAIN, "region not inside the rhs patch");
  const double* s0 = at(*src, region.lo.c[0], region.lo.c[1]);
  const int ph = phase_of(s0);
  if (dst && phase_of(at(*dst, region.lo.c[0], region.lo.c[1])) != ph)
    return fail(PX_ERR_ALIGN, "src and dst have different 16-byte phases at region.lo");
  if (rhs && phase_of(at(*rhs, region.lo.c[0], region.lo.c[1])) != ph)
    return fail(PX_ERR_ALIGN, "src and rhs have different 16-byte phases at region.lo");
  if (dst && (mode == MODE_RELAX || mode == MODE_APPLY || mode == MODE_MRHS)) {
    const char* s_lo = (const char*)src->data;
    const char* s_hi = (const char*)(src->data + (int64_t)(ext(src->box, 1) - 1) * src->ld + ext(src->box, 0));
    const char* d_lo = (const char*)dst->data;
    const char* d_hi = (const char*)(dst->data + (int64_t)(ext(dst->box, 1) - 1) * dst->ld + ext(dst->box, 0));
    if (s_lo < d_hi && d_lo < s_hi) return fail(PX_ERR_ARG, "input and output patches overlap");
  }
  a->src = s0;
  a->rhs = rhs ? at(*rhs, region.lo.c[0], region.lo.c[1]) : nullptr;
  a->dst = dst ? at(*dst, region.lo.c[0], region.lo.c[1]) : nullptr;
  a->ld_src = src->ld;
  a->ld_rhs = rhs ? rhs->ld : 0;
  a->ld_dst = dst ? dst->ld : 0;
  a->nx = ext(region, 0);
  a->ny = ext(region, 1);
  a->phase = ph;
  a->src_x0 = src->box.lo.c[0] - region.lo.c[0];
  a->src_x1 = src->box.hi.c[0] - region.lo.c[0];
  a->scale = scale;
  a->lambda = lambda;
  return PX_OK;
}

uint64_t layout_generation(const px_layout* l) { return l ? l->gen : 0; }

double stencil_scale(int stencil, double h) {
  return stencil == PX_MEHRSTELLEN_9PT ? 1.0 / (6.0 * h * h) : 1.0 / (h * h);
}

static px_status attach_norms(int mode, StreamLaunch* a, double* d_norms) {
  if (!d_norms) return PX_OK;
  a->norms.out_max = d_norms;
  a->norms.out_sum = d_norms + 1;
  a->norms.counter = reinterpret_cast<unsigned int*>(d_norms + 2);
  a->norms.partials = d_norms + 4;
  a->norms.offset = 0;
  a->norms.expected = launch_blocks(mode, *a);
  return PX_OK;
}

}  // namespace px

extern "C" {

px_status px_stencil_apply(int32_t stencil, double scale, const px_patch* src, px_patch* dst,
                           px_box dest_box, void* stream) {
  StreamLaunch a;
  if (!dst) return fail(PX_ERR_ARG, "null dst");
  PX_TRY(make_stream_launch(MODE_APPLY, stencil, scale, 0.0, src, nullptr, dst, dest_box, &a));
  return launch_stream(MODE_APPLY, stencil, a, (cudaStream_t)stream);
}

px_status px_relax_step(const px_relax_params* p, const px_patch* phi_in, px_patch* phi_out,
                        const px_patch* rhs, px_box region, double* d_norms, void* stream) {
  if (!p) return fail(PX_ERR_ARG, "null params");
  if (!phi_out || !rhs) return fail(PX_ERR_ARG, "null phi_out or rhs");
  if (!(p->h > 0.0)) return fail(PX_ERR_ARG, "h must be positive");
  StreamLaunch a;
  PX_TRY(make_stream_launch(MODE_RELAX, p->stencil, stencil_scale(p->stencil, p->h), p->lambda,
                            phi_in, rhs, phi_out, region, &a));
  if (empty(region)) {
    if (d_norms)
      return cuda_check(cudaMemsetAsync(d_norms, 0, 2 * sizeof(double), (cudaStream_t)stream),
                        "memset norms");
    return PX_OK;
  }
  attach_norms(MODE_RELAX, &a, d_norms);
  return launch_stream(MODE_RELAX, p->stencil, a, (cudaStream_t)stream);
}

int32_t px_relax_variant(const px_patch* phi_in, const px_patch* phi_out, const px_patch* rhs,
                         px_box region) {
  StreamLaunch a;
  px_patch out = phi_out ? *phi_out : px_patch{};
  if (make_stream_launch(MODE_RELAX, PX_LAPLACE_5PT, 1.0, 0.0, phi_in, rhs, phi_out ? &out : nullptr,
                         region, &a) != PX_OK)
    return -1;
  return bulk_eligible(MODE_RELAX, a) ? 1 : 0;
}

px_status px_relax_block(const px_relax_params* p, int32_t k, const px_patch* phi_in,
                         px_patch* phi_out, const px_patch* rhs, px_box region, double* d_norms,
                         void* stream) {
  if (!p) return fail(PX_ERR_ARG, "null params");
  if (!phi_out || !rhs) return fail(PX_ERR_ARG, "null phi_out or rhs");
  if (!(p->h > 0.0)) return fail(PX_ERR_ARG, "h must be positive");
  if (k != 2 && k != 4) return fail(PX_ERR_UNSUPPORTED, "k=%d not built (2 or 4)", k);
  StreamLaunch a;
  PX_TRY(make_stream_launch(MODE_RELAX, p->stencil, stencil_scale(p->stencil, p->h), p->lambda,
                            phi_in, rhs, phi_out, region, &a));
  if (empty(region)) return PX_OK;
  if (!contains(phi_in->box, grow(region, k)))
    return fail(PX_ERR_DOMAIN, "phi_in must cover the region grown by k=%d", k);
  if (!contains(rhs->box, grow(region, k)))
    return fail(PX_ERR_DOMAIN, "rhs must cover the region grown by k=%d", k);
  if (a.phase != 0 || (a.nx & 1))
    return fail(PX_ERR_ALIGN, "temporal blocking needs a 16-byte aligned region start and an even width");
  TbLaunch x;
  std::memset(&x, 0, sizeof x);
  if (d_norms) {
    x.lvl[0].out_max = d_norms;
    x.lvl[0].out_sum = d_norms + 1;
    x.lvl[0].counter = reinterpret_cast<unsigned int*>(d_norms + 2);
    x.lvl[0].partials = d_norms + 4;
    x.lvl[0].offset = 0;
    x.lvl[0].expected = tb_blocks(k, a);
  }
  return launch_tb(p->stencil, k, a, x, (cudaStream_t)stream);
}

px_status px_residual_norm(const px_relax_params* p, const px_patch* phi, const px_patch* rhs,
                           px_box region, double* d_norms, void* stream) {
  if (!p || !d_norms || !rhs) return fail(PX_ERR_ARG, "null argument");
  if (!(p->h > 0.0)) return fail(PX_ERR_ARG, "h must be positive");
  StreamLaunch a;
  PX_TRY(make_stream_launch(MODE_RESID, p->stencil, stencil_scale(p->stencil, p->h), 0.0, phi,
                            rhs, nullptr, region, &a));
  if (empty(region))
    return cuda_check(cudaMemsetAsync(d_norms, 0, 2 * sizeof(double), (cudaStream_t)stream),
                      "memset norms");
  attach_norms(MODE_RESID, &a, d_norms);
  return launch_stream(MODE_RESID, p->stencil, a, (cudaStream_t)stream);
}

px_status px_mehrstellen_rhs(const px_patch* rho, px_patch* f, px_box region, void* stream) {
  if (!f) return fail(PX_ERR_ARG, "null f");
  StreamLaunch a;
  PX_TRY(make_stream_launch(MODE_MRHS, PX_LAPLACE_5PT, 1.0 / 12.0, 0.0, rho, nullptr, f, region,
                            &a));
  return launch_stream(MODE_MRHS, PX_LAPLACE_5PT, a, (cudaStream_t)stream);
}

px_status px_init_field(const px_layout* l, int32_t rank, px_patch* dst, int32_t kind,
                        uint64_t seed, int32_t k, int32_t l_wave, void* stream) {
  PX_TRY(check_patch(dst, "dst"));
  if (kind < PX_FIELD_ZERO || kind > PX_FIELD_SINE) return fail(PX_ERR_ARG, "bad field kind");
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  if (!contains(dst->box, li.owned)) return fail(PX_ERR_SHAPE, "patch does not cover the slab");
  return launch_init_field(l, rank, *dst, kind, seed, k, l_wave, (cudaStream_t)stream);
}

px_status px_fill_ghosts(const px_layout* l, int32_t rank, px_patch* phi, void* stream) {
  PX_TRY(check_patch(phi, "phi"));
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  if (!contains(phi->box, li.alloc))
    return fail(PX_ERR_SHAPE, "patch does not cover the ghosted slab");
  return launch_fill_ghosts(l, rank, *phi, (cudaStream_t)stream);
}

}  // extern "C"
