// px_solve.cu -- communicator (NCCL over NVLink/NVSwitch), ghost exchange
// and the N-sweep solve driver of libprotox (figure `Proto`, P:156-175,
// with stencil + update + norm fused into one kernel per sweep).
//
// Per sweep, for a slab decomposition over P ranks:
//   compute stream:  boundary rows [0,g) and [ny-g,ny) of φ'   (fused ghost
//                    images along x, and at Dirichlet faces along y)
//   comm stream:     NCCL grouped send/recv of those rows into the
//                    neighbours' ghost rows (full padded rows -> corners right)
//   compute stream:  interior rows [g, ny-g) of φ' -- overlaps the exchange
//   next sweep:      waits on the exchange event.
// Residual norms of every recorded iterate land in a device ring (max, Σr²);
// one ncclAllReduce (max) + one (sum) over the ring at the end
// (computeMaxResidualAcrossProcs, batched -- the solve runs a fixed
// sweep count, R23).  Single-rank layouts skip NCCL: the fused
// kernel writes its own periodic/Dirichlet images in both dimensions.
// The whole sweep sequence can be captured once into a CUDA graph.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys timelines, no link dependency

#include "px_internal.h"

// NVTX range for the scope (host side: marks the enqueue of a solve phase
// and, in px_solve, the whole host-synchronous call)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Peer-memory halo state (px_comm_p2p_export / _import, px_comm_enable_p2p).
// Control block of a rank (one cudaMalloc, exported over CUDA IPC), u64 words:
enum : int {
  CTL_FROM_LO = 0,    // arrivals pushed by the rank below
  CTL_FROM_HI = 1,    // arrivals pushed by the rank above
  CTL_EPOCH = 2,      // [2] arrival base of the current solve, [3] previous solve's arrivals
  CTL_AR_ARRIVE = 4,  // peer norm all-reduce: mailboxes published by peers
  CTL_AR_DONE = 5,    //   mailboxes read by peers
  CTL_AR_ROUND = 6,   //   own round counter
  CTL_TIMEOUT = 7,    // waits of this rank that gave up (px_spin_until): the communicator is broken
  CTL_MBOX = 8,       // mailbox: 2 * PX_MBOX_ENTRIES doubles
};
static constexpr size_t CTL_BYTES = (CTL_MBOX + 2 * px::PX_MBOX_ENTRIES) * sizeof(unsigned long long);

struct P2PState {
  bool exported = false, enabled = false;
  uint64_t gen = 0;                             // changes with every (re)registration: part of the plan key
  uint64_t layout_gen = 0;
  int32_t rank = 0;
  const double* bufs[2] = {nullptr, nullptr};   // own registered φ (A) and scratch (B)
  double* peer_lo[2] = {nullptr, nullptr};      // lower neighbour's A, B (patch data pointers)
  double* peer_hi[2] = {nullptr, nullptr};      // upper neighbour's A, B
  unsigned long long* ctl = nullptr;            // own control block
  std::vector<unsigned long long*> ctl_of;      // every rank's control block (mapped; own at [rank])
  std::vector<void*> opened;                    // IPC-mapped peer allocations
};

// One 256-byte record per rank (px_comm_p2p_export): IPC handles of the
// allocations holding A, B and the control block, and the offsets into them.
struct P2PBlob {
  uint32_t magic;
  int32_t rank, nranks, pad;
  int64_t ld, n0;                 // slab pitch and width (checked on import)
  cudaIpcMemHandle_t h[3];        // A, B, control block
  uint64_t off[3];
};
static_assert(sizeof(P2PBlob) <= PX_P2P_BLOB_BYTES, "P2P blob size");
static constexpr uint32_t P2P_MAGIC = 0x50583250u;  // "PX2P"

struct px_comm {
  ncclComm_t nccl = nullptr;   // null: peer-memory-only communicator (px_comm_create_peer)
  int32_t nranks = 1, rank = 0, device = 0;
  cudaStream_t stream = nullptr;
  bool self_exchange = false;  // 1 rank, periodic: exchange ghost rows with itself (test mode)
  P2PState p2p;
};

namespace px {

static px_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PX_OK;
  return fail(PX_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

static px_status check_rank_patch(const px_layout* l, int32_t rank, const px_patch* p,
                                  const char* name, px_local_info* li) {
  PX_TRY(check_patch(p, name));
  PX_TRY(local_info(l, rank, li));
  if (p->box.lo.c[0] != li->alloc.lo.c[0] || p->box.lo.c[1] != li->alloc.lo.c[1] ||
      p->box.hi.c[0] != li->alloc.hi.c[0] || p->box.hi.c[1] != li->alloc.hi.c[1])
    return fail(PX_ERR_SHAPE, "%s: patch box is not rank %d's ghosted slab", name, rank);
  if (p->ld != li->ld) return fail(PX_ERR_SHAPE, "%s: ld %lld != layout ld %lld", name,
                                   (long long)p->ld, (long long)li->ld);
  return PX_OK;
}

// NCCL row exchange of one rank (y-ghost rows from the neighbours), posted
// in the order of px_layout_halo_plan inside one group.
// Does this (layout, communicator) pair exchange ghost rows over NCCL?
static bool comm_exchanges(const px_layout* l, const px_comm* c) {
  return c && (l->nranks > 1 || (c->self_exchange && l->bc == PX_BC_PERIODIC));
}

static px_status nccl_rows(const px_layout* l, px_comm* c, int32_t rank, const px_patch& p,
                           cudaStream_t s) {
  px_halo_op ops[4];
  int32_t n = 0;
  PX_TRY(halo_plan(l, rank, ops, &n, c->self_exchange));
  PX_TRY(nccl_check(ncclGroupStart(), "ncclGroupStart"));
  for (int32_t i = 0; i < n; ++i) {
    double* buf = p.data + ops[i].offset;
    ncclResult_t r = ops[i].is_recv
                         ? ncclRecv(buf, (size_t)ops[i].count, ncclDouble, ops[i].peer, c->nccl, s)
                         : ncclSend(buf, (size_t)ops[i].count, ncclDouble, ops[i].peer, c->nccl, s);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_check(r, ops[i].is_recv ? "ncclRecv" : "ncclSend");
    }
  }
  return nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

// The same plan executed among all slabs held on ONE device: each receive
// is served by the matching send of the peer (k-th send to this rank fills
// its k-th receive from that peer) with a device-to-device copy.
static px_status local_rows(const px_layout* l, const px_patch* parts, cudaStream_t s) {
  for (int32_t r = 0; r < l->nranks; ++r) {
    px_halo_op ops[4];
    int32_t n = 0;
    PX_TRY(px_layout_halo_plan(l, r, ops, &n));
    for (int32_t i = 0; i < n; ++i) {
      if (!ops[i].is_recv) continue;
      int32_t k = 0;  // ordinal of this receive among receives from the peer
      for (int32_t j = 0; j < i; ++j) k += (ops[j].is_recv && ops[j].peer == ops[i].peer);
      px_halo_op pops[4];
      int32_t pn = 0;
      PX_TRY(px_layout_halo_plan(l, ops[i].peer, pops, &pn));
      int32_t seen = 0, match = -1;
      for (int32_t j = 0; j < pn; ++j)
        if (!pops[j].is_recv && pops[j].peer == r && seen++ == k) match = j;
      if (match < 0) return fail(PX_ERR_STATE, "halo plan mismatch between ranks %d and %d", r, ops[i].peer);
      PX_TRY(cuda_check(cudaMemcpyAsync(parts[r].data + ops[i].offset,
                                        parts[ops[i].peer].data + pops[match].offset,
                                        (size_t)ops[i].count * sizeof(double),
                                        cudaMemcpyDeviceToDevice, s),
                        "local exchange copy"));
    }
  }
  return PX_OK;
}

// ------------------------------------------------------------ solve plans
struct PlanKey {
  uint64_t layout_gen;
  const px_comm* comm;
  uint64_t p2p_gen;  // the communicator's peer registration (a cached graph bakes in its mode and pointers)
  int32_t rank, stencil, nsweeps, norm_every, k, nparts;
  double h, lambda;
  std::vector<const double*> ptrs;
  std::vector<int64_t> rhs_geom;  // per part: rhs box lo/hi and ld (baked into captured launches)
  cudaStream_t stream;
  bool operator==(const PlanKey& o) const {
    return layout_gen == o.layout_gen && comm == o.comm && p2p_gen == o.p2p_gen && rank == o.rank && stencil == o.stencil &&
           nsweeps == o.nsweeps && norm_every == o.norm_every && k == o.k && nparts == o.nparts &&
           h == o.h && lambda == o.lambda && ptrs == o.ptrs && rhs_geom == o.rhs_geom && stream == o.stream;
  }
};

struct Plan {
  PlanKey key;
  int32_t n_entries = 0;
  double* d_max = nullptr;      // ring of recorded norms
  double* d_sum = nullptr;
  double* d_ws = nullptr;       // per region: counter (2 doubles) + partials
  int64_t ws_len = 0, ws_stride = 0;
  cudaGraphExec_t exec = nullptr;
  int64_t launches_per_run = 0;
  cudaEvent_t ev_bnd = nullptr, ev_comm = nullptr;
  std::string kernels;          // sweep kernels the solve enqueues (px_last_solve_kernels)
  double* d_res = nullptr;      // shared-memory-resident solve: flags, row mailboxes, partials
  ~Plan() {
    if (d_res) cudaFree(d_res);
    if (exec) cudaGraphExecDestroy(exec);
    if (d_max) cudaFree(d_max);
    if (d_sum) cudaFree(d_sum);
    if (d_ws) cudaFree(d_ws);
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    if (ev_comm) cudaEventDestroy(ev_comm);
  }
};

// PROTOX_RESIDENT=0 (read once) disables the shared-memory-resident solve
// (A/B against the L2 persistent kernel).
static bool resident_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PROTOX_RESIDENT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static std::vector<std::unique_ptr<Plan>>& plans() {
  static std::vector<std::unique_ptr<Plan>> v;
  return v;
}

int plan_cache_cap() {
  static int cap = 0;
  if (!cap) {
    const char* e = getenv("PROTOX_PLAN_CACHE");
    cap = e ? atoi(e) : 32;
    if (cap < 1) cap = 1;
  }
  return cap;
}

void drop_layout_plans(uint64_t gen) {
  auto& v = plans();
  const bool any = std::any_of(v.begin(), v.end(), [gen](const std::unique_ptr<Plan>& p) { return p->key.layout_gen == gen; });
  if (any) {
    cudaDeviceSynchronize();  // a dropped plan's graph may still be in flight
    v.erase(std::remove_if(v.begin(), v.end(), [gen](const std::unique_ptr<Plan>& p) { return p->key.layout_gen == gen; }),
            v.end());
  }
  mg_drop_layout_plans(gen);
}

struct SolveCtx {
  const px_layout* l;
  px_comm* c;
  int32_t rank;
  const px_relax_params* p;
  const px_solve_opts* o;
  int32_t nparts;
  const px_patch* phi;
  const px_patch* scr;
  const px_patch* rhs;
  Plan* plan;
  cudaStream_t s;
};

// fused ghost images of a part's sweep
static GhostSpec ghost_spec(const px_layout* l, const px_local_info& li, const px_box& region,
                            bool single_rank) {
  GhostSpec gs;
  std::memset(&gs, 0, sizeof gs);
  gs.g = l->ghost;
  gs.n[0] = ext(li.owned, 0);
  gs.n[1] = ext(li.owned, 1);
  gs.o[0] = region.lo.c[0] - li.owned.lo.c[0];
  gs.o[1] = region.lo.c[1] - li.owned.lo.c[1];
  int mx = l->bc == PX_BC_PERIODIC ? GH_WRAP : (l->bc == PX_BC_DIRICHLET_CC ? GH_REFLECT : GH_NONE);
  gs.mode[0][0] = gs.mode[0][1] = mx;
  if (l->bc == PX_BC_PERIODIC && single_rank) {
    gs.mode[1][0] = gs.mode[1][1] = GH_WRAP;
  } else if (l->bc == PX_BC_DIRICHLET_CC) {
    gs.mode[1][0] = li.nbr_lo < 0 ? GH_REFLECT : GH_NONE;
    gs.mode[1][1] = li.nbr_hi < 0 ? GH_REFLECT : GH_NONE;
  }
  return gs;
}

// The launches of one sweep (or of the final residual when resid=true).
struct SweepLaunch {
  StreamLaunch a;
  int32_t blocks;
};

static px_status build_part_launches(const SolveCtx& x, int32_t part, const px_patch& in,
                                     const px_patch& out, bool resid, bool split,
                                     std::vector<SweepLaunch>& v) {
  const int32_t rank = x.c ? x.rank : (x.nparts > 1 ? part : 0);
  px_local_info li;
  PX_TRY(local_info(x.l, rank, &li));
  const int32_t g = x.l->ghost, ny = ext(li.owned, 1);
  std::vector<px_box> regions;
  const px_box& ow = li.owned;
  if (split && ny > 2 * g) {
    regions.push_back(mkbox(ow.lo.c[0], ow.lo.c[1], ow.hi.c[0], ow.lo.c[1] + g - 1));
    regions.push_back(mkbox(ow.lo.c[0], ow.hi.c[1] - g + 1, ow.hi.c[0], ow.hi.c[1]));
    regions.push_back(mkbox(ow.lo.c[0], ow.lo.c[1] + g, ow.hi.c[0], ow.hi.c[1] - g));
  } else {
    regions.push_back(ow);
  }
  const double scale = stencil_scale(x.p->stencil, x.p->h);
  for (const px_box& rg : regions) {
    SweepLaunch sl;
    px_patch outp = out;
    PX_TRY(make_stream_launch(resid ? MODE_RESID : MODE_RELAX, x.p->stencil, scale, x.p->lambda,
                              &in, &x.rhs[part], resid ? nullptr : &outp, rg, &sl.a));
    if (!resid) sl.a.gs = ghost_spec(x.l, li, rg, x.l->nranks == 1 && !comm_exchanges(x.l, x.c));
    sl.blocks = launch_blocks(resid ? MODE_RESID : MODE_RELAX, sl.a);
    v.push_back(sl);
  }
  return PX_OK;
}

// Norm-slot workspace region j (one per level of a temporal-blocking pass):
// a ticket counter (2 doubles) followed by 2 partials per block.
static double* ws_region(Plan* plan, int32_t j) { return plan->d_ws + (int64_t)j * plan->ws_stride; }

static void set_slot(std::vector<SweepLaunch>& v, size_t first, Plan* plan, int32_t entry) {
  int32_t total = 0;
  for (size_t i = first; i < v.size(); ++i) total += v[i].blocks;
  int32_t off = 0;
  for (size_t i = first; i < v.size(); ++i) {
    NormSlot& ns = v[i].a.norms;
    if (entry < 0) {
      std::memset(&ns, 0, sizeof ns);
      continue;
    }
    ns.out_max = plan->d_max + entry;
    ns.out_sum = plan->d_sum + entry;
    ns.counter = reinterpret_cast<unsigned int*>(ws_region(plan, 0));
    ns.partials = ws_region(plan, 0) + 2;
    ns.offset = off;
    ns.expected = total;
    off += v[i].blocks;
  }
}

static px_status exchange_all(const SolveCtx& x, const px_patch* parts) {
  if (x.c) {
    PX_TRY(launch_fill_ghosts(x.l, x.rank, parts[0], x.s));
    if (comm_exchanges(x.l, x.c)) {
      PX_TRY(cuda_check(cudaEventRecord(x.plan->ev_bnd, x.s), "event record"));
      PX_TRY(cuda_check(cudaStreamWaitEvent(x.c->stream, x.plan->ev_bnd, 0), "stream wait"));
      PX_TRY(nccl_rows(x.l, x.c, x.rank, parts[0], x.c->stream));
      PX_TRY(cuda_check(cudaEventRecord(x.plan->ev_comm, x.c->stream), "event record"));
      PX_TRY(cuda_check(cudaStreamWaitEvent(x.s, x.plan->ev_comm, 0), "stream wait"));
    }
    return PX_OK;
  }
  for (int32_t r = 0; r < x.nparts; ++r) PX_TRY(launch_fill_ghosts(x.l, x.nparts > 1 ? r : 0, parts[r], x.s));
  if (x.nparts > 1) PX_TRY(local_rows(x.l, parts, x.s));
  return PX_OK;
}

// Copy the ghost cells at the domain faces of a rank's slab (x-ghost columns
// of every row; full ghost rows at y faces) from `a` to `b`.
static px_status copy_face_ghosts(const px_layout* l, int32_t rank, const px_patch& a,
                                  const px_patch& b, cudaStream_t s) {
  px_local_info li;
  PX_TRY(local_info(l, rank, &li));
  const int32_t g = l->ghost, nx = ext(li.owned, 0), ny = ext(li.owned, 1);
  const size_t pitch = li.ld * sizeof(double);
  const int32_t x0 = li.owned.lo.c[0], y0 = li.owned.lo.c[1];
  for (int side = 0; side < 2; ++side) {
    const int32_t xs = side ? x0 + nx : x0 - g;
    PX_TRY(cuda_check(cudaMemcpy2DAsync(at(b, xs, y0), pitch, at(a, xs, y0), pitch, g * sizeof(double),
                                        ny, cudaMemcpyDeviceToDevice, s), "copy ghost columns"));
  }
  const size_t row = ext(li.alloc, 0) * sizeof(double);
  if (li.nbr_lo < 0)
    PX_TRY(cuda_check(cudaMemcpy2DAsync(at(b, x0 - g, y0 - g), pitch, at(a, x0 - g, y0 - g), pitch, row, g,
                                        cudaMemcpyDeviceToDevice, s), "copy ghost rows"));
  if (li.nbr_hi < 0)
    PX_TRY(cuda_check(cudaMemcpy2DAsync(at(b, x0 - g, y0 + ny), pitch, at(a, x0 - g, y0 + ny), pitch, row, g,
                                        cudaMemcpyDeviceToDevice, s), "copy ghost rows"));
  return PX_OK;
}

// Whole single-box solve in one launch (K9) when the box fits in shared memory.
static bool smallbox_path(const SolveCtx& x) {
  if (x.c || x.nparts != 1 || x.l->nranks != 1 || x.l->ghost != 1) return false;
  if (x.o->temporal_k > 1) return false;
  const int32_t nx = ext(x.l->domain, 0), ny = ext(x.l->domain, 1);
  return nx * ny <= 16384 && smallbox_fits(nx, ny);
}

static px_status enqueue_smallbox(const SolveCtx& x) {
  px_local_info li;
  PX_TRY(local_info(x.l, 0, &li));
  const int32_t N = x.o->nsweeps, E = x.o->norm_every;
  SmallBox b;
  std::memset(&b, 0, sizeof b);
  const int32_t x0 = li.owned.lo.c[0], y0 = li.owned.lo.c[1];
  const px_patch& out = (N % 2) ? x.scr[0] : x.phi[0];  // the buffer the sweep-by-sweep path ends in
  b.phi_in = at(x.phi[0], x0, y0);
  b.phi_out = at(out, x0, y0);
  b.rhs = at(x.rhs[0], x0, y0);
  b.ld_in = x.phi[0].ld;
  b.ld_out = out.ld;
  b.ld_rhs = x.rhs[0].ld;
  b.nx = ext(li.owned, 0);
  b.ny = ext(li.owned, 1);
  b.g = 1;
  b.bc = x.l->bc;
  b.stencil = x.p->stencil;
  b.scale = stencil_scale(x.p->stencil, x.p->h);
  b.lambda = x.p->lambda;
  b.nsweeps = N;
  b.every = E;
  b.final_norm = E >= 0;
  b.d_max = x.plan->d_max;
  b.d_sum = x.plan->d_sum;
  if (!contains(x.rhs[0].box, li.owned)) return fail(PX_ERR_SHAPE, "rhs does not cover the box");
  return launch_smallbox(b, x.s);
}

// Norm all-reduce over peer memory (control blocks of every rank mapped).
static px_status peer_allreduce(const px_comm* c, double* d_max, double* d_sum, int32_t n, cudaStream_t s) {
  const P2PState& st = c->p2p;
  if (c->nranks > PX_PEER_MAX) return fail(PX_ERR_UNSUPPORTED, "peer all-reduce: more than %d ranks", PX_PEER_MAX);
  PeerAllreduce ar;
  std::memset(&ar, 0, sizeof ar);
  ar.d_max = d_max;
  ar.d_sum = d_sum;
  ar.n = n;
  ar.nranks = c->nranks;
  ar.rank = c->rank;
  ar.mbox_own = reinterpret_cast<double*>(st.ctl + CTL_MBOX);
  for (int32_t r = 0; r < c->nranks; ++r) {
    ar.mbox[r] = reinterpret_cast<const double*>(st.ctl_of[r] + CTL_MBOX);
    ar.arrive[r] = st.ctl_of[r] + CTL_AR_ARRIVE;
    ar.done[r] = st.ctl_of[r] + CTL_AR_DONE;
  }
  ar.own_arrive = st.ctl + CTL_AR_ARRIVE;
  ar.own_done = st.ctl + CTL_AR_DONE;
  ar.round = st.ctl + CTL_AR_ROUND;
  ar.err = st.ctl + CTL_TIMEOUT;
  return launch_peer_allreduce(ar, s);
}

// Does this solve run in the fused peer-memory push mode?  Needs registered
// buffers (either order), k = 1 and a slab the TMA kernel can push from.
// *G = arrivals per side per sweep, *swap = phi is the registered scratch.
static bool p2p_mode(const SolveCtx& x, int32_t* G, bool* swap) {
  if (!x.c || !comm_exchanges(x.l, x.c) || x.nparts != 1) return false;
  const P2PState& st = x.c->p2p;
  if (!st.enabled || st.layout_gen != layout_generation(x.l) || st.rank != x.rank) return false;
  if (x.o->temporal_k > 1 || x.o->nsweeps <= 0) return false;
  if (x.phi[0].data == st.bufs[0] && x.scr[0].data == st.bufs[1]) {
    *swap = false;
  } else if (x.phi[0].data == st.bufs[1] && x.scr[0].data == st.bufs[0]) {
    *swap = true;
  } else {
    return false;
  }
  px_local_info li;
  if (local_info(x.l, x.rank, &li) != PX_OK) return false;
  if (ext(li.owned, 1) <= 2 * x.l->ghost) return false;
  StreamLaunch a;
  px_patch outp = x.scr[0];
  if (make_stream_launch(MODE_RELAX, x.p->stencil, stencil_scale(x.p->stencil, x.p->h), x.p->lambda, &x.phi[0],
                         &x.rhs[0], &outp, li.owned, &a) != PX_OK)
    return false;
  a.ps.on = 1;
  a.ps.g = x.l->ghost;
  *G = bulk_push_arrivals(a);
  return *G > 0;
}

// Push-mode exchange of φ^0: local ghost fill, then the boundary rows (full
// padded rows) into both buffers of each neighbour, one arrival per side.
static px_status push_init(const SolveCtx& x, const px_local_info& li) {
  PX_TRY(launch_fill_ghosts(x.l, x.rank, x.phi[0], x.s));
  const P2PState& st = x.c->p2p;
  const int32_t g = x.l->ghost, x0 = li.owned.lo.c[0];
  PushInit pi;
  std::memset(&pi, 0, sizeof pi);
  pi.src_lo = at(x.phi[0], x0 - g, li.owned.lo.c[1]);
  pi.src_hi = at(x.phi[0], x0 - g, li.owned.hi.c[1] - g + 1);
  pi.ld = x.phi[0].ld;
  pi.row_len = ext(li.owned, 0) + 2 * g;
  pi.g = g;
  for (int side = 0; side < 2; ++side) {
    const int32_t pr = side == 0 ? li.nbr_lo : li.nbr_hi;
    if (pr < 0) continue;
    px_local_info nli;
    PX_TRY(local_info(x.l, pr, &nli));
    const int32_t ty = side == 0 ? nli.owned.hi.c[1] + 1 : nli.owned.lo.c[1] - g;  // their ghost rows
    const int64_t off = (int64_t)(x0 - g - nli.alloc.lo.c[0]) + (int64_t)(ty - nli.alloc.lo.c[1]) * nli.ld;
    for (int b = 0; b < 2; ++b) pi.dst[side][b] = (side == 0 ? st.peer_lo[b] : st.peer_hi[b]) + off;
    pi.rflag[side] = st.ctl_of[pr] + (side == 0 ? CTL_FROM_HI : CTL_FROM_LO);
  }
  return launch_push_init(pi, x.s);
}

// PROTOX_WRAP=1 (A/B, read once): periodic single-rank sweeps on the TMA
// kernel read the periodic images of their boundary rows / columns in place
// (no images, no ghost fill per sweep).  Off by default: measured at BJ.C3
// (scripts/c3_wrap_ab.sh) 248.6-250.8 vs 251.2-251.4
// Gcell-updates/s with the fill kernels between the sweeps, with or without
// programmatic dependent launches -- the back-to-back chain of sweep grids
// costs more than the two small fill launches it removes.
static bool wrap_enabled() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("PROTOX_WRAP");
    w = (e && e[0] == '1') ? 1 : 0;
  }
  return w == 1;
}

// Slab size (cells) from which a k = 1 sweep fills its ghost ring with a
// separate kernel instead of fused images (PROTOX_SEP_FILL_CELLS, read once:
// tests lower it to reach the path at small sizes).
static int64_t sep_fill_cells() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("PROTOX_SEP_FILL_CELLS");
    v = e ? atoll(e) : ((int64_t)64 << 20);
    if (v < 0) v = 0;
  }
  return v;
}

// Enqueue the whole solve on x.s (directly, or under graph capture).
static px_status enqueue_solve(const SolveCtx& x) {
  const int32_t N = x.o->nsweeps, E = x.o->norm_every;
  Plan* plan = x.plan;
  const bool nccl_multi = comm_exchanges(x.l, x.c);
  if (smallbox_path(x)) return enqueue_smallbox(x);
  // fused peer-memory push (px_comm_p2p_import): no NCCL call in the solve
  int32_t G = 0;
  bool swap = false;
  const bool p2p = p2p_mode(x, &G, &swap);
  if (x.c && !x.c->nccl && !p2p && comm_exchanges(x.l, x.c))
    return fail(PX_ERR_UNSUPPORTED,
                "a peer-memory communicator solves only in push mode (registered buffers, temporal_k = 1, "
                "even slab width, more than 2g rows)");
  px_local_info pli;
  PX_TRY(local_info(x.l, x.c ? x.rank : 0, &pli));
  // exchange ghosts of φ^0
  NvtxRange r_ex(p2p ? "protox/exchange_phi0 (peer push)" : "protox/exchange_phi0");
  if (p2p) {
    PX_TRY(launch_epoch_bump(x.c->p2p.ctl + CTL_EPOCH, PX_PUSH_INIT_CTAS + (unsigned long long)x.o->nsweeps * G, x.s));
    PX_TRY(push_init(x, pli));
  } else {
    PX_TRY(exchange_all(x, x.phi));
  }
  // FIXED_GHOSTS: the caller's ghost cells at domain faces belong to every
  // iterate (oracle R5); copy them into the scratch buffer once.
  if (x.l->bc == PX_BC_FIXED_GHOSTS) {
    for (int32_t part = 0; part < x.nparts; ++part)
      PX_TRY(copy_face_ghosts(x.l, x.c ? x.rank : part, x.phi[part], x.scr[part], x.s));
  }
  const px_patch* cur = x.phi;
  const px_patch* nxt = x.scr;
  const int32_t K = x.o->temporal_k > 1 ? x.o->temporal_k : 1;
  int32_t it = 0;
  // temporal blocking: K sweeps per pass, ghost exchange every K sweeps
  // single-rank problems below the TMA kernel's size: all sweeps in one
  // cooperative launch (launch latency would dominate one kernel per sweep)
  if (K == 1 && !x.c && x.nparts == 1 && x.l->nranks == 1 && N > 0) {
    px_local_info li;
    PX_TRY(local_info(x.l, 0, &li));
    const int32_t nx = ext(li.owned, 0), ny = ext(li.owned, 1);
    int rgrid = 0, rmax = 0;
    size_t rsmem = 0;
    if (resident_enabled() && resident_plan(nx, ny, &rgrid, &rmax, &rsmem)) {
      // the iterate fits in the SMs' shared memory: it stays there for all N sweeps
      ResidentLaunch rl;
      std::memset(&rl, 0, sizeof rl);
      const px_patch& A = x.phi[0];
      const px_patch& B = (N & 1) ? x.scr[0] : x.phi[0];
      rl.phi_in = at(A, li.owned.lo.c[0], li.owned.lo.c[1]);
      rl.phi_out = at(B, li.owned.lo.c[0], li.owned.lo.c[1]);
      rl.rhs = at(x.rhs[0], li.owned.lo.c[0], li.owned.lo.c[1]);
      rl.ld_in = A.ld;
      rl.ld_out = B.ld;
      rl.ld_rhs = x.rhs[0].ld;
      rl.nx = nx;
      rl.ny = ny;
      rl.rmax = rmax;
      const int m = x.l->bc == PX_BC_PERIODIC ? GH_WRAP : x.l->bc == PX_BC_DIRICHLET_CC ? GH_REFLECT : GH_NONE;
      rl.xmode[0] = rl.xmode[1] = rl.ymode[0] = rl.ymode[1] = m;
      rl.scale = stencil_scale(x.p->stencil, x.p->h);
      rl.lambda = x.p->lambda;
      rl.nsweeps = N;
      rl.every = E;
      rl.final_norm = E >= 0;
      rl.n_entries = plan->n_entries;
      rl.d_max = plan->d_max;
      rl.d_sum = plan->d_sum;
      if (!plan->d_res) return fail(PX_ERR_STATE, "resident workspace missing from the plan");
      rl.ws = plan->d_res;
      return launch_resident(x.p->stencil, rl, rgrid, rsmem, x.s);
    }
    if ((int64_t)nx * ny < (int64_t)4 * 1024 * 1024) {
      PersistLaunch pl;
      std::memset(&pl, 0, sizeof pl);
      const double scale = stencil_scale(x.p->stencil, x.p->h);
      px_patch A = x.phi[0], B = x.scr[0];
      PX_TRY(make_stream_launch(MODE_RELAX, x.p->stencil, scale, x.p->lambda, &A, &x.rhs[0], &B, li.owned, &pl.a0));
      PX_TRY(make_stream_launch(MODE_RELAX, x.p->stencil, scale, x.p->lambda, &B, &x.rhs[0], &A, li.owned, &pl.a1));
      PX_TRY(make_stream_launch(MODE_RESID, x.p->stencil, scale, 0.0, &A, &x.rhs[0], nullptr, li.owned, &pl.r0));
      PX_TRY(make_stream_launch(MODE_RESID, x.p->stencil, scale, 0.0, &B, &x.rhs[0], nullptr, li.owned, &pl.r1));
      if (pl.a0.phase == pl.a1.phase) {
        pl.a0.gs = pl.a1.gs = ghost_spec(x.l, li, li.owned, true);
        const int32_t grid = persist_grid();
        pl.nsweeps = N;
        pl.every = E;
        pl.final_norm = E >= 0;
        pl.d_max = plan->d_max;
        pl.d_sum = plan->d_sum;
        pl.partials = ws_region(plan, 0);
        pl.gx = (nx + pl.a0.phase + 511) / 512;
        pl.rows = persist_rows(nx + pl.a0.phase, ny, grid);
        pl.gy = (ny + pl.rows - 1) / pl.rows;
        return launch_persist(x.p->stencil, pl, grid, x.s);
      }
    }
  }
  while (K > 1 && it + K <= N) {
    std::vector<StreamLaunch> la(x.nparts);
    std::vector<TbLaunch> tl(x.nparts);
    std::vector<int32_t> blocks(x.nparts);
    int32_t total = 0;
    for (int32_t part = 0; part < x.nparts; ++part) {
      const int32_t rank = x.c ? x.rank : (x.nparts > 1 ? part : 0);
      px_local_info li;
      PX_TRY(local_info(x.l, rank, &li));
      px_patch outp = nxt[part];
      PX_TRY(make_stream_launch(MODE_RELAX, x.p->stencil, stencil_scale(x.p->stencil, x.p->h),
                                x.p->lambda, &cur[part], &x.rhs[part], &outp, li.owned, &la[part]));
      // no fused ghost images: the x-face strips would write an image per
      // row and level-K cell and, as items of the static schedule, hold the
      // whole pass back (a pass over 32768² took 5.47 ms in a solve vs 4.40 ms
      // without images); one ghost fill per pass (below) is ~10 µs
      la[part].gs.g = 0;
      std::memset(&tl[part], 0, sizeof(TbLaunch));
      const bool fixed = x.l->bc == PX_BC_FIXED_GHOSTS;
      tl[part].fix[0][0] = tl[part].fix[0][1] = fixed;
      tl[part].fix[1][0] = fixed && li.nbr_lo < 0;
      tl[part].fix[1][1] = fixed && li.nbr_hi < 0;
      const bool dir = x.l->bc == PX_BC_DIRICHLET_CC;  // per-level odd reflection at domain faces
      tl[part].refl[0][0] = tl[part].refl[0][1] = dir;
      tl[part].refl[1][0] = dir && li.nbr_lo < 0;
      tl[part].refl[1][1] = dir && li.nbr_hi < 0;
      blocks[part] = tb_blocks(K, la[part]);
      total += blocks[part];
    }
    int32_t off = 0;
    for (int32_t part = 0; part < x.nparts; ++part) {
      for (int32_t t = 0; t < K; ++t) {
        const int32_t m = it + t;
        NormSlot& ns = tl[part].lvl[t];
        if (E > 0 && m % E == 0) {
          ns.out_max = plan->d_max + m / E;
          ns.out_sum = plan->d_sum + m / E;
          ns.counter = reinterpret_cast<unsigned int*>(ws_region(plan, t));
          ns.partials = ws_region(plan, t) + 2;
          ns.offset = off;
          ns.expected = total;
        }
      }
      off += blocks[part];
    }
    for (int32_t part = 0; part < x.nparts; ++part)
      PX_TRY(launch_tb(x.p->stencil, K, la[part], tl[part], x.s));
    for (int32_t part = 0; part < x.nparts; ++part)  // the ghost cells this part fills itself
      PX_TRY(launch_fill_ghosts(x.l, x.c ? x.rank : (x.nparts > 1 ? part : 0), nxt[part], x.s));
    if (nccl_multi) {
      PX_TRY(cuda_check(cudaEventRecord(plan->ev_bnd, x.s), "event record"));
      PX_TRY(cuda_check(cudaStreamWaitEvent(x.c->stream, plan->ev_bnd, 0), "stream wait"));
      PX_TRY(nccl_rows(x.l, x.c, x.rank, nxt[0], x.c->stream));
      PX_TRY(cuda_check(cudaEventRecord(plan->ev_comm, x.c->stream), "event record"));
      PX_TRY(cuda_check(cudaStreamWaitEvent(x.s, plan->ev_comm, 0), "stream wait"));
    } else if (x.nparts > 1) {
      PX_TRY(local_rows(x.l, nxt, x.s));
    }
    std::swap(cur, nxt);
    it += K;
  }
  // Fused halo push over peer memory: ONE k_bulk launch per sweep stores the
  // slab's boundary rows into the neighbours' ghost rows and counts arrivals;
  // its boundary items wait for the neighbours' pushes of the previous sweep
  // (φ^0's rows: push_init).  No NCCL call and no comm stream per sweep.
  PushSpec ps;
  std::memset(&ps, 0, sizeof ps);
  if (p2p) {
    const P2PState& st = x.c->p2p;
    ps.on = 1;
    ps.g = x.l->ghost;
    ps.epoch = st.ctl + CTL_EPOCH;
    ps.err = st.ctl + CTL_TIMEOUT;
    const GhostSpec gsp = ghost_spec(x.l, pli, pli.owned, false);  // x images of the pushed rows
    ps.xg = gsp.g;
    ps.xn0 = gsp.n[0];
    ps.xm0 = gsp.mode[0][0];
    ps.xm1 = gsp.mode[0][1];
    for (int side = 0; side < 2; ++side) {
      const int32_t pr = side == 0 ? pli.nbr_lo : pli.nbr_hi;
      if (pr < 0) continue;
      ps.rflag[side] = st.ctl_of[pr] + (side == 0 ? CTL_FROM_HI : CTL_FROM_LO);
      ps.wflag[side] = st.ctl + (side == 0 ? CTL_FROM_LO : CTL_FROM_HI);
    }
  }
  NvtxRange r_sw(p2p ? "protox/sweeps (fused push)" : nccl_multi ? "protox/sweeps (NCCL halo)" : "protox/sweeps");
  // one launch per sweep (push mode, or one part without a NCCL exchange):
  // each sweep kernel is a programmatic dependent of the previous one, so
  // its launch and prologue overlap the previous sweep's tail
  const bool one_launch = p2p || (!nccl_multi && x.nparts == 1);
  const int32_t it_first = it;
  // A single-rank slab of >= 64 M cells writes its ghost ring with one fill
  // kernel per sweep instead of fused images: measured per sweep over the
  // sweep kernel alone (profiles/round2_fill_vs_images.jsonl) fused images
  // cost +0.1 / +3.5 / +6.9 / +5.0 % at 2048 / 4096 / 8192 / 16384 rows of
  // 16384 columns, the separate fill +1.4 / +2.4 / +3.3 / +3.0 %.
  // (the push path too: its pushed rows carry their corner images themselves)
  const bool sep_fill = ((!x.c && x.nparts == 1 && x.l->nranks == 1) || p2p) &&
                        (int64_t)ext(pli.owned, 0) * ext(pli.owned, 1) >= sep_fill_cells();
  const bool wrap_ok = !x.c && x.nparts == 1 && x.l->nranks == 1 && x.l->bc == PX_BC_PERIODIC && wrap_enabled();
  bool any_wrap = false;
  for (; it < N; ++it) {
    const int32_t slot = (E > 0 && it % E == 0) ? it / E : -1;
    std::vector<SweepLaunch> v;
    for (int32_t part = 0; part < x.nparts; ++part)
      PX_TRY(build_part_launches(x, part, cur[part], nxt[part], false, nccl_multi && !p2p, v));
    if (p2p) {  // the push-mode launch has its own geometry: count its blocks for the norm slot
      v[0].a.ps = ps;
      v[0].blocks = launch_blocks(MODE_RELAX, v[0].a);
    }
    set_slot(v, 0, plan, slot);
    if (one_launch && v.size() == 1 && it > it_first) v[0].a.pdl = 1;
    if (p2p) {
      const P2PState& st = x.c->p2p;
      const int nb = ((swap ? 1 : 0) + it + 1) & 1;  // the neighbours' buffer this sweep writes (their "next")
      const int32_t g = x.l->ghost, x0 = pli.owned.lo.c[0];
      StreamLaunch& a = v[0].a;
      if (sep_fill) a.gs.g = 0;
      a.ps.wcount = PX_PUSH_INIT_CTAS + (unsigned long long)it * G;
      a.ps.rel = it > 0;  // publish sweep it-1's pushes
      for (int side = 0; side < 2; ++side) {
        const int32_t pr = side == 0 ? pli.nbr_lo : pli.nbr_hi;
        if (pr < 0) continue;
        px_local_info nli;
        PX_TRY(local_info(x.l, pr, &nli));
        const int32_t ty = side == 0 ? nli.owned.hi.c[1] + 1 : nli.owned.lo.c[1] - g;  // their ghost rows
        double* base = side == 0 ? st.peer_lo[nb] : st.peer_hi[nb];
        a.ps.rdst[side] = base + (int64_t)(x0 - nli.alloc.lo.c[0]) + (int64_t)(ty - nli.alloc.lo.c[1]) * nli.ld;
      }
      PX_TRY(launch_stream(MODE_RELAX, x.p->stencil, a, x.s));
      if (sep_fill) PX_TRY(launch_fill_ghosts(x.l, x.rank, nxt[0], x.s));  // own x ghosts, y faces
    } else if (nccl_multi) {
      // boundary rows, exchange on the comm stream, interior concurrently
      const bool split = v.size() == 3;
      PX_TRY(launch_stream(MODE_RELAX, x.p->stencil, v[0].a, x.s));
      if (split) PX_TRY(launch_stream(MODE_RELAX, x.p->stencil, v[1].a, x.s));
      PX_TRY(cuda_check(cudaEventRecord(plan->ev_bnd, x.s), "event record"));
      PX_TRY(cuda_check(cudaStreamWaitEvent(x.c->stream, plan->ev_bnd, 0), "stream wait"));
      PX_TRY(nccl_rows(x.l, x.c, x.rank, nxt[0], x.c->stream));
      PX_TRY(cuda_check(cudaEventRecord(plan->ev_comm, x.c->stream), "event record"));
      if (split) PX_TRY(launch_stream(MODE_RELAX, x.p->stencil, v[2].a, x.s));
      PX_TRY(cuda_check(cudaStreamWaitEvent(x.s, plan->ev_comm, 0), "stream wait"));
    } else {
      // a whole periodic single-rank domain on the TMA kernel reads the
      // periodic images of its boundary rows / columns straight from the
      // interior: no images written, no ghost fill per sweep
      const bool wr = wrap_ok && v.size() == 1 && bulk_eligible(MODE_RELAX, v[0].a);
      if (wr) {
        v[0].a.wrap = 1;
        v[0].a.gs.g = 0;
        any_wrap = true;
      } else if (sep_fill) {
        v[0].a.gs.g = 0;
      }
      for (auto& sl : v) PX_TRY(launch_stream(MODE_RELAX, x.p->stencil, sl.a, x.s));
      if (sep_fill && !wr) PX_TRY(launch_fill_ghosts(x.l, 0, nxt[0], x.s));
      if (x.nparts > 1) PX_TRY(local_rows(x.l, nxt, x.s));
    }
    std::swap(cur, nxt);
  }
  const int32_t entry = plan->n_entries - 1;
  if (p2p) {  // φ^N's ghost rows: the last sweep's pushes must have arrived
    PushSpec w = ps;
    w.wcount = PX_PUSH_INIT_CTAS + (unsigned long long)N * G;
    w.rel = 1;  // publish the last sweep's pushes
    PX_TRY(launch_wait(w, x.s));
  }
  // φ^N leaves with its ghost ring filled, as the fused-image sweeps leave it
  // (and the final residual pass reads it)
  if (any_wrap) PX_TRY(launch_fill_ghosts(x.l, 0, cur[0], x.s));
  if (E >= 0) {
    std::vector<SweepLaunch> v;
    for (int32_t part = 0; part < x.nparts; ++part)
      PX_TRY(build_part_launches(x, part, cur[part], cur[part], true, false, v));
    set_slot(v, 0, plan, entry);
    for (auto& sl : v) PX_TRY(launch_stream(MODE_RESID, x.p->stencil, sl.a, x.s));
  }
  NvtxRange r_ar("protox/norm_allreduce");
  if (p2p && plan->n_entries > 0) {
    PX_TRY(peer_allreduce(x.c, plan->d_max, plan->d_sum, plan->n_entries, x.s));
  } else if (nccl_multi && plan->n_entries > 0) {
    // max|r| as u64 bit patterns (|r| >= 0, so the order of the patterns is the
    // order of the values, and a NaN -- exponent all ones, sign clear -- is
    // above +inf): exact and NaN-propagating on every rank (R7).
    PX_TRY(nccl_check(ncclAllReduce(plan->d_max, plan->d_max, plan->n_entries, ncclUint64,
                                    ncclMax, x.c->nccl, x.s), "ncclAllReduce(max)"));
    PX_TRY(nccl_check(ncclAllReduce(plan->d_sum, plan->d_sum, plan->n_entries, ncclDouble,
                                    ncclSum, x.c->nccl, x.s), "ncclAllReduce(sum)"));
  }
  return PX_OK;
}

static int32_t count_entries(int32_t N, int32_t E) {
  if (E < 0) return 0;
  return (E > 0 ? (N + E - 1) / E : 0) + 1;
}

}  // namespace px

using namespace px;

namespace px {
// accessors for the 3D slab solve (px3d.cu)
void* comm_nccl(const px_comm* c) { return (void*)c->nccl; }
int32_t comm_nranks(const px_comm* c) { return c->nranks; }
int32_t comm_rank(const px_comm* c) { return c->rank; }
bool comm_self_exchange(const px_comm* c) { return c->self_exchange; }
}  // namespace px

extern "C" {

px_status px_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(PX_ERR_ARG, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId u;
  PX_TRY(nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId"));
  std::memcpy(id, &u, 128);
  return PX_OK;
}

static px_status comm_streams(px_comm* c) {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  return cuda_check(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi), "comm stream");
}

px_status px_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                         px_comm** out) {
  if (!id || !out) return fail(PX_ERR_ARG, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PX_ERR_ARG, "bad rank/nranks");
  PX_TRY(cuda_check(cudaSetDevice(device), "cudaSetDevice"));
  std::unique_ptr<px_comm> c(new px_comm());
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  PX_TRY(nccl_check(ncclCommInitRank(&c->nccl, nranks, u, rank), "ncclCommInitRank"));
  if (nranks == 1) {
    const char* e = getenv("PROTOX_NCCL_SELF_EXCHANGE");
    c->self_exchange = e && e[0] == '1';
  }
  PX_TRY(comm_streams(c.get()));
  *out = c.release();
  return PX_OK;
}

px_status px_comm_create_peer(int32_t nranks, int32_t rank, int32_t device, px_comm** out) {
  if (!out) return fail(PX_ERR_ARG, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PX_ERR_ARG, "bad rank/nranks");
  if (nranks > PX_PEER_MAX) return fail(PX_ERR_UNSUPPORTED, "peer communicator: at most %d ranks", PX_PEER_MAX);
  PX_TRY(cuda_check(cudaSetDevice(device), "cudaSetDevice"));
  std::unique_ptr<px_comm> c(new px_comm());
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (nranks == 1) {
    const char* e = getenv("PROTOX_NCCL_SELF_EXCHANGE");
    c->self_exchange = e && e[0] == '1';
  }
  PX_TRY(comm_streams(c.get()));
  *out = c.release();
  return PX_OK;
}

static uint64_t next_p2p_gen() {
  static uint64_t g = 0;
  return ++g;
}

static void p2p_close(P2PState& st) {
  for (void* b : st.opened) cudaIpcCloseMemHandle(b);
  st.opened.clear();
  st.ctl_of.clear();
  st.enabled = false;
  st.gen = next_p2p_gen();
}

void px_comm_destroy(px_comm* c) {
  if (!c) return;
  px::release3_for_comm(c);
  // drop plans that reference this communicator
  auto& v = plans();
  v.erase(std::remove_if(v.begin(), v.end(), [c](const std::unique_ptr<Plan>& p) { return p->key.comm == c; }),
          v.end());
  p2p_close(c->p2p);
  if (c->p2p.ctl) cudaFree(c->p2p.ctl);
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// base address of the allocation containing p (driver API, fetched at run
// time so the library does not link libcuda)
typedef int (*MemGetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);
static px_status alloc_base(const void* p, void** base, size_t* off) {
  static MemGetAddressRangeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
      return fail(PX_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    fn = (MemGetAddressRangeFn)f;
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)p) != 0) return fail(PX_ERR_CUDA, "cuMemGetAddressRange failed");
  *base = (void*)(uintptr_t)b;
  *off = (size_t)((uintptr_t)p - (uintptr_t)b);
  return PX_OK;
}

px_status px_comm_p2p_export(px_comm* c, const px_layout* l, int32_t rank, const px_patch* phi,
                             const px_patch* phi_scratch, uint8_t* blob) {
  if (!c || !l || !phi || !phi_scratch || !blob) return fail(PX_ERR_ARG, "null argument");
  if (c->nranks != l->nranks || c->rank != rank)
    return fail(PX_ERR_STATE, "communicator (rank %d of %d) does not match layout/rank", c->rank, c->nranks);
  px_local_info li;
  PX_TRY(check_rank_patch(l, rank, phi, "phi", &li));
  PX_TRY(check_rank_patch(l, rank, phi_scratch, "phi_scratch", &li));
  if (!comm_exchanges(l, c))
    return fail(PX_ERR_UNSUPPORTED, "peer halo push needs a multi-rank layout (or the 1-rank periodic self-exchange mode)");
  if (phi->data == phi_scratch->data) return fail(PX_ERR_ARG, "phi and phi_scratch must differ");
  P2PState& st = c->p2p;
  p2p_close(st);
  if (!st.ctl) PX_TRY(cuda_check(cudaMalloc(&st.ctl, CTL_BYTES), "cudaMalloc control block"));
  // counters restart at zero: no peer can push before it imports this record
  PX_TRY(cuda_check(cudaMemset(st.ctl, 0, CTL_BYTES), "memset control block"));
  PX_TRY(cuda_check(cudaDeviceSynchronize(), "memset control block"));
  st.bufs[0] = phi->data;
  st.bufs[1] = phi_scratch->data;
  st.layout_gen = layout_generation(l);
  st.rank = rank;
  P2PBlob mine;
  std::memset(&mine, 0, sizeof mine);
  mine.magic = P2P_MAGIC;
  mine.rank = rank;
  mine.nranks = c->nranks;
  mine.ld = li.ld;
  mine.n0 = ext(li.owned, 0);
  if (c->nranks > 1) {
    const void* ptrs[3] = {phi->data, phi_scratch->data, st.ctl};
    for (int i = 0; i < 3; ++i) {
      void* base = nullptr;
      size_t off = 0;
      PX_TRY(alloc_base(ptrs[i], &base, &off));
      PX_TRY(cuda_check(cudaIpcGetMemHandle(&mine.h[i], base), "cudaIpcGetMemHandle"));
      mine.off[i] = off;
    }
  }
  std::memset(blob, 0, PX_P2P_BLOB_BYTES);
  std::memcpy(blob, &mine, sizeof mine);
  st.exported = true;
  return PX_OK;
}

px_status px_comm_p2p_import(px_comm* c, const px_layout* l, const uint8_t* blobs) {
  if (!c || !l || !blobs) return fail(PX_ERR_ARG, "null argument");
  P2PState& st = c->p2p;
  if (!st.exported || st.layout_gen != layout_generation(l))
    return fail(PX_ERR_STATE, "px_comm_p2p_import before px_comm_p2p_export of this layout");
  p2p_close(st);
  std::vector<P2PBlob> all(c->nranks);
  px_local_info li;
  PX_TRY(local_info(l, st.rank, &li));
  for (int32_t r = 0; r < c->nranks; ++r) {
    std::memcpy(&all[r], blobs + (size_t)r * PX_P2P_BLOB_BYTES, sizeof(P2PBlob));
    if (all[r].magic != P2P_MAGIC || all[r].rank != r || all[r].nranks != c->nranks)
      return fail(PX_ERR_ARG, "p2p record %d is not rank %d's export for %d ranks", r, r, c->nranks);
    if (all[r].ld != li.ld || all[r].n0 != ext(li.owned, 0))
      return fail(PX_ERR_SHAPE, "p2p record %d: slab pitch/width differ from this rank's layout", r);
  }
  st.ctl_of.assign(c->nranks, nullptr);
  st.ctl_of[st.rank] = st.ctl;
  if (c->nranks == 1) {  // self-exchange: the neighbour is this rank
    for (int b = 0; b < 2; ++b) st.peer_lo[b] = st.peer_hi[b] = const_cast<double*>(st.bufs[b]);
    st.enabled = true;
    st.gen = next_p2p_gen();
    return PX_OK;
  }
  auto open = [&](int32_t r, int i, void** out) -> px_status {
    void* b = nullptr;
    PX_TRY(cuda_check(cudaIpcOpenMemHandle(&b, all[r].h[i], cudaIpcMemLazyEnablePeerAccess),
                      "cudaIpcOpenMemHandle"));
    st.opened.push_back(b);
    *out = (uint8_t*)b + all[r].off[i];
    return PX_OK;
  };
  px_status stt = PX_OK;
  for (int32_t r = 0; r < c->nranks && stt == PX_OK; ++r) {  // every rank's control block (all-reduce)
    if (r == st.rank) continue;
    void* p = nullptr;
    stt = open(r, 2, &p);
    st.ctl_of[r] = (unsigned long long*)p;
  }
  const int32_t peers[2] = {li.nbr_lo, li.nbr_hi};
  double* mapped[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  for (int side = 0; side < 2 && stt == PX_OK; ++side) {
    const int32_t pr = peers[side];
    if (pr < 0) continue;
    if (side == 1 && pr == peers[0]) {  // same neighbour on both sides (P = 2): map once
      mapped[1][0] = mapped[0][0];
      mapped[1][1] = mapped[0][1];
      continue;
    }
    for (int i = 0; i < 2 && stt == PX_OK; ++i) {
      void* p = nullptr;
      stt = open(pr, i, &p);
      mapped[side][i] = (double*)p;
    }
  }
  if (stt != PX_OK) {
    p2p_close(st);
    return stt;
  }
  for (int b = 0; b < 2; ++b) {
    st.peer_lo[b] = mapped[0][b];
    st.peer_hi[b] = mapped[1][b];
  }
  st.enabled = true;
  st.gen = next_p2p_gen();
  return PX_OK;
}

px_status px_comm_enable_p2p(px_comm* c, const px_layout* l, int32_t rank, const px_patch* phi,
                             const px_patch* phi_scratch) {
  if (!c) return fail(PX_ERR_ARG, "null argument");
  std::vector<uint8_t> all((size_t)PX_P2P_BLOB_BYTES * c->nranks);
  uint8_t* mine = all.data() + (size_t)PX_P2P_BLOB_BYTES * rank;
  PX_TRY(px_comm_p2p_export(c, l, rank, phi, phi_scratch, mine));
  if (c->nranks > 1) {
    if (!c->nccl) return fail(PX_ERR_STATE, "px_comm_enable_p2p needs NCCL; use px_comm_p2p_export/_import");
    // all-gather the records over NCCL
    const size_t sz = PX_P2P_BLOB_BYTES;
    uint8_t* d = nullptr;
    PX_TRY(cuda_check(cudaMalloc(&d, sz * (c->nranks + 1)), "cudaMalloc exchange"));
    px_status stt = cuda_check(cudaMemcpy(d + sz * c->nranks, mine, sz, cudaMemcpyHostToDevice), "H2D");
    if (stt == PX_OK)
      stt = nccl_check(ncclAllGather(d + sz * c->nranks, d, sz, ncclUint8, c->nccl, c->stream), "ncclAllGather");
    if (stt == PX_OK) stt = cuda_check(cudaStreamSynchronize(c->stream), "all-gather");
    if (stt == PX_OK) stt = cuda_check(cudaMemcpy(all.data(), d, sz * c->nranks, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d);
    PX_TRY(stt);
  }
  return px_comm_p2p_import(c, l, all.data());
}

px_status px_comm_allreduce_norms(px_comm* c, double* d_max, double* d_sum, int32_t n,
                                  void* stream) {
  if (!c || !d_max || !d_sum || n < 0) return fail(PX_ERR_ARG, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (!c->nccl) {
    if (c->nranks == 1) return PX_OK;
    if (!c->p2p.enabled) return fail(PX_ERR_STATE, "peer communicator: px_comm_p2p_import first");
    return peer_allreduce(c, d_max, d_sum, n, s);
  }
  PX_TRY(nccl_check(ncclGroupStart(), "ncclGroupStart"));
  // max as u64 bit patterns of non-negative doubles (NaN-propagating, R7)
  PX_TRY(nccl_check(ncclAllReduce(d_max, d_max, n, ncclUint64, ncclMax, c->nccl, s), "ncclAllReduce"));
  PX_TRY(nccl_check(ncclAllReduce(d_sum, d_sum, n, ncclDouble, ncclSum, c->nccl, s), "ncclAllReduce"));
  return nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

px_status px_exchange_ghosts(const px_layout* l, px_comm* c, int32_t rank, px_patch* phi,
                             void* stream) {
  px_local_info li;
  PX_TRY(check_rank_patch(l, rank, phi, "phi", &li));
  if (!c && l->nranks != 1) return fail(PX_ERR_ARG, "multi-rank layout needs a communicator");
  if (c && (c->nranks != l->nranks || c->rank != rank))
    return fail(PX_ERR_STATE, "communicator (rank %d of %d) does not match layout/rank", c->rank,
                c->nranks);
  cudaStream_t s = (cudaStream_t)stream;
  if (comm_exchanges(l, c) && !c->nccl)
    return fail(PX_ERR_UNSUPPORTED, "px_exchange_ghosts: the peer-memory communicator exchanges inside px_solve only");
  PX_TRY(launch_fill_ghosts(l, rank, *phi, s));
  if (comm_exchanges(l, c)) PX_TRY(nccl_rows(l, c, rank, *phi, s));
  return PX_OK;
}

px_status px_exchange_ghosts_local(const px_layout* l, const px_patch* parts, void* stream) {
  if (!l || !parts) return fail(PX_ERR_ARG, "null argument");
  px_local_info li;
  for (int32_t r = 0; r < l->nranks; ++r) PX_TRY(check_rank_patch(l, r, &parts[r], "part", &li));
  cudaStream_t s = (cudaStream_t)stream;
  for (int32_t r = 0; r < l->nranks; ++r) PX_TRY(launch_fill_ghosts(l, r, parts[r], s));
  return local_rows(l, parts, s);
}

}  // extern "C"

static thread_local std::string tl_last_kernels;  // px_last_solve_kernels

// Validate, find or build the plan, and enqueue the N sweeps on `stream`
// (graph replay or direct launches).  Nothing is synchronised: the recorded
// norms are in plan->d_max/d_sum and φ^N is in phi_scratch iff *odd.
static px_status solve_enqueue(const px_layout* l, px_comm* c, int32_t rank, const px_relax_params* p,
                               const px_solve_opts* o, px_patch* phi, px_patch* phi_scratch,
                               const px_patch* rhs, void* stream, Plan** plan_out, bool* odd_out,
                               int32_t* nparts_out) {
  if (!l || !p || !o || !phi || !phi_scratch || !rhs) return fail(PX_ERR_ARG, "null argument");
  if (o->nsweeps < 0) return fail(PX_ERR_ARG, "nsweeps must be >= 0");
  if (!(p->h > 0.0)) return fail(PX_ERR_ARG, "h must be positive");
  if (p->stencil != PX_LAPLACE_5PT && p->stencil != PX_MEHRSTELLEN_9PT)
    return fail(PX_ERR_ARG, "bad stencil %d", p->stencil);
  if (o->temporal_k < 0) return fail(PX_ERR_ARG, "temporal_k must be >= 0");
  if (o->temporal_k > 1) {
    if (o->temporal_k != 2 && o->temporal_k != 4)
      return fail(PX_ERR_UNSUPPORTED, "temporal_k=%d not built (1, 2 or 4)", o->temporal_k);
    if (o->temporal_k > l->ghost)
      return fail(PX_ERR_UNSUPPORTED, "temporal_k=%d exceeds the ghost width %d", o->temporal_k, l->ghost);
    if (ext(l->domain, 0) % 2)
      return fail(PX_ERR_UNSUPPORTED, "temporal blocking needs an even domain width");
  }
  int32_t nparts = 1;
  if (c) {
    if (c->nranks != l->nranks || c->rank != rank)
      return fail(PX_ERR_STATE, "communicator (rank %d of %d) does not match layout/rank",
                  c->rank, c->nranks);
  } else {
    nparts = l->nranks;
    rank = 0;
  }
  px_local_info li;
  for (int32_t i = 0; i < nparts; ++i) {
    const int32_t r = c ? rank : i;
    PX_TRY(check_rank_patch(l, r, &phi[i], "phi", &li));
    PX_TRY(check_rank_patch(l, r, &phi_scratch[i], "phi_scratch", &li));
    PX_TRY(check_patch(&rhs[i], "rhs"));
    if (!contains(rhs[i].box, li.owned)) return fail(PX_ERR_SHAPE, "rhs does not cover the slab");
    if (((uintptr_t)phi[i].data / 8 + 0) % 2 != ((uintptr_t)phi_scratch[i].data / 8) % 2)
      return fail(PX_ERR_ALIGN, "phi and phi_scratch have different 16-byte phases");
  }
  cudaStream_t s = (cudaStream_t)stream;
  PlanKey key;
  key.layout_gen = layout_generation(l);
  key.comm = c;
  key.p2p_gen = c ? c->p2p.gen : 0;
  key.rank = rank;
  key.stencil = p->stencil;
  key.nsweeps = o->nsweeps;
  key.norm_every = o->norm_every;
  key.k = o->temporal_k > 1 ? o->temporal_k : 1;
  key.nparts = nparts;
  key.h = p->h;
  key.lambda = p->lambda;
  for (int32_t i = 0; i < nparts; ++i) {
    key.ptrs.push_back(phi[i].data);
    key.ptrs.push_back(phi_scratch[i].data);
    key.ptrs.push_back(rhs[i].data);
    for (int d = 0; d < 2; ++d) {
      key.rhs_geom.push_back(rhs[i].box.lo.c[d]);
      key.rhs_geom.push_back(rhs[i].box.hi.c[d]);
    }
    key.rhs_geom.push_back(rhs[i].ld);
  }
  key.stream = s;
  Plan* plan = nullptr;
  for (auto& pl : plans())
    if (pl->key == key) plan = pl.get();
  if (!plan) {
    std::unique_ptr<Plan> np(new Plan());
    np->key = key;
    np->n_entries = count_entries(o->nsweeps, o->norm_every);
    const int32_t ne = std::max(np->n_entries, 1);
    int64_t maxblocks = 0;
    for (int32_t i = 0; i < nparts; ++i) {
      px_local_info lj;
      PX_TRY(local_info(l, c ? rank : i, &lj));
      // split launches add at most 2 extra partial rows of blocks
      maxblocks += stream_blocks(ext(lj.owned, 0), ext(lj.owned, 1), 1) + 2 * stream_blocks(ext(lj.owned, 0), 1, 1);
    }
    np->ws_stride = std::max<int64_t>(2 + 2 * maxblocks, 4 * 1024);  // >= 4 x persistent grid
    np->ws_len = np->ws_stride * (o->temporal_k > 1 ? o->temporal_k : 1);
    PX_TRY(cuda_check(cudaMalloc(&np->d_max, ne * sizeof(double)), "cudaMalloc ring"));
    PX_TRY(cuda_check(cudaMalloc(&np->d_sum, ne * sizeof(double)), "cudaMalloc ring"));
    PX_TRY(cuda_check(cudaMalloc(&np->d_ws, np->ws_len * sizeof(double)), "cudaMalloc ws"));
    PX_TRY(cuda_check(cudaMemset(np->d_ws, 0, np->ws_len * sizeof(double)), "memset ws"));
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fill before any user-stream work
    {  // workspace of the shared-memory-resident solve (allocated here: not during graph capture)
      px_local_info l0;
      PX_TRY(local_info(l, c ? rank : 0, &l0));
      int rg = 0, rm = 0;
      size_t rsm = 0;
      if (!c && nparts == 1 && l->nranks == 1 && o->temporal_k <= 1 && o->nsweeps > 0 &&
          resident_plan(ext(l0.owned, 0), ext(l0.owned, 1), &rg, &rm, &rsm))
        PX_TRY(cuda_check(cudaMalloc(&np->d_res, resident_ws_doubles(ext(l0.owned, 0), rg, np->n_entries) *
                                                     sizeof(double)),
                          "cudaMalloc resident workspace"));
    }
    PX_TRY(cuda_check(cudaEventCreateWithFlags(&np->ev_bnd, cudaEventDisableTiming), "event"));
    PX_TRY(cuda_check(cudaEventCreateWithFlags(&np->ev_comm, cudaEventDisableTiming), "event"));
    plan = np.get();
    plans().push_back(std::move(np));
  }
  plan_touch(plans(), plan);
  SolveCtx x{l, c, rank, p, o, nparts, phi, phi_scratch, rhs, plan, s};
  if (o->use_graph && !s) return fail(PX_ERR_ARG, "use_graph needs a non-default stream");
  take_noted_kernels();
  if (o->use_graph) {
    if (!plan->exec) {
      const int64_t before = px_kernel_launch_count();
      PX_TRY(cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture"));
      px_status st = enqueue_solve(x);
      plan->kernels = take_noted_kernels();
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      if (st != PX_OK) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();  // do not leave a capture-time error for the next call
        return st;
      }
      PX_TRY(cuda_check(ce, "end capture"));
      plan->launches_per_run = px_kernel_launch_count() - before;
      count_launches(-plan->launches_per_run);
      ce = cudaGraphInstantiate(&plan->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) {
        plan->exec = nullptr;
        cudaGetLastError();
      }
      PX_TRY(cuda_check(ce, "graph instantiate"));
    }
    PX_TRY(cuda_check(cudaGraphLaunch(plan->exec, s), "graph launch"));
    count_launches(plan->launches_per_run);
  } else {
    PX_TRY(enqueue_solve(x));
    plan->kernels = take_noted_kernels();
  }
  tl_last_kernels = plan->kernels;
  // φ^N is in the buffer the last pass wrote: one buffer swap per sweep, or
  // per temporal-blocking pass of K sweeps plus one per remaining sweep.
  const int32_t K = o->temporal_k > 1 ? o->temporal_k : 1;
  const int32_t nswaps = K > 1 ? o->nsweeps / K + o->nsweeps % K : o->nsweeps;
  *plan_out = plan;
  *odd_out = (nswaps % 2) == 1;
  *nparts_out = nparts;
  return PX_OK;
}

extern "C" {

px_status px_solve(const px_layout* l, px_comm* c, int32_t rank, const px_relax_params* p,
                   const px_solve_opts* o, px_patch* phi, px_patch* phi_scratch,
                   const px_patch* rhs, double* h_norms, int32_t cap, int32_t* n_written,
                   int32_t* in_scratch, void* stream) {
  if (cap < 0 || (cap > 0 && !h_norms)) return fail(PX_ERR_ARG, "bad norm output");
  NvtxRange r_solve("protox/px_solve");
  Plan* plan = nullptr;
  bool odd = false;
  int32_t nparts = 1;
  PX_TRY(solve_enqueue(l, c, rank, p, o, phi, phi_scratch, rhs, stream, &plan, &odd, &nparts));
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t ne = plan->n_entries;
  std::vector<double> hm(ne), hs(ne);
  if (ne > 0) {
    PX_TRY(cuda_check(cudaMemcpyAsync(hm.data(), plan->d_max, ne * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H norms"));
    PX_TRY(cuda_check(cudaMemcpyAsync(hs.data(), plan->d_sum, ne * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H norms"));
  }
  if (odd && !in_scratch) {
    for (int32_t i = 0; i < nparts; ++i) {
      const px_patch& a = phi_scratch[i];
      const px_patch& b = phi[i];
      PX_TRY(cuda_check(cudaMemcpy2DAsync(b.data, b.ld * sizeof(double), a.data, a.ld * sizeof(double),
                                          ext(a.box, 0) * sizeof(double), ext(a.box, 1),
                                          cudaMemcpyDeviceToDevice, s), "copy result"));
    }
  }
  PX_TRY(cuda_check(cudaStreamSynchronize(s), "solve"));
  if (c && c->p2p.enabled) {  // a peer wait that gave up (lost or stalled peer): report, do not hang
    unsigned long long to = 0;
    PX_TRY(cuda_check(cudaMemcpy(&to, c->p2p.ctl + CTL_TIMEOUT, sizeof to, cudaMemcpyDeviceToHost), "timeout flag"));
    if (to) return fail(PX_ERR_STATE, "peer-memory halo wait timed out (%llu waits): a peer is lost or stalled", to);
  }
  if (c && c->nccl) {
    ncclResult_t ar;
    ncclCommGetAsyncError(c->nccl, &ar);
    PX_TRY(nccl_check(ar, "NCCL async error"));
  }
  const int32_t nw = std::min(ne, cap);
  for (int32_t j = 0; j < nw; ++j) {
    h_norms[2 * j] = hm[j];
    h_norms[2 * j + 1] = hs[j];
  }
  if (n_written) *n_written = nw;
  if (in_scratch) *in_scratch = odd ? 1 : 0;
  return PX_OK;
}

px_status px_solve_async(const px_layout* l, px_comm* c, int32_t rank, const px_relax_params* p,
                         const px_solve_opts* o, px_patch* phi, px_patch* phi_scratch, const px_patch* rhs,
                         double* d_norms, int32_t cap, int32_t* n_written, int32_t* in_scratch, void* stream) {
  if (cap < 0 || (cap > 0 && !d_norms)) return fail(PX_ERR_ARG, "bad norm output");
  NvtxRange r_solve("protox/px_solve_async");
  Plan* plan = nullptr;
  bool odd = false;
  int32_t nparts = 1;
  PX_TRY(solve_enqueue(l, c, rank, p, o, phi, phi_scratch, rhs, stream, &plan, &odd, &nparts));
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t nw = std::min(plan->n_entries, cap);
  if (nw > 0) {  // the norm ring interleaved into d_norms (max, Σ) per entry, stream-ordered
    PX_TRY(cuda_check(cudaMemcpy2DAsync(d_norms, 2 * sizeof(double), plan->d_max, sizeof(double), sizeof(double), nw,
                                        cudaMemcpyDeviceToDevice, s), "norms"));
    PX_TRY(cuda_check(cudaMemcpy2DAsync(d_norms + 1, 2 * sizeof(double), plan->d_sum, sizeof(double), sizeof(double),
                                        nw, cudaMemcpyDeviceToDevice, s), "norms"));
  }
  if (odd && !in_scratch) {
    for (int32_t i = 0; i < nparts; ++i) {
      const px_patch& a = phi_scratch[i];
      const px_patch& b = phi[i];
      PX_TRY(cuda_check(cudaMemcpy2DAsync(b.data, b.ld * sizeof(double), a.data, a.ld * sizeof(double),
                                          ext(a.box, 0) * sizeof(double), ext(a.box, 1),
                                          cudaMemcpyDeviceToDevice, s), "copy result"));
    }
  }
  if (n_written) *n_written = nw;
  if (in_scratch) *in_scratch = odd ? 1 : 0;
  return PX_OK;
}

// ----------------------------------------------------------- host e2e path
struct HostBufs {
  uint64_t gen = 0;
  double *phi = nullptr, *scr = nullptr, *rhs = nullptr;
  int64_t elems = 0;
  cudaStream_t s = nullptr;
  void release() {
    if (phi) cudaFree(phi);
    if (scr) cudaFree(scr);
    if (rhs) cudaFree(rhs);
    phi = scr = rhs = nullptr;
    elems = 0;
    gen = 0;
  }
};
static HostBufs g_host;

px_status px_solve_host(const px_layout* l, const px_relax_params* p, const px_solve_opts* o,
                        const double* h_phi0, const double* h_rho, double* h_phi_out,
                        double* h_norms, int32_t cap, int32_t* n_written, void* stream) {
  if (!l || !p || !o || !h_phi0 || !h_rho || !h_phi_out) return fail(PX_ERR_ARG, "null argument");
  if (l->nranks != 1) return fail(PX_ERR_UNSUPPORTED, "px_solve_host needs a single-rank layout");
  px_local_info li;
  PX_TRY(local_info(l, 0, &li));
  if (g_host.elems != li.alloc_elems || g_host.gen != layout_generation(l)) {
    g_host.release();
    size_t b = li.alloc_elems * sizeof(double);
    PX_TRY(cuda_check(cudaMalloc(&g_host.phi, b), "cudaMalloc"));
    PX_TRY(cuda_check(cudaMalloc(&g_host.scr, b), "cudaMalloc"));
    PX_TRY(cuda_check(cudaMalloc(&g_host.rhs, b), "cudaMalloc"));
    PX_TRY(cuda_check(cudaMemset(g_host.phi, 0, b), "memset"));
    PX_TRY(cuda_check(cudaMemset(g_host.scr, 0, b), "memset"));
    PX_TRY(cuda_check(cudaMemset(g_host.rhs, 0, b), "memset"));
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fill before any user-stream work
    g_host.elems = li.alloc_elems;
    g_host.gen = layout_generation(l);
  }
  px_patch ph, sc, rh;
  PX_TRY(px_layout_patch(l, 0, g_host.phi, &ph));
  PX_TRY(px_layout_patch(l, 0, g_host.scr, &sc));
  PX_TRY(px_layout_patch(l, 0, g_host.rhs, &rh));
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t n0 = ext(li.owned, 0), n1 = ext(li.owned, 1);
  const size_t w = n0 * sizeof(double), dp = li.ld * sizeof(double);
  PX_TRY(cuda_check(cudaMemcpy2DAsync(at(ph, li.owned.lo.c[0], li.owned.lo.c[1]), dp, h_phi0, w, w,
                                      n1, cudaMemcpyHostToDevice, s), "H2D phi"));
  PX_TRY(cuda_check(cudaMemcpy2DAsync(at(rh, li.owned.lo.c[0], li.owned.lo.c[1]), dp, h_rho, w, w,
                                      n1, cudaMemcpyHostToDevice, s), "H2D rho"));
  if (o->temporal_k > 1) PX_TRY(launch_fill_ghosts(l, 0, rh, s));  // ρ ghosts for the halo levels
  int32_t in_scr = 0;
  PX_TRY(px_solve(l, nullptr, 0, p, o, &ph, &sc, &rh, h_norms, cap, n_written, &in_scr, stream));
  const px_patch& res = in_scr ? sc : ph;
  PX_TRY(cuda_check(cudaMemcpy2DAsync(h_phi_out, w, at(res, li.owned.lo.c[0], li.owned.lo.c[1]), dp, w,
                                      n1, cudaMemcpyDeviceToHost, s), "D2H phi"));
  return cuda_check(cudaStreamSynchronize(s), "solve_host");
}

// Pipelined host path: NSET device buffer sets; the copy-in stream, the
// compute stream and the copy-out stream are ordered by events so that the
// H2D of problem i+1 and the D2H of problem i-1 run on the copy engines
// while problem i is being solved.  Three sets let the H2D of problem i+1
// and the D2H of problem i-1 run at the same time (full-duplex PCIe).
constexpr int NSET = 3;
struct BatchBufs {
  uint64_t gen = 0;
  int64_t elems = 0;
  int32_t ne = 0;
  double* d[NSET][3] = {};  // phi, scr, rhs per set
  double* h_ring[NSET] = {};  // pinned (max, sum) staging per set
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in[NSET] = {}, ev_done[NSET] = {}, ev_free[NSET] = {};
  void release_fields() {
    for (auto& set : d)
      for (auto& q : set) {
        if (q) cudaFree(q);
        q = nullptr;
      }
    for (auto& h : h_ring) {
      if (h) cudaFreeHost(h);
      h = nullptr;
    }
    elems = 0;
    gen = 0;
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
};
static BatchBufs g_batch;

px_status px_solve_host_batch(const px_layout* l, const px_relax_params* p, const px_solve_opts* o,
                              int32_t nprob, const double* const* h_phi0, const double* const* h_rho,
                              double* const* h_phi_out, double* h_norms, int32_t cap, int32_t* n_written,
                              void* stream) {
  if (!l || !p || !o || !h_rho || !h_phi_out) return fail(PX_ERR_ARG, "null argument");
  if (nprob < 0) return fail(PX_ERR_ARG, "nprob must be >= 0");
  if (cap < 0 || (cap > 0 && !h_norms)) return fail(PX_ERR_ARG, "bad norm output");
  if (l->nranks != 1) return fail(PX_ERR_UNSUPPORTED, "px_solve_host_batch needs a single-rank layout");
  if (!stream) return fail(PX_ERR_ARG, "px_solve_host_batch needs a non-default compute stream");
  for (int32_t i = 0; i < nprob; ++i)
    if (!h_rho[i] || !h_phi_out[i]) return fail(PX_ERR_ARG, "null host buffer for problem %d", i);
  if (nprob == 0) return PX_OK;
  px_local_info li;
  PX_TRY(local_info(l, 0, &li));
  BatchBufs& B = g_batch;
  const int32_t ne = count_entries(o->nsweeps, o->norm_every);
  if (!B.s_in) {
    PX_TRY(cuda_check(cudaStreamCreateWithFlags(&B.s_in, cudaStreamNonBlocking), "stream"));
    PX_TRY(cuda_check(cudaStreamCreateWithFlags(&B.s_out, cudaStreamNonBlocking), "stream"));
    PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_start, cudaEventDisableTiming), "event"));
    for (int b = 0; b < NSET; ++b) {
      PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_in[b], cudaEventDisableTiming), "event"));
      PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_done[b], cudaEventDisableTiming), "event"));
      PX_TRY(cuda_check(cudaEventCreateWithFlags(&B.ev_free[b], cudaEventDisableTiming), "event"));
    }
  }
  if (B.elems != li.alloc_elems || B.gen != layout_generation(l) || B.ne < ne) {
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "sync before realloc"));
    B.release_fields();
    const size_t b = li.alloc_elems * sizeof(double);
    for (auto& set : B.d)
      for (auto& q : set) {
        PX_TRY(cuda_check(cudaMalloc(&q, b), "cudaMalloc"));
        PX_TRY(cuda_check(cudaMemset(q, 0, b), "memset"));
      }
    PX_TRY(cuda_check(cudaDeviceSynchronize(), "init zero-fill"));  // the legacy-stream fill before any user-stream work
    for (auto& h : B.h_ring)
      PX_TRY(cuda_check(cudaMallocHost(&h, 2 * (size_t)std::max(ne, 1) * sizeof(double)), "cudaMallocHost"));
    B.elems = li.alloc_elems;
    B.gen = layout_generation(l);
    B.ne = std::max(ne, 1);
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t n0 = ext(li.owned, 0), n1 = ext(li.owned, 1);
  const size_t w = n0 * sizeof(double), dp = li.ld * sizeof(double);
  const size_t alloc_bytes = li.alloc_elems * sizeof(double);
  // the copy streams start after the work already on the compute stream
  PX_TRY(cuda_check(cudaEventRecord(B.ev_start, s), "event"));
  PX_TRY(cuda_check(cudaStreamWaitEvent(B.s_in, B.ev_start, 0), "wait"));
  PX_TRY(cuda_check(cudaStreamWaitEvent(B.s_out, B.ev_start, 0), "wait"));
  bool pending[NSET] = {};
  int32_t pend_i[NSET] = {};
  auto harvest = [&](int b) -> px_status {  // host side of problem pend_i[b]: norms out of staging
    if (!pending[b]) return PX_OK;
    PX_TRY(cuda_check(cudaEventSynchronize(B.ev_free[b]), "batch D2H"));
    const int32_t i = pend_i[b];
    const int32_t nw = std::min(ne, cap);
    for (int32_t j = 0; j < nw; ++j) {
      h_norms[(size_t)i * 2 * cap + 2 * j] = B.h_ring[b][j];
      h_norms[(size_t)i * 2 * cap + 2 * j + 1] = B.h_ring[b][B.ne + j];
    }
    if (n_written) n_written[i] = nw;
    pending[b] = false;
    return PX_OK;
  };
  for (int32_t i = 0; i < nprob; ++i) {
    const int b = i % NSET;
    PX_TRY(harvest(b));  // problem i-NSET has left set b (host wait: its D2H is done)
    px_patch ph, sc, rh;
    PX_TRY(px_layout_patch(l, 0, B.d[b][0], &ph));
    PX_TRY(px_layout_patch(l, 0, B.d[b][1], &sc));
    PX_TRY(px_layout_patch(l, 0, B.d[b][2], &rh));
    // ---- copy in (s_in)
    if (h_phi0 && h_phi0[i]) {
      PX_TRY(cuda_check(cudaMemcpy2DAsync(at(ph, li.owned.lo.c[0], li.owned.lo.c[1]), dp, h_phi0[i], w, w, n1,
                                          cudaMemcpyHostToDevice, B.s_in), "H2D phi"));
    } else {
      PX_TRY(cuda_check(cudaMemsetAsync(B.d[b][0], 0, alloc_bytes, B.s_in), "zero phi"));
    }
    PX_TRY(cuda_check(cudaMemcpy2DAsync(at(rh, li.owned.lo.c[0], li.owned.lo.c[1]), dp, h_rho[i], w, w, n1,
                                        cudaMemcpyHostToDevice, B.s_in), "H2D rho"));
    PX_TRY(cuda_check(cudaEventRecord(B.ev_in[b], B.s_in), "event"));
    // ---- solve (compute stream)
    PX_TRY(cuda_check(cudaStreamWaitEvent(s, B.ev_in[b], 0), "wait"));
    if (o->temporal_k > 1) PX_TRY(launch_fill_ghosts(l, 0, rh, s));
    Plan* plan = nullptr;
    bool odd = false;
    int32_t nparts = 1;
    PX_TRY(solve_enqueue(l, nullptr, 0, p, o, &ph, &sc, &rh, stream, &plan, &odd, &nparts));
    PX_TRY(cuda_check(cudaEventRecord(B.ev_done[b], s), "event"));
    // ---- copy out (s_out)
    PX_TRY(cuda_check(cudaStreamWaitEvent(B.s_out, B.ev_done[b], 0), "wait"));
    const px_patch& res = odd ? sc : ph;
    PX_TRY(cuda_check(cudaMemcpy2DAsync(h_phi_out[i], w, at(res, li.owned.lo.c[0], li.owned.lo.c[1]), dp, w, n1,
                                        cudaMemcpyDeviceToHost, B.s_out), "D2H phi"));
    if (plan->n_entries > 0) {
      PX_TRY(cuda_check(cudaMemcpyAsync(B.h_ring[b], plan->d_max, plan->n_entries * sizeof(double),
                                        cudaMemcpyDeviceToHost, B.s_out), "D2H norms"));
      PX_TRY(cuda_check(cudaMemcpyAsync(B.h_ring[b] + B.ne, plan->d_sum, plan->n_entries * sizeof(double),
                                        cudaMemcpyDeviceToHost, B.s_out), "D2H norms"));
    }
    PX_TRY(cuda_check(cudaEventRecord(B.ev_free[b], B.s_out), "event"));
    pending[b] = true;
    pend_i[b] = i;
  }
  // join: the compute stream ends after the last copy out
  for (int b = 0; b < NSET; ++b)
    if (pending[b]) PX_TRY(cuda_check(cudaStreamWaitEvent(s, B.ev_free[b], 0), "wait"));
  for (int b = 0; b < NSET; ++b) PX_TRY(harvest(b));
  return cuda_check(cudaStreamSynchronize(s), "solve_host_batch");
}

const char* px_last_solve_kernels(void) { return tl_last_kernels.c_str(); }

void px_release_cached(void) {
  px_mg_release();
  plans().clear();
  g_host.release();
  g_batch.release();
}

}  // extern "C"
