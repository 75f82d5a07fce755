// px_internal.h -- internal declarations shared by the libprotox sources.
// Nothing here is part of the ABI (include/protox.h is).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "protox.h"

namespace px {

// ---- errors --------------------------------------------------------------
px_status fail(px_status s, const char* fmt, ...);
void clear_error();

#define PX_TRY(expr)                   \
  do {                                 \
    px_status _s = (expr);             \
    if (_s != PX_OK) return _s;        \
  } while (0)

// ---- geometry helpers ------------------------------------------------------
inline int32_t ext(const px_box& b, int d) {
  return b.lo.c[d] > b.hi.c[d] ? 0 : b.hi.c[d] - b.lo.c[d] + 1;
}
inline bool empty(const px_box& b) { return b.lo.c[0] > b.hi.c[0] || b.lo.c[1] > b.hi.c[1]; }
inline bool contains(const px_box& outer, const px_box& inner) {
  if (empty(inner)) return true;
  return inner.lo.c[0] >= outer.lo.c[0] && inner.lo.c[1] >= outer.lo.c[1] &&
         inner.hi.c[0] <= outer.hi.c[0] && inner.hi.c[1] <= outer.hi.c[1];
}
inline px_box mkbox(int32_t x0, int32_t y0, int32_t x1, int32_t y1) {
  px_box b;
  b.lo.c[0] = x0;
  b.lo.c[1] = y0;
  b.hi.c[0] = x1;
  b.hi.c[1] = y1;
  return b;
}
inline px_box grow(const px_box& b, int32_t r) {
  return mkbox(b.lo.c[0] - r, b.lo.c[1] - r, b.hi.c[0] + r, b.hi.c[1] + r);
}
// pointer to cell (x, y) of a patch
inline double* at(const px_patch& p, int32_t x, int32_t y) {
  return p.data + (int64_t)(x - p.box.lo.c[0]) + (int64_t)(y - p.box.lo.c[1]) * p.ld;
}

}  // namespace px

// the opaque layout (defined here so the solve driver can read it)
struct px_layout {
  px_box domain;
  px_point box_size;
  int32_t ghost;
  px_bc bc;
  int32_t nranks;
  int32_t nbx, nby;                 // box grid
  std::vector<int32_t> row_lo;      // rank r owns box-rows [row_lo[r], row_lo[r+1])
  int64_t ld;                       // common row pitch of every rank's patch
  uint64_t gen;                     // unique id (plan-cache key)
};

namespace px {

// ---- kernel-side descriptors ----------------------------------------------
enum : int { MODE_RELAX = 0, MODE_RESID = 1, MODE_APPLY = 2, MODE_MRHS = 3 };
enum : int { GH_NONE = 0, GH_WRAP = 1, GH_REFLECT = 2 };

// Which ghost images a relax sweep writes along with each owned cell
// (fused exchange).  For dimension d, side 0 = lo, 1 = hi:
// a cell within `g` of that face also writes its image there.
struct GhostSpec {
  int32_t mode[2][2];   // [dim][side]
  int32_t n[2];         // extent of the owned box (the image shift for WRAP)
  int32_t o[2];         // region.lo - owned.lo
  int32_t g;            // depth written (0: no images)
};

// Norm reduction slot: `expected` blocks over one or more launches write
// partials[offset + block]; the last one to finish reduces them in fixed
// order into out[0] (max|r|) and out[1] (Σr²) and re-zeroes *counter.
struct NormSlot {
  double* out_max;      // null: no norms
  double* out_sum;
  double* partials;
  unsigned int* counter;
  int32_t offset;
  int32_t expected;
};

// Fused halo push over peer memory (px_solve P2P mode).  ONE
// k_bulk launch per sweep over the whole owned slab.  Its work items of the
// first and last row chunk run first (every one is some CTA's first item); at
// their end they store rows [0,g) and [ny-g,ny) of φ' (with their x images,
// so corners are right) straight into the lo / hi neighbour's ghost rows
// (16-byte stores over NVLink).  The NEXT sweep's kernel publishes them: its
// CTA 0 counts one arrival per side on the neighbours' counters (relaxed,
// system scope -- the pushing grid has completed, so its stores are
// performed), and its boundary CTAs wait until their own counter reaches
// base + wcount (acquire) before any thread reads a ghost row.  Counters never
// reset: the base (*epoch) advances by each solve's own arrivals, so solves
// may differ in N.  Side 0 = lo (rank below), 1 = hi.
struct PushSpec {
  double* rdst[2];                 // neighbour's ghost-row cell matching region.lo.x (null: no push)
  unsigned long long* rflag[2];    // neighbour's arrival counter to bump
  unsigned long long* wflag[2];    // own arrival counter to wait on (null: no wait)
  const unsigned long long* epoch; // own arrival base (arrivals of all earlier solves)
  unsigned long long wcount;       // arrivals needed within this solve, per side
  int32_t g;                       // rows pushed per side (the ghost width)
  int32_t on;                      // any push / wait: boundary chunks are scheduled first
  int32_t rel;                     // publish the previous sweep's pushes (CTA 0, at kernel start)
  int32_t xg, xn0, xm0, xm1;       // x images of pushed cells (corners): depth, owned width, lo/hi modes
  unsigned long long* err;         // own timed-out-wait counter (px_spin_until)
};

struct StreamLaunch {
  const double* src;  // φ_in at region.lo
  const double* rhs;  // rhs at region.lo (may be null in APPLY mode)
  double* dst;        // output at region.lo
  int64_t ld_src, ld_rhs, ld_dst;
  int32_t nx, ny;     // region extent
  int32_t phase;      // 1 if region.lo is not 16-byte aligned (pairs start at column -1)
  int32_t src_x0, src_x1;  // readable column range of src relative to region.lo
  double scale, lambda;
  GhostSpec gs;
  NormSlot norms;     // norms.out_max == null: none
  PushSpec ps;        // fused halo push / wait (k_bulk only)
  int32_t pdl;        // launch as a programmatic dependent of the previous kernel (k_bulk only)
  int32_t wrap;       // k_bulk only: the region is a whole periodic single-rank domain -- φ rows -1 / ny
                      // and columns -1 / nx are read from rows ny-1 / 0 and columns nx-1 / 0 (the
                      // ghost ring is not read, so no images or ghost fill are needed per sweep)
};

// Extra launch state of a temporal-blocking pass (px_tb.cu).
struct TbLaunch {
  NormSlot lvl[4];   // norms of the residual computed at level t (iterate base+t-1)
  int32_t fix[2][2]; // FIXED faces: ghost cells there keep their level-0 value
  int32_t refl[2][2]; // DIRICHLET_CC faces: the first ghost column / row of every
                      // level is re-derived by odd reflection (wide kernel only)
};
int32_t tb_blocks(int K, const StreamLaunch& a);
px_status launch_tb(int stencil, int K, const StreamLaunch& a, const TbLaunch& x, cudaStream_t s);

// A whole single-box solve in one launch (px_smallbox.cu, K9).
struct SmallBox {
  const double* phi_in;   // cell (0,0) of the input patch
  double* phi_out;        // cell (0,0) of the output patch (may equal phi_in)
  const double* rhs;      // cell (0,0) of the rhs patch
  int64_t ld_in, ld_out, ld_rhs;
  int nx, ny, g;
  int bc;
  int stencil;
  double scale, lambda;
  int nsweeps, every;     // norms of φ^s for s % every == 0 (every <= 0: none)
  int final_norm;         // record the residual of φ^N
  double* d_max;          // norm ring
  double* d_sum;
};
bool smallbox_fits(int nx, int ny);
// the same solve on a cluster of 8 CTAs with DSMEM halo exchange (px_cluster.cu)
bool cluster_box_eligible(const SmallBox& b);  // incl. its norm partials
px_status launch_cluster_box(const SmallBox& b, cudaStream_t s);

// All sweeps of a single-rank solve in one cooperative launch (px_kernels.cu).
struct PersistLaunch {
  StreamLaunch a0, a1;     // RELAX A -> B (even sweeps), B -> A (odd sweeps)
  StreamLaunch r0, r1;     // RESID on A, on B (final residual)
  int nsweeps, every, final_norm;
  double* d_max;
  double* d_sum;
  double* partials;        // 2 x 2 x grid doubles
  int rows, gx, gy;        // tile grid (SW_COLS columns x rows)
};
int32_t persist_rows(int32_t nx, int32_t ny, int32_t grid);

// All sweeps of a single-rank solve with the iterate resident in shared
// memory (px_resident.cu): CTA c of G owns rows [c*ny/G, (c+1)*ny/G) and
// exchanges only its first and last row with its two neighbours per sweep
// through L2 (flag handshake, no grid barrier).
struct ResidentLaunch {
  const double* phi_in;   // cell (0,0) of φ^0 (ghost ring filled)
  double* phi_out;        // cell (0,0) of the buffer that receives φ^N (+ ghost ring)
  const double* rhs;      // cell (0,0) of the right-hand side
  int64_t ld_in, ld_out, ld_rhs;
  int nx, ny, rmax;       // extent; max rows per CTA
  int xmode[2], ymode[2]; // GH_WRAP / GH_REFLECT / GH_NONE (fixed ghosts)
  double scale, lambda;
  int nsweeps, every, final_norm, n_entries;
  double* d_max;
  double* d_sum;
  double* ws;             // resident_ws_doubles(...) doubles, zero not required
  int unroll;             // set by launch_resident: unrolled column walk (rmax <= 7)
};
size_t resident_ws_doubles(int nx, int grid, int n_entries);
// CTAs and dynamic shared memory of the resident kernel for an nx x ny
// problem; false if it does not fit (or nx is odd).
bool resident_plan(int nx, int ny, int* grid, int* rmax, size_t* smem);
px_status launch_resident(int stencil, const ResidentLaunch& r, int grid, size_t smem, cudaStream_t s);
int32_t stream_launch_blocks_ldg(const StreamLaunch& a);
px_status launch_stream_ldg(int mode, int stencil, const StreamLaunch& a, cudaStream_t s);
// arrivals a push-mode k_bulk launch of `a` counts per side (1); 0 if the
// launch cannot push (not bulk-eligible, or its boundary items would not all
// be first items of its CTAs)
int32_t bulk_push_arrivals(const StreamLaunch& a);
// publish the last sweep's pushes (ps.rel), then wait (on the device) until
// both own counters of `ps` reach base + wcount
px_status launch_wait(const PushSpec& ps, cudaStream_t s);
// copy the full padded rows [0,g) / [ny-g,ny) of a slab (x ghosts included)
// into the neighbours' ghost rows of both their buffers, then count
// PX_PUSH_INIT_CTAS arrivals per side (the exchange of φ^0 in push mode)
constexpr int PX_PUSH_INIT_CTAS = 32;
struct PushInit {
  const double* src_lo;            // own padded row 0 (x = -g)
  const double* src_hi;            // own padded row ny-g
  double* dst[2][2];               // [side][buffer]: neighbour's ghost row start (x = -g)
  unsigned long long* rflag[2];
  int64_t ld;
  int32_t row_len, g;
};
px_status launch_push_init(const PushInit& pi, cudaStream_t s);
// Norm all-reduce over peer memory (one CTA): every rank publishes its ring
// in its mailbox, counts an arrival on every peer, reads all mailboxes in
// rank order (max over the u64 bit patterns, Σ in rank order: every rank gets
// the same bits), then counts a "done" on every peer before its mailbox may
// be reused.
constexpr int PX_PEER_MAX = 16;
constexpr int PX_MBOX_ENTRIES = 2048;
struct PeerAllreduce {
  double* d_max;
  double* d_sum;
  int32_t n, nranks, rank;
  double* mbox_own;                          // 2 * PX_MBOX_ENTRIES doubles
  const double* mbox[PX_PEER_MAX];           // every rank's mailbox (own included)
  unsigned long long* arrive[PX_PEER_MAX];   // every rank's arrive counter
  unsigned long long* done[PX_PEER_MAX];     // every rank's done counter
  unsigned long long* own_arrive;
  unsigned long long* own_done;
  unsigned long long* round;                 // own round counter
  unsigned long long* err;                   // own timed-out-wait counter (px_spin_until)
};
px_status launch_peer_allreduce(const PeerAllreduce& ar, cudaStream_t s);
px_status launch_epoch_bump(unsigned long long* epoch, unsigned long long per_solve, cudaStream_t s);
int32_t persist_grid();
px_status launch_persist(int stencil, const PersistLaunch& p, int grid, cudaStream_t s);
px_status launch_smallbox(const SmallBox& b, cudaStream_t s);

// upper bound of the thread blocks a relax/residual launch over a region uses
constexpr int32_t BULK_MAX_GRID = 512;
int32_t stream_blocks(int32_t nx, int32_t ny, int32_t phase);
// blocks the launch of `a` will actually use (norm slot accounting)
int32_t launch_blocks(int mode, const StreamLaunch& a);
// the TMA bulk-copy kernel (px_bulk.cu)
bool bulk_eligible(int mode, const StreamLaunch& a);
int32_t bulk_blocks(const StreamLaunch& a);
px_status launch_bulk(int mode, int stencil, const StreamLaunch& a, cudaStream_t s);
// launchers (px_kernels.cu); return PX_ERR_CUDA on launch failure
px_status launch_stream(int mode, int stencil, const StreamLaunch& a, cudaStream_t s);
px_status launch_fill_ghosts(const px_layout* l, int32_t rank, const px_patch& p, cudaStream_t s);
// ghost fill of an nx x ny region at o (cell (0,0)), depth g: x faces by mode
// mx for rows [0,ny), then y faces by my_lo / my_hi over the full padded rows
// (corners by the product rule)
px_status launch_fill_ghosts_raw(double* o, int64_t ld, int nx, int ny, int g, int mx, int my_lo, int my_hi,
                                 cudaStream_t s);
px_status launch_init_field(const px_layout* l, int32_t rank, const px_patch& p, int kind,
                            uint64_t seed, int k, int lw, cudaStream_t s);
px_status cuda_check(cudaError_t e, const char* what);
void count_launches(int64_t n);
// sweep-kernel names of the current solve (px_last_solve_kernels)
void note_kernel(const char* name);
std::string take_noted_kernels();

// ---- bounded plan caches (px_solve, px_mg_solve) --------------------------
// A cached plan owns device workspace, events and a CUDA graph exec.  The
// caches keep the most recently used plans only (PROTOX_PLAN_CACHE, default
// 32); a plan is also dropped when its layout is destroyed.
int plan_cache_cap();
// Move `p` to the most-recently-used end of `v` and evict the least recently
// used plans beyond the cap (after a device synchronisation: an evicted plan's
// graph may still be in flight).
template <class T>
void plan_touch(std::vector<std::unique_ptr<T>>& v, T* p) {
  auto it = std::find_if(v.begin(), v.end(), [p](const std::unique_ptr<T>& q) { return q.get() == p; });
  if (it != v.end() && it + 1 != v.end()) std::rotate(it, it + 1, v.end());
  const size_t cap = (size_t)plan_cache_cap();
  if (v.size() > cap) {
    cudaDeviceSynchronize();
    v.erase(v.begin(), v.begin() + (v.size() - cap));
  }
}
void drop_layout_plans(uint64_t layout_gen);     // px_solve.cu (all caches)
void mg_drop_layout_plans(uint64_t layout_gen);  // px_mg.cu

// communicator accessors (px_solve.cu) for the 3D slab solve (px3d.cu)
void* comm_nccl(const px_comm* c);  // ncclComm_t
int32_t comm_nranks(const px_comm* c);
int32_t comm_rank(const px_comm* c);
bool comm_self_exchange(const px_comm* c);
void release3_for_comm(const px_comm* c);  // px3d.cu

// validation helpers (px_host.cpp)
px_status check_patch(const px_patch* p, const char* name);
px_status local_info(const px_layout* l, int32_t rank, px_local_info* out);
px_status make_stream_launch(int mode, int stencil, double scale, double lambda,
                             const px_patch* src, const px_patch* rhs, px_patch* dst,
                             px_box region, StreamLaunch* a);
double stencil_scale(int stencil, double h);
uint64_t layout_generation(const px_layout* l);
px_status halo_plan(const px_layout* l, int32_t rank, px_halo_op ops[4], int32_t* nops, bool allow_self);

}  // namespace px
