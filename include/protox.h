/*
 * protox.h -- C ABI of libprotox, the B200-native fused 2D Poisson point-Jacobi
 * relaxation of ProtoX (arXiv 2307.07931; /root/reference/PAPER.md = "P").
 *
 * The method (figure `Proto` P:154-180): on a domain Ω split into
 * boxes with ghost cells, iterate
 *     φ ← φ + λ (Δ_h φ − ρ)                  (Eq.3)
 * where Δ_h φ = scale · S(φ), S the 5-point stencil [0,1,0;1,-4,1;0,1,0]
 * (Eq.1) with scale = 1/h², and report the residual
 * r = Δ_h φ − ρ by its max norm (Eq.7) and Σr².
 * ProtoX fuses stencil, update and norm into one loop; libprotox
 * fuses them into one memory-bound CUDA pass per sweep on sm_100a.
 *
 * Conventions (all calls):
 *  - Every call returns px_status; nothing throws or aborts across the ABI.
 *    On failure px_last_error() holds a thread-local message.
 *  - Arguments are validated before anything is enqueued; a failed call
 *    enqueues no work.
 *  - x = dimension 0 = fastest in memory; cell (x, y) of a patch is
 *    data[(x - box.lo.c[0]) + (y - box.lo.c[1]) * ld]  (layout fixed by the
 *    index arithmetic of Fig. ProtoX).
 *  - Field memory (φ, φ', ρ, norm buffers) is ALLOCATED BY THE CALLER
 *    (e.g. torch tensors) with sizes from px_layout_local / px_norm_buffer_len.
 *    The library never frees or retains caller memory beyond a call, except
 *    that px_solve's cached CUDA-graph plans capture the pointers (see there).
 *  - `px_stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Device-side calls are asynchronous on that stream unless stated.
 *  - Handles (px_layout, px_comm) are not thread-safe.
 *  - fp64 throughout.  All kernels evaluate each cell with the same
 *    expression tree as the oracle, each * and + rounded separately
 *    (DESIGN.md §3 R10), so results are bit-identical to oracle/ for any h, λ.
 */
#ifndef PROTOX_H
#define PROTOX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PX_API_VERSION 1

typedef enum {
  PX_OK = 0,
  PX_ERR_ARG = 1,         /* null pointer, bad enum, non-positive size          */
  PX_ERR_SHAPE = 2,       /* layout/patch shape mismatch     */
  PX_ERR_DOMAIN = 3,      /* point outside box, stencil reads outside src patch */
  PX_ERR_ALIGN = 4,       /* ld odd, or phi/rhs/out 16-byte phases differ       */
  PX_ERR_UNSUPPORTED = 5, /* valid request this build does not implement       */
  PX_ERR_CUDA = 6,        /* CUDA runtime error (message has the CUDA string)   */
  PX_ERR_NCCL = 7,        /* NCCL error                                          */
  PX_ERR_STATE = 8        /* handle in the wrong state                           */
} px_status;

const char* px_status_str(px_status s);
/* Thread-local detail of the last failing call on this thread, e.g.
 * "stencil domain violation at i=(63,0) tap=(1,0)".  Empty if none. */
const char* px_last_error(void);
int32_t px_api_version(void);

/* ------------------------------------------------------------------ geometry
 * Point in Z² and Box B = [lo, hi] with INCLUSIVE corners.
 * A box is empty iff lo.c[d] > hi.c[d] for some d.  Host-only, pure. */
typedef struct { int32_t c[2]; } px_point;
typedef struct { px_point lo, hi; } px_box;

int64_t px_box_size(px_box b);                    /* 0 if empty                      */
int32_t px_box_is_empty(px_box b);
px_box px_box_grow(px_box b, int32_t r);          /* lo-r, hi+r; may become empty    */
px_box px_box_intersect(px_box a, px_box b);      /* componentwise max lo / min hi   */
/* Ordinal of p in b, dimension 0 fastest: (p0-lo0) + (p1-lo1)*(hi0-lo0+1).
 * PX_ERR_DOMAIN if p is not in b (e.g. box [(-1,-1),(64,64)]: (0,0) -> 67,
 * (1,0) -> 68, (0,1) -> 133, the offsets of Fig. ProtoX). */
px_status px_box_ordinal(px_box b, px_point p, int64_t* out);

/* ---------------------------------------------------------- layout (Proto's
 * box decomposition of Ω) ------------------------------
 * The domain is split into boxes of box_size (must divide the domain).
 * Boxes are assigned to ranks as SLABS of whole box-rows along y (dimension 1,
 * the slow one), contiguous by rank.  Each rank stores its slab as ONE ghosted
 * patch; boxes are logical tiles inside it.
 *
 * Boundary conditions (DESIGN.md §3 R5):
 *   PERIODIC      Proto's model problems: ghosts wrap around Ω.
 *   DIRICHLET_CC  cell-centred homogeneous Dirichlet: the ghost at depth t
 *                 outside a face holds minus the interior cell at depth t
 *                 (x=-t <- -φ(t-1)); corners take the product of the signs.
 *   FIXED_GHOSTS  ghost cells outside Ω belong to the caller and are never
 *                 written (inter-rank ghosts are still exchanged). */
typedef enum { PX_BC_PERIODIC = 0, PX_BC_DIRICHLET_CC = 1, PX_BC_FIXED_GHOSTS = 2 } px_bc;
/* Partitions: slabs only.  SURVEY §8(b) sketches PX_PART_TILES (a 2D grid of
 * ranks); §8(e) makes tiles optional and it is not built: with ≤ 8 GPUs a
 * slab's two halo rows are contiguous (one 16-B-vector push per row inside
 * the sweep kernel), and the halo per rank at P = 8 over 16384² is 2 × 131 KB
 * per sweep, < 0.1 % of the sweep's HBM bytes. */
typedef enum { PX_PART_SLABS = 0 } px_partition;
typedef struct px_layout px_layout; /* opaque, library-owned */

/* domain: interior cells of Ω (must be non-empty; lo may be any point).
 * ghost: ghost width g, 1 <= g <= 16 and g <= box size; temporal blocking
 * with k sweeps per exchange needs g >= k.  nranks >= 1 and
 * nranks <= number of box-rows.  PX_ERR_SHAPE if box_size does not divide the
 * domain.  *out must be released with px_layout_destroy. */
px_status px_layout_create(px_box domain, px_point box_size, int32_t ghost, px_bc bc,
                           int32_t nranks, px_partition part, px_layout** out);
void px_layout_destroy(px_layout* l);
px_status px_layout_num_boxes(const px_layout* l, int32_t* n);
/* Box ibox (ordered dim-0 fastest over the box grid) and its owning rank. */
px_status px_layout_box(const px_layout* l, int32_t ibox, px_box* box, int32_t* owner);

/* Storage of one rank's slab (caller allocates alloc_elems doubles, 16-byte
 * aligned, e.g. a torch.float64 CUDA tensor):
 *   owned          interior cells of the slab
 *   alloc          owned grown by g (the ghosted box the patch covers)
 *   ld             row pitch in elements: roundup(n0 + 32, 16) (16 padding
 *                  columns on each side hold the g ghost columns)
 *   patch_offset   element offset of alloc.lo from the allocation start
 *                  (= 16 - g, so that interior column 0 sits at element 16 of
 *                  every row: 128-byte aligned rows for TMA / v2.f64 access)
 *   alloc_elems    ld * (rows of alloc)
 *   nbr_lo/nbr_hi  rank owning the cells just below/above the slab in y,
 *                  -1 at a non-periodic domain face. */
typedef struct {
  px_box owned, alloc;
  int64_t ld, patch_offset, alloc_elems;
  int32_t nbr_lo, nbr_hi;
} px_local_info;
px_status px_layout_local(const px_layout* l, int32_t rank, px_local_info* out);

/* ------------------------------------------------------------------ patches
 * A device view of caller-owned memory: data points at cell box.lo, rows
 * are ld elements apart.  (px_layout_patch builds the view of a rank's slab
 * from the allocation start.) */
typedef struct {
  double* data;
  px_box box;
  int64_t ld;
} px_patch;
px_status px_layout_patch(const px_layout* l, int32_t rank, double* alloc_base, px_patch* out);

/* Halo plan of one rank (host-only, pure): the y-ghost-row transfers of one
 * exchange, in the order the library posts them inside one NCCL group --
 * send up (to nbr_hi), send down (to nbr_lo), recv from down, recv from up.
 * Between two ranks NCCL matches sends and receives in posting order, so
 * the k-th send to a peer fills that peer's k-th receive from this rank.
 * Each span starts at x = -g of its first row and holds `count` =
 * (g-1)*ld + (n0+2g) elements (whole ghosted rows; the row padding rides
 * along), `offset` elements from patch.data of the rank's px_layout_patch.
 * Ranks at a non-periodic face have fewer ops; a one-rank layout has none
 * (its periodic wrap is local).  ops must hold 4 entries. */
typedef struct {
  int32_t peer;    /* rank sent to / received from               */
  int32_t is_recv; /* 0 = send, 1 = receive                      */
  int32_t row;     /* first global row y of the span              */
  int32_t nrows;   /* g                                           */
  int64_t offset;  /* element offset from patch.data (x = -g, y = row) */
  int64_t count;   /* elements in the span                        */
} px_halo_op;
px_status px_layout_halo_plan(const px_layout* l, int32_t rank, px_halo_op ops[4], int32_t* nops);

/* ----------------------------------------------------------------- kernels */
typedef enum {
  PX_LAPLACE_5PT = 0,
  PX_MEHRSTELLEN_9PT = 1,
  PX_LAPLACE_7PT_3D = 2,
  PX_MEHRSTELLEN_27PT_3D = 3
} px_stencil;
/* stencil: taps in the fixed order W,E,S,N(1),C(-4) for 5-point; W,E,S,N(4),
 * SW,SE,NW,NE(1),C(-20) for Mehrstellen (not in the paper, BASELINE config 5).
 * scale = 1/(h*h) (5-point) or 1/(6*h*h) (9-point), computed in double on the
 * host.  lambda is the Jacobi factor λ of Eq.3 (paper: h²/4D; an
 * explicit parameter here, R1). */
typedef struct {
  int32_t stencil;
  int32_t reserved;
  double h;
  double lambda;
} px_relax_params;

/* Norm buffers.  A device buffer of px_norm_buffer_len(region) doubles,
 * ZERO-INITIALISED ONCE by the caller (the kernels restore its scratch to
 * zero).  After a norm-producing call completes, buf[0] = max|r| (NaN if any
 * r is NaN) and buf[1] = Σ r² over the region's cells (deterministic
 * fixed-order reduction).  The grid L2 norm is sqrt(h² · buf[1]).
 * Calls sharing one buffer must be ordered on one stream. */
int64_t px_norm_buffer_len(px_box region);

/* dst(i) = scale · S(src)(i) for i in dest_box (Eq.1; Proto's
 * laplace(phiPatch, wgt)).  PX_ERR_DOMAIN (naming the first point and
 * tap) if grow(dest_box, 1) is not inside src->box or dest_box not inside
 * dst->box. */
px_status px_stencil_apply(int32_t stencil, double scale, const px_patch* src, px_patch* dst,
                           px_box dest_box, void* stream);

/* One fused sweep on one patch over `region` (Fig. ProtoX semantics,
 * P:218-238): for every cell, r = scale·S(φ_in) − rhs, φ_out = φ_in + λ·r.
 * Ghosts of φ_in must be valid; φ_out outside region is not written.
 * If d_norms != NULL it receives the norms of r, i.e. the residual of φ_in
 * (the PRE-update iterate, as the fused code reports it).
 * φ_in and φ_out must not overlap.  PX_ERR_ALIGN unless all ld are even and
 * φ_in, φ_out, rhs have the same 16-byte phase at region.lo. */
px_status px_relax_step(const px_relax_params* p, const px_patch* phi_in, px_patch* phi_out,
                        const px_patch* rhs, px_box region, double* d_norms, void* stream);

/* k fused sweeps in ONE pass over memory (temporal blocking, DESIGN.md §6
 * K7): φ_out = k Jacobi sweeps of φ_in over `region`, bit-identical to k
 * px_relax_step calls.  k in {2, 4}.  φ_in must hold valid values on
 * grow(region, k) and rhs on grow(region, k): cells outside the region are
 * advanced along with it as ordinary cells (the semantics of periodic
 * images and inter-rank ghost copies); their results are not written.
 * d_norms (optional) receives the norms of the residual of φ_in, as in
 * px_relax_step.  Needs a 16-byte aligned region start and an even width
 * (PX_ERR_ALIGN otherwise). */
px_status px_relax_block(const px_relax_params* p, int32_t k, const px_patch* phi_in,
                         px_patch* phi_out, const px_patch* rhs, px_box region, double* d_norms,
                         void* stream);

/* Residual norms of φ as given (computeMaxResidualAcrossProcs, single
 * patch): r = scale·S(φ) − rhs over region, into d_norms (required). */
px_status px_residual_norm(const px_relax_params* p, const px_patch* phi, const px_patch* rhs,
                           px_box region, double* d_norms, void* stream);

/* Mehrstellen right-hand side f = ρ + (1/12)·S5(ρ) over region (DESIGN.md
 * R18): fourth-order correction; ρ's ghosts must be filled. */
px_status px_mehrstellen_rhs(const px_patch* rho, px_patch* f, px_box region, void* stream);

/* Device synthetic fields over a rank's patch (its owned cells; ghosts are
 * then filled with px_fill_ghosts).  kind:
 *   PX_FIELD_ZERO  0
 *   PX_FIELD_HASH  ((splitmix64(seed ^ (i + j*n0)) >> 11) * 2^-53) * 2 - 1 over
 *                  global cell (i, j) relative to domain.lo, n0 = domain width
 *                  (bit-identical to paper_2307_07931_b200/inputs.py)
 *   PX_FIELD_SINE  sin(kπx) sin(lπy), x = (i+½)/n0, y = (j+½)/n1 */
typedef enum { PX_FIELD_ZERO = 0, PX_FIELD_HASH = 1, PX_FIELD_SINE = 2 } px_field;
px_status px_init_field(const px_layout* l, int32_t rank, px_patch* dst, int32_t kind,
                        uint64_t seed, int32_t k, int32_t l_wave, void* stream);

/* Fill the ghost cells a rank can fill locally: the x-ghosts of every row
 * (a slab always spans the domain in x: periodic wrap / Dirichlet
 * reflection), then full-width y-ghost rows at domain faces (reflection) or,
 * when the rank owns the whole domain, by periodic wrap.  Two phases (x then
 * y over full rows) so corners are right. */
px_status px_fill_ghosts(const px_layout* l, int32_t rank, px_patch* phi, void* stream);

/* ------------------------------------------------------------ communicator
 * One process per GPU.  The 128-byte NCCL unique id is created on rank 0
 * (px_comm_unique_id) and broadcast by the caller (torch.distributed). */
typedef struct px_comm px_comm;
px_status px_comm_unique_id(uint8_t id[128]);
px_status px_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                         px_comm** out);
void px_comm_destroy(px_comm* c);
/* Global all-reduce of n residual norms in device memory: d_max[i] by max,
 * d_sum[i] by sum (computeMaxResidualAcrossProcs).  NCCL on an NCCL
 * communicator; over peer memory on a px_comm_create_peer one (after
 * px_comm_p2p_import; Σ then in rank order).  d_max must hold
 * non-negative values (|r|, NaN with the sign bit clear): the max is taken
 * over their IEEE-754 bit patterns as uint64 (ncclUint64, ncclMax), which
 * orders non-negative doubles exactly and puts NaN above +inf, so a NaN on
 * any rank makes the global max NaN (reading R7; ncclMax on ncclDouble
 * gives no NaN guarantee).  Σr² is summed as doubles (NaN propagates). */
px_status px_comm_allreduce_norms(px_comm* c, double* d_max, double* d_sum, int32_t n,
                                  void* stream);

/* Peer-memory communicator: no NCCL.  Its ranks exchange ghost rows and
 * residual norms only through the fused peer-memory push below
 * (px_comm_p2p_export / px_comm_p2p_import), so px_solve with it needs push
 * mode (registered buffers, temporal_k = 1, even slab width, more than 2g
 * rows per slab; else PX_ERR_UNSUPPORTED), and px_exchange_ghosts /
 * px3_solve_comm refuse it.  Lets ranks that share one GPU (tests) or run
 * without NCCL use the path.  At most 16 ranks. */
px_status px_comm_create_peer(int32_t nranks, int32_t rank, int32_t device, px_comm** out);

/* Fused halo push over peer memory (NVLink / NVSwitch; "information is
 * exchanged between the boxes", P:173 computeMaxResidualAcrossProcs).
 *
 * Registration is two calls so the caller can move the records over any
 * process group:
 *   px_comm_p2p_export: register this rank's two solve buffers (φ and its
 *     scratch, as later passed to px_solve, in either order) and write this
 *     rank's PX_P2P_BLOB_BYTES record (CUDA IPC handles of the allocations
 *     holding them and of a library-owned control block; offsets; slab
 *     pitch).  Resets this rank's arrival counters, so every rank must
 *     export before any rank imports.
 *   px_comm_p2p_import: blobs = the nranks records in rank order (an
 *     all-gather of the exports); maps the slab neighbours' buffers and every
 *     rank's control block.  PX_ERR_ARG / PX_ERR_SHAPE if a record is not the
 *     matching rank's export for this layout.
 * px_comm_enable_p2p = export + NCCL all-gather + import (NCCL communicator).
 *
 * Afterwards px_solve (temporal_k = 1) runs ONE relax kernel per sweep over
 * the whole slab.  Its work items holding the first and last g rows are
 * scheduled first (each is the first item of its thread block) and, at their
 * end, store those rows of φ' -- with their x images, so corners are right --
 * straight into the neighbours' ghost rows (16-byte stores over NVLink).  The
 * next sweep's kernel publishes them: its first block counts one arrival per
 * side on the neighbours' counters (relaxed, system scope: the pushing grid
 * has completed, so its stores are performed -- no system-scope fence inside
 * a sweep), and its boundary blocks wait for their own counter (acquire)
 * before any thread reads a ghost row.  φ^0's rows are pushed by one small
 * kernel at the start; the norm ring is all-reduced over peer memory at the
 * end (every rank publishes its ring in its control block, reads all of them
 * in rank order: max over the u64 bit patterns -- NaN-propagating --, Σ in
 * rank order, so every rank gets the same bits).  No NCCL call and no
 * comm-stream hop in the solve.  Counters are cumulative (never reset after
 * export), so repeated solves of any lengths and CUDA graph replay are safe
 * as long as all ranks run the same sequence of solves.  Push mode needs an
 * even slab width, more than 2g rows per slab and a slab no wider than
 * 148 x 512 columns (else px_solve uses the NCCL exchange, or fails with
 * PX_ERR_UNSUPPORTED on a peer-memory communicator).  Buffers must outlive
 * the registration.  A one-rank periodic layout in self-exchange mode
 * (PROTOX_NCCL_SELF_EXCHANGE=1)
 * pushes to itself (test).  DIRICHLET_CC, PERIODIC and FIXED_GHOSTS. */
#define PX_P2P_BLOB_BYTES 256
px_status px_comm_p2p_export(px_comm* c, const px_layout* l, int32_t rank, const px_patch* phi,
                             const px_patch* phi_scratch, uint8_t* blob);
px_status px_comm_p2p_import(px_comm* c, const px_layout* l, const uint8_t* blobs);
px_status px_comm_enable_p2p(px_comm* c, const px_layout* l, int32_t rank, const px_patch* phi,
                             const px_patch* phi_scratch);

/* Full ghost exchange of rank `rank`'s patch: px_fill_ghosts, then the
 * y-ghost rows from the neighbour ranks over NCCL (full padded rows, so
 * corners are right).  c may be NULL only if the layout has one rank. */
px_status px_exchange_ghosts(const px_layout* l, px_comm* c, int32_t rank, px_patch* phi,
                             void* stream);

/* Exchange among ALL slabs of a multi-rank layout held on ONE device
 * (local transport: device-to-device copies).  parts[r] is rank r's patch. */
px_status px_exchange_ghosts_local(const px_layout* l, const px_patch* parts, void* stream);

/* ------------------------------------------------------------------- solve
 * N-sweep solve (figure `Proto`, fused).  nsweeps >= 0.
 * norm_every = E: record the global residual norms of φ^(jE) for every
 * jE < N (computed inside the sweep that consumes φ^(jE)), plus a final
 * entry for φ^N; E = 0: final entry only; E < 0: no norms.
 * temporal_k: sweeps per ghost exchange (1, or k in {2, 4} with k <= ghost
 * width: temporal blocking; every BC -- DIRICHLET_CC faces
 * re-derive their first ghost column/row by odd reflection after each of the
 * k levels, so a pass is exactly k plain sweeps).  use_graph: capture the sweep sequence in a CUDA
 * graph cached per (layout, comm, params, opts, pointers, stream); the
 * captured pointers must stay valid while the layout lives.
 *
 * Parts: with c == NULL the layout must have exactly one rank, or be solved
 * entirely on this device: then phi/phi_scratch/rhs are arrays of
 * nranks patches (local transport).  With an NCCL communicator they are
 * this rank's single patch.
 *
 * Host-synchronous.  On return h_norms[2j], h_norms[2j+1] hold (max|r|, Σr²)
 * of entry j (global over all ranks), *n_written the number of entries
 * (capped at cap), and φ^N is in phi (*in_scratch = 0) or in phi_scratch
 * (*in_scratch = 1: an odd number of buffer swaps -- one per sweep, or with
 * temporal_k = K one per K-sweep pass plus one per remaining sweep).  If
 * in_scratch is NULL, φ^N is copied into phi.
 * Inputs: phi holds φ^0 (ghosts need not be filled), rhs holds the
 * right-hand side (ρ, or f from px_mehrstellen_rhs) on owned cells plus, for
 * temporal_k > 1, its ghosts to depth k filled (px_exchange_ghosts). */
typedef struct {
  int32_t nsweeps;
  int32_t norm_every;
  int32_t temporal_k;
  int32_t use_graph;
} px_solve_opts;
px_status px_solve(const px_layout* l, px_comm* c, int32_t rank, const px_relax_params* p,
                   const px_solve_opts* o, px_patch* phi, px_patch* phi_scratch,
                   const px_patch* rhs, double* h_norms, int32_t cap, int32_t* n_written,
                   int32_t* in_scratch, void* stream);

/* px_solve without the host round trip (the same hot path):
 * everything is enqueued on `stream` and the call returns at once.  The
 * recorded norms go to DEVICE memory: d_norms[2j], d_norms[2j+1] = (max|r|,
 * Σr²) of entry j (global over all ranks), written stream-ordered after the
 * solve; *n_written and *in_scratch are known on return (they depend on the
 * options only).  For back-to-back solves of a pipeline (and the device-timed
 * bench); NCCL asynchronous errors surface at the next px_solve or
 * synchronising call.  Arguments, caching and errors otherwise as px_solve. */
px_status px_solve_async(const px_layout* l, px_comm* c, int32_t rank, const px_relax_params* p,
                         const px_solve_opts* o, px_patch* phi, px_patch* phi_scratch,
                         const px_patch* rhs, double* d_norms, int32_t cap, int32_t* n_written,
                         int32_t* in_scratch, void* stream);

/* End-to-end solve on HOST arrays (single rank): copies φ^0 and ρ
 * (n1 x n0 interior, dim-0 fastest, pinned or pageable host memory) to the
 * device, solves, copies φ^N back to h_phi_out.  Device buffers are
 * library-owned and cached by shape between calls (freed by
 * px_release_cached).  h_norms as in px_solve. */
px_status px_solve_host(const px_layout* l, const px_relax_params* p, const px_solve_opts* o,
                        const double* h_phi0, const double* h_rho, double* h_phi_out,
                        double* h_norms, int32_t cap, int32_t* n_written, void* stream);
/* Pipelined end-to-end solves of nprob independent problems on HOST arrays
 * (single rank, same layout / parameters / options for all): the H2D of
 * problem i+1 and the D2H of problem i-1 run on the copy engines (two
 * library streams) while problem i is solved on `stream`, over three
 * library-owned device buffer sets (cached like px_solve_host's).
 *   h_phi0[i]  n1 x n0 interior, dim-0 fastest; h_phi0 == NULL or
 *              h_phi0[i] == NULL: φ^0 = 0 (zero-filled on the device)
 *   h_rho[i]   right-hand side, same shape (required)
 *   h_phi_out[i] receives φ^N (required)
 *   h_norms    nprob * cap (max|r|, Σr²) pairs, problem i at h_norms[2*cap*i]
 *              (as px_solve); n_written: nprob counts, or NULL
 * Host buffers should be page-locked (cudaHostAlloc / cudaHostRegister) for
 * the copies to overlap the solves; pageable memory is correct but
 * serialises.  `stream` must be a non-default stream; work already on it
 * precedes the batch, and on return (host-synchronous) it is idle.
 * Results are bit-identical to nprob calls of px_solve_host. */
px_status px_solve_host_batch(const px_layout* l, const px_relax_params* p, const px_solve_opts* o,
                              int32_t nprob, const double* const* h_phi0, const double* const* h_rho,
                              double* const* h_phi_out, double* h_norms, int32_t cap, int32_t* n_written,
                              void* stream);
void px_release_cached(void);

/* Multigrid V-cycle with the fused relax sweep as smoother (SURVEY §8(f)
 * NEXT rank 2; multigrid is a Proto use of stencils, and ProtoX
 * future work; the cycle itself is DESIGN.md readings
 * R-MG1..R-MG6).  Levels l = 0..levels-1 with (n0 >> l) x (n1 >> l) cells,
 * h_l = 2^l h, λ_l = 4^l λ, the stencil of p and the layout's boundary rule
 * (homogeneous on l >= 1).  V(l): on the coarsest level nu_coarse sweeps;
 * else nu1 sweeps, f_{l+1} = −R(scale·S(φ_l) − f_l) (2x2 average),
 * φ_{l+1} = 0, V(l+1), φ_l += P φ_{l+1} (cell-centred bilinear), nu2 sweeps.
 * Single-rank layout, PERIODIC or DIRICHLET_CC; n0, n1 divisible by
 * 2^(levels-1), else PX_ERR_SHAPE.  phi holds φ^0 on entry (ghosts need not
 * be filled) and the result (with its ghost ring) on return; phi_scratch is
 * a second caller buffer of the same layout; rhs holds f on the owned cells.
 * Coarse-level buffers are library-owned, cached per (layout, params, opts,
 * pointers, stream) with the CUDA graph of the whole solve (use_graph),
 * freed by px_mg_release / px_release_cached.  h_norms[2k], [2k+1] =
 * (max|r|, Σr²) of the finest iterate after k cycles, k = 0..ncycles.
 * Host-synchronous.  Bit-identical to the oracle's orc_mg_solve. */
typedef struct {
  int32_t levels;
  int32_t nu1, nu2;
  int32_t nu_coarse;
  int32_t ncycles;
  int32_t use_graph;
} px_mg_opts;
px_status px_mg_solve(const px_layout* l, const px_relax_params* p, const px_mg_opts* o, px_patch* phi,
                      px_patch* phi_scratch, const px_patch* rhs, double* h_norms, int32_t cap,
                      int32_t* n_written, void* stream);
void px_mg_release(void);

/* ---------------------------------------------------------------------- 3D
 * The 3D relaxation.  The paper's Point and Box
 * are dimension-generic (Z^D), λ = h²/(4D);
 * the stencil PX_LAPLACE_7PT_3D (or PX_MEHRSTELLEN_27PT_3D, below) has taps W,E,S,N,B,T (offsets −x,+x,−y,+y,
 * −z,+z; weight 1) and C (−6) in that order, scale = 1/(h·h) (DESIGN.md
 * R-3D1); per cell r = scale·L − rhs, φ' = φ + λ·r, every operation rounded
 * once -- bit-identical to the oracle's orc3_solve.  Single device.
 *
 * A 3D patch over CALLER-OWNED device memory: cell (x, y, z) at
 * data[x + y·ld + z·plane], data pointing at cell (0,0,0); n = extents,
 * ghost = g (1..16).  The memory must cover cells (−2 .. n0+1, −g .. n1+g−1,
 * −g .. n2+g−1) (the TMA boxes read one column beyond the ghost layer);
 * data 16-byte aligned, ld and plane even; PX_ERR_ALIGN / PX_ERR_SHAPE
 * otherwise.  px3_layout gives a conforming layout: ld, plane, the element
 * offset of cell (0,0,0) in an allocation of alloc_elems doubles. */
typedef struct {
  double* data;
  int32_t n[3];
  int32_t ghost;
  int64_t ld, plane;
} px_patch3;
px_status px3_layout(const int32_t n[3], int32_t ghost, int64_t* ld, int64_t* plane, int64_t* origin,
                     int64_t* alloc_elems);
/* Norm buffer of px3_norm_buffer_len() doubles, zero-initialised once, with
 * the 2D norm-buffer protocol (buf[0] = max|r|, buf[1] = Σr²). */
int64_t px3_norm_buffer_len(void);
/* Synthetic field on the owned cells: kind 0 zeros, 1 the counter hash
 * u = splitmix64(seed ^ (x + n0·(y + n1·(z + z0)))), ((u >> 11)·2^-53)·2 − 1,
 * z0 = the global index of the patch's first plane (a z-slab's px3_slab z0;
 * 0 for a whole domain), so every decomposition gets the same field. */
px_status px3_init_field(px_patch3* p, int32_t kind, uint64_t seed, int32_t z0, void* stream);
/* 27-point variant (PX_MEHRSTELLEN_27PT_3D, R-3D4; not in the
 * paper -- the 3D counterpart of the BASELINE config-5 Mehrstellen stencil):
 * taps faces W,E,S,N,B,T (14), edges xy, xz, yz (3), corners z-major (1),
 * centre (−128), scale = 1/(30·h·h); fourth order with the right-hand side
 * f = ρ + (1/12)·S7(ρ) from px3_mehrstellen_rhs (ρ's ghosts filled; rho and
 * f distinct patches of one layout). */
px_status px3_mehrstellen_rhs(const px_patch3* rho, px_patch3* f, void* stream);
/* Ghost layer by the boundary rule (R-3D2): PERIODIC wrap,
 * DIRICHLET_CC odd reflection, phased x, y, z (edges and corners by the
 * product rule); FIXED_GHOSTS: nothing.  g <= every extent. */
px_status px3_fill_ghosts(px_bc bc, px_patch3* p, void* stream);
/* One fused sweep over all cells (ghosts of φ_in must be valid): φ_out =
 * φ_in + λ(scale·S(φ_in) − rhs); d_norms (optional, px3 norm buffer) gets
 * the residual norms of φ_in.  phi_in, phi_out, rhs: same extents and ghost
 * width; φ_in and φ_out must differ.  Asynchronous on stream. */
px_status px3_relax_step(const px_relax_params* p, const px_patch3* phi_in, px_patch3* phi_out,
                         const px_patch3* rhs, double* d_norms, void* stream);
/* Residual norms of φ as given (Eq.7; ghosts must be valid) into d_norms. */
px_status px3_residual_norm(const px_relax_params* p, const px_patch3* phi, const px_patch3* rhs,
                            double* d_norms, void* stream);
/* N-sweep solve (figure `Proto` in 3D, fused): per sweep the ghost fill of bc
 * then one fused sweep; norm schedule, h_norms / cap / n_written / in_scratch
 * exactly as px_solve (temporal_k must be <= 1).  use_graph: the sequence is
 * captured once into a CUDA graph cached per (bc, params, opts, patches,
 * stream) until px3_release.  Host-synchronous. */
px_status px3_solve(px_bc bc, const px_relax_params* p, const px_solve_opts* o, px_patch3* phi,
                    px_patch3* phi_scratch, const px_patch3* rhs, double* h_norms, int32_t cap,
                    int32_t* n_written, int32_t* in_scratch, void* stream);
/* z-slab decomposition of a 3D domain (n2 planes) over nranks ranks, the 3D
 * counterpart of the 2D slab partitioner: rank r owns planes
 * [z0, z1) = [r·n2/P, (r+1)·n2/P).  PX_ERR_SHAPE if n2 < nranks. */
px_status px3_slab(int32_t n2, int32_t nranks, int32_t rank, int32_t* z0, int32_t* z1);
/* px3_solve on this rank's z-slab of a domain split over the communicator's
 * ranks (patches hold the rank's n2 = z1 - z0 planes): per sweep the x / y
 * ghosts locally, the z ghost planes from the slab neighbours in one NCCL
 * group (send up, send down, recv down, recv up) -- a periodic ring, or the
 * boundary rule at the global z faces -- then the fused sweep; the recorded
 * norms are all-reduced over the ranks once at the end (ncclMax, ncclSum).
 * A one-rank communicator created with PROTOX_NCCL_SELF_EXCHANGE=1 exchanges
 * its periodic z planes with itself (test mode). */
px_status px3_solve_comm(px_comm* c, px_bc bc, const px_relax_params* p, const px_solve_opts* o, px_patch3* phi,
                         px_patch3* phi_scratch, const px_patch3* rhs, double* h_norms, int32_t cap,
                         int32_t* n_written, int32_t* in_scratch, void* stream);
/* px3_solve (figure `Proto`, per problem) for nprob independent
 * problems given as HOST arrays -- the 3D counterpart of px_solve_host_batch.  Every array is a dense (n[2], n[1],
 * n[0]) fp64 block of owned cells, x fastest; h_rho[i] is read, h_phi_out[i]
 * (φ^N) written; h_phi0 NULL (or a NULL entry) = zero initial guess.  The
 * library owns three device buffer sets (fields with `ghost` ghost layers,
 * px3_layout pitches), each with its own cached plan / CUDA graph, so problem
 * i's H2D and problem i-1's D2H (two internal copy streams) overlap problem
 * i's solve on `stream` (required, non-default).  Norms: h_norms[i·2·cap + 2j
 * + {0,1}] and n_written[i] as px3_solve.  bc PERIODIC or DIRICHLET_CC
 * (host arrays carry no ghosts: PX_ERR_UNSUPPORTED for FIXED_GHOSTS).  Host
 * buffers should be pinned for the copies to overlap.  Host-synchronous;
 * px3_release frees the buffers. */
px_status px3_solve_host_batch(px_bc bc, const px_relax_params* p, const px_solve_opts* o, const int32_t n[3],
                               int32_t ghost, int32_t nprob, const double* const* h_phi0,
                               const double* const* h_rho, double* const* h_phi_out, double* h_norms, int32_t cap,
                               int32_t* n_written, void* stream);
void px3_release(void);

/* Diagnostics: number of kernel launches libprotox enqueued so far in this
 * process (graph replays count their kernel nodes). */
int64_t px_kernel_launch_count(void);
/* Diagnostics: the sweep kernels the calling thread's last px_solve (or
 * px_solve_host / px_solve_host_batch) enqueued, '+'-separated in launch
 * order, e.g. "k_bulk", "k_stream+k_bulk" (boundary rows + interior),
 * "k_tbw", "k_resident", "k_persist", "k_cluster_box", "k_smallbox".  The
 * string is library-owned and valid until the thread's next solve; "" before
 * the first. */
const char* px_last_solve_kernels(void);
/* Diagnostics: which relax kernel a px_relax_step over `region` would run:
 * 1 = TMA bulk-copy pipeline (16-byte aligned region start, even width,
 * >= 4M cells), 0 = register-streaming LDG.128 kernel, <0 = invalid args.
 * Setting PROTOX_KERNEL=ldg in the environment (read once) forces 0. */
int32_t px_relax_variant(const px_patch* phi_in, const px_patch* phi_out, const px_patch* rhs,
                         px_box region);

/* Proto's UNFUSED pointwise update (forallInPlace(jacobiUpdate), figure
 * `Proto`; Eq.3): φ ← φ + λ(temp − rhs) in place over region,
 * with temp = scale·S(φ) from px_stencil_apply.  With px_stencil_apply and
 * px_residual_norm it forms the unfused Proto sequence that the fused sweep
 * replaces -- a measurement baseline (the paper's fused-vs-unfused
 * comparison, on the GPU), bit-identical to px_relax_step.
 * PX_ERR_DOMAIN if region is not inside every patch.  Asynchronous. */
px_status px_pointwise_update(px_patch* phi, const px_patch* temp, const px_patch* rhs, double lambda,
                              px_box region, void* stream);

/* Measurement helper (not part of the method): the streaming ceiling of the
 * GPU for the sweep's access pattern.  variant 0: c[i] = a[i] + b[i] (2 reads,
 * 1 write, like the fused sweep); variant 1: c[i] = a[i] (copy).  n even,
 * pointers 16-byte aligned, device memory.  Asynchronous on stream. */
px_status px_stream_ceiling(const double* a, const double* b, double* c, int64_t n,
                            int32_t variant, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PROTOX_H */
