"""Thin ctypes binding of libprotox (include/protox.h), same names as the C ABI.

Argument marshalling only: every step of the method runs in libprotox's CUDA
kernels.  PyTorch supplies device memory (float64 tensors), streams
(``torch.cuda.Stream``) and process groups (only to broadcast the NCCL id).
There is no fallback: if ``libprotox.so`` is missing or fails to load, every
call raises.
"""
from __future__ import annotations

import ctypes
import types
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# PROTOX_LIB: another build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("PROTOX_LIB") or os.path.join(_PKG, "libprotox.so")

# ---------------------------------------------------------------- constants
PX_OK, PX_ERR_ARG, PX_ERR_SHAPE, PX_ERR_DOMAIN, PX_ERR_ALIGN = 0, 1, 2, 3, 4
PX_ERR_UNSUPPORTED, PX_ERR_CUDA, PX_ERR_NCCL, PX_ERR_STATE = 5, 6, 7, 8
PX_BC_PERIODIC, PX_BC_DIRICHLET_CC, PX_BC_FIXED_GHOSTS = 0, 1, 2
PX_PART_SLABS = 0
PX_LAPLACE_5PT, PX_MEHRSTELLEN_9PT, PX_LAPLACE_7PT_3D, PX_MEHRSTELLEN_27PT_3D = 0, 1, 2, 3
PX_FIELD_ZERO, PX_FIELD_HASH, PX_FIELD_SINE = 0, 1, 2


class px_point(ctypes.Structure):
    _fields_ = [("c", ctypes.c_int32 * 2)]


class px_box(ctypes.Structure):
    _fields_ = [("lo", px_point), ("hi", px_point)]

    def __repr__(self):
        return f"px_box(({self.lo.c[0]},{self.lo.c[1]}),({self.hi.c[0]},{self.hi.c[1]}))"

    def tuple(self):
        return (self.lo.c[0], self.lo.c[1], self.hi.c[0], self.hi.c[1])


class px_local_info(ctypes.Structure):
    _fields_ = [("owned", px_box), ("alloc", px_box), ("ld", ctypes.c_int64),
                ("patch_offset", ctypes.c_int64), ("alloc_elems", ctypes.c_int64),
                ("nbr_lo", ctypes.c_int32), ("nbr_hi", ctypes.c_int32)]


class px_halo_op(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("is_recv", ctypes.c_int32), ("row", ctypes.c_int32),
                ("nrows", ctypes.c_int32), ("offset", ctypes.c_int64), ("count", ctypes.c_int64)]


class px_patch(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("box", px_box), ("ld", ctypes.c_int64)]


class px_relax_params(ctypes.Structure):
    _fields_ = [("stencil", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("h", ctypes.c_double), ("lam", ctypes.c_double)]


class px_solve_opts(ctypes.Structure):
    _fields_ = [("nsweeps", ctypes.c_int32), ("norm_every", ctypes.c_int32),
                ("temporal_k", ctypes.c_int32), ("use_graph", ctypes.c_int32)]


class px_patch3(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("n", ctypes.c_int32 * 3), ("ghost", ctypes.c_int32),
                ("ld", ctypes.c_int64), ("plane", ctypes.c_int64)]


class px_mg_opts(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("nu1", ctypes.c_int32), ("nu2", ctypes.c_int32),
                ("nu_coarse", ctypes.c_int32), ("ncycles", ctypes.c_int32), ("use_graph", ctypes.c_int32)]


def point(x, y) -> px_point:
    p = px_point()
    p.c[0], p.c[1] = int(x), int(y)
    return p


def box(x0, y0, x1, y1) -> px_box:
    return px_box(point(x0, y0), point(x1, y1))


# ---------------------------------------------------------------- loading
_lib = None

EXPORTS = [
    "px_status_str", "px_last_error", "px_api_version",
    "px_box_size", "px_box_is_empty", "px_box_grow", "px_box_intersect", "px_box_ordinal",
    "px_layout_create", "px_layout_destroy", "px_layout_num_boxes", "px_layout_box",
    "px_layout_local", "px_layout_patch", "px_layout_halo_plan", "px_norm_buffer_len",
    "px_stencil_apply", "px_relax_step", "px_relax_block", "px_residual_norm", "px_mehrstellen_rhs",
    "px_init_field", "px_fill_ghosts",
    "px_comm_unique_id", "px_comm_create", "px_comm_destroy", "px_comm_allreduce_norms",
    "px_comm_enable_p2p", "px_comm_create_peer", "px_comm_p2p_export", "px_comm_p2p_import",
    "px_exchange_ghosts", "px_exchange_ghosts_local",
    "px_solve", "px_solve_async", "px_solve_host", "px_solve_host_batch", "px_release_cached", "px_mg_solve", "px_mg_release", "px_kernel_launch_count",
    "px_last_solve_kernels",
    "px_relax_variant", "px_stream_ceiling", "px_pointwise_update",
    "px3_layout", "px3_norm_buffer_len", "px3_init_field", "px3_fill_ghosts", "px3_relax_step",
    "px3_residual_norm", "px3_solve", "px3_solve_host_batch", "px3_release", "px3_mehrstellen_rhs", "px3_slab", "px3_solve_comm",
]


class _Older:
    """Attribute sink over an older libprotox build (PROTOX_LIB A/B runs)."""

    def __init__(self, L):
        self._L = L

    def __getattr__(self, name):
        try:
            return getattr(self._L, name)
        except AttributeError:
            return types.SimpleNamespace()


def lib():
    """Load libprotox.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libprotox.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    real = L
    if os.environ.get("PROTOX_LIB"):
        L = _Older(L)  # an older build (A/B): symbols it lacks are skipped
    st, i32, i64, vp = ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    P = ctypes.POINTER
    L.px_status_str.restype = ctypes.c_char_p
    L.px_status_str.argtypes = [st]
    L.px_last_error.restype = ctypes.c_char_p
    L.px_api_version.restype = i32
    L.px_box_size.restype = i64
    L.px_box_size.argtypes = [px_box]
    L.px_box_is_empty.restype = i32
    L.px_box_is_empty.argtypes = [px_box]
    L.px_box_grow.restype = px_box
    L.px_box_grow.argtypes = [px_box, i32]
    L.px_box_intersect.restype = px_box
    L.px_box_intersect.argtypes = [px_box, px_box]
    L.px_box_ordinal.restype = st
    L.px_box_ordinal.argtypes = [px_box, px_point, P(i64)]
    L.px_layout_create.restype = st
    L.px_layout_create.argtypes = [px_box, px_point, i32, st, i32, st, P(vp)]
    L.px_layout_destroy.restype = None
    L.px_layout_destroy.argtypes = [vp]
    L.px_layout_num_boxes.restype = st
    L.px_layout_num_boxes.argtypes = [vp, P(i32)]
    L.px_layout_box.restype = st
    L.px_layout_box.argtypes = [vp, i32, P(px_box), P(i32)]
    L.px_layout_local.restype = st
    L.px_layout_local.argtypes = [vp, i32, P(px_local_info)]
    L.px_layout_patch.restype = st
    L.px_layout_patch.argtypes = [vp, i32, vp, P(px_patch)]
    L.px_layout_halo_plan.restype = st
    L.px_layout_halo_plan.argtypes = [vp, i32, P(px_halo_op), P(i32)]
    L.px_norm_buffer_len.restype = i64
    L.px_norm_buffer_len.argtypes = [px_box]
    L.px_stencil_apply.restype = st
    L.px_stencil_apply.argtypes = [i32, ctypes.c_double, P(px_patch), P(px_patch), px_box, vp]
    L.px_relax_step.restype = st
    L.px_relax_step.argtypes = [P(px_relax_params), P(px_patch), P(px_patch), P(px_patch), px_box, vp, vp]
    L.px_relax_block.restype = st
    L.px_relax_block.argtypes = [P(px_relax_params), i32, P(px_patch), P(px_patch), P(px_patch), px_box, vp, vp]
    L.px_residual_norm.restype = st
    L.px_residual_norm.argtypes = [P(px_relax_params), P(px_patch), P(px_patch), px_box, vp, vp]
    L.px_mehrstellen_rhs.restype = st
    L.px_mehrstellen_rhs.argtypes = [P(px_patch), P(px_patch), px_box, vp]
    L.px_init_field.restype = st
    L.px_init_field.argtypes = [vp, i32, P(px_patch), i32, ctypes.c_uint64, i32, i32, vp]
    L.px_fill_ghosts.restype = st
    L.px_fill_ghosts.argtypes = [vp, i32, P(px_patch), vp]
    L.px_comm_unique_id.restype = st
    L.px_comm_unique_id.argtypes = [ctypes.c_char_p]
    L.px_comm_create.restype = st
    L.px_comm_create.argtypes = [ctypes.c_char_p, i32, i32, i32, P(vp)]
    L.px_comm_destroy.restype = None
    L.px_comm_destroy.argtypes = [vp]
    L.px_comm_enable_p2p.restype = st
    L.px_comm_enable_p2p.argtypes = [vp, vp, i32, P(px_patch), P(px_patch)]
    L.px_comm_create_peer.restype = st
    L.px_comm_create_peer.argtypes = [i32, i32, i32, P(vp)]
    L.px_comm_p2p_export.restype = st
    L.px_comm_p2p_export.argtypes = [vp, vp, i32, P(px_patch), P(px_patch), ctypes.c_char_p]
    L.px_comm_p2p_import.restype = st
    L.px_comm_p2p_import.argtypes = [vp, vp, ctypes.c_char_p]
    L.px_comm_allreduce_norms.restype = st
    L.px_comm_allreduce_norms.argtypes = [vp, vp, vp, i32, vp]
    L.px_exchange_ghosts.restype = st
    L.px_exchange_ghosts.argtypes = [vp, vp, i32, P(px_patch), vp]
    L.px_exchange_ghosts_local.restype = st
    L.px_exchange_ghosts_local.argtypes = [vp, P(px_patch), vp]
    L.px_solve.restype = st
    L.px_solve.argtypes = [vp, vp, i32, P(px_relax_params), P(px_solve_opts), P(px_patch),
                           P(px_patch), P(px_patch), P(ctypes.c_double), i32, P(i32), P(i32), vp]
    L.px_solve_async.restype = st
    L.px_solve_async.argtypes = [vp, vp, i32, P(px_relax_params), P(px_solve_opts), P(px_patch),
                           P(px_patch), P(px_patch), P(ctypes.c_double), i32, P(i32), P(i32), vp]
    L.px_solve_host.restype = st
    L.px_solve_host.argtypes = [vp, P(px_relax_params), P(px_solve_opts), vp, vp, vp,
                                P(ctypes.c_double), i32, P(i32), vp]
    L.px_solve_host_batch.restype = st
    L.px_solve_host_batch.argtypes = [vp, P(px_relax_params), P(px_solve_opts), i32, vp, vp, vp,
                                      P(ctypes.c_double), i32, P(i32), vp]
    L.px_mg_solve.restype = st
    L.px_mg_solve.argtypes = [vp, P(px_relax_params), P(px_mg_opts), P(px_patch), P(px_patch), P(px_patch),
                              P(ctypes.c_double), i32, P(i32), vp]
    L.px_mg_release.restype = None
    L.px_release_cached.restype = None
    L.px_kernel_launch_count.restype = i64
    L.px_last_solve_kernels.restype = ctypes.c_char_p
    L.px_stream_ceiling.restype = st
    L.px_stream_ceiling.argtypes = [vp, vp, vp, i64, i32, vp]
    L.px_pointwise_update.restype = st
    L.px_pointwise_update.argtypes = [P(px_patch), P(px_patch), P(px_patch), ctypes.c_double, px_box, vp]
    L.px3_layout.restype = st
    L.px3_layout.argtypes = [P(i32), i32, P(i64), P(i64), P(i64), P(i64)]
    L.px3_norm_buffer_len.restype = i64
    L.px3_init_field.restype = st
    L.px3_init_field.argtypes = [P(px_patch3), i32, ctypes.c_uint64, i32, vp]
    L.px3_fill_ghosts.restype = st
    L.px3_fill_ghosts.argtypes = [st, P(px_patch3), vp]
    L.px3_relax_step.restype = st
    L.px3_relax_step.argtypes = [P(px_relax_params), P(px_patch3), P(px_patch3), P(px_patch3), vp, vp]
    L.px3_residual_norm.restype = st
    L.px3_residual_norm.argtypes = [P(px_relax_params), P(px_patch3), P(px_patch3), vp, vp]
    L.px3_solve.restype = st
    L.px3_solve.argtypes = [st, P(px_relax_params), P(px_solve_opts), P(px_patch3), P(px_patch3), P(px_patch3),
                            P(ctypes.c_double), i32, P(i32), P(i32), vp]
    L.px3_solve_host_batch.restype = st
    L.px3_solve_host_batch.argtypes = [st, P(px_relax_params), P(px_solve_opts), P(i32), i32, i32, vp, vp, vp,
                                       P(ctypes.c_double), i32, P(i32), vp]
    L.px3_release.restype = None
    L.px3_slab.restype = st
    L.px3_slab.argtypes = [i32, i32, i32, P(i32), P(i32)]
    L.px3_solve_comm.restype = st
    L.px3_solve_comm.argtypes = [vp, st, P(px_relax_params), P(px_solve_opts), P(px_patch3), P(px_patch3),
                                 P(px_patch3), P(ctypes.c_double), i32, P(i32), P(i32), vp]
    L.px3_mehrstellen_rhs.restype = st
    L.px3_mehrstellen_rhs.argtypes = [P(px_patch3), P(px_patch3), vp]
    L.px_relax_variant.restype = i32
    L.px_relax_variant.argtypes = [P(px_patch), P(px_patch), P(px_patch), px_box]
    _lib = real
    return real


class PxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{lib().px_status_str(status).decode()}: {msg}")
        self.status = status


def _check(status: int):
    if status != PX_OK:
        raise PxError(status, lib().px_last_error().decode())


def _stream(stream) -> int | None:
    """Accept a torch.cuda.Stream, an int handle or None (torch's current stream)."""
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream or None
    if isinstance(stream, int):
        return stream or None
    return stream.cuda_stream or None


# ---------------------------------------------------------------- geometry
def box_size(b: px_box) -> int:
    return lib().px_box_size(b)


def box_is_empty(b: px_box) -> bool:
    return bool(lib().px_box_is_empty(b))


def box_grow(b: px_box, r: int) -> px_box:
    return lib().px_box_grow(b, r)


def box_intersect(a: px_box, b: px_box) -> px_box:
    return lib().px_box_intersect(a, b)


def box_ordinal(b: px_box, p: px_point) -> int:
    out = ctypes.c_int64()
    _check(lib().px_box_ordinal(b, p, ctypes.byref(out)))
    return out.value


# ---------------------------------------------------------------- layout
class Layout:
    """px_layout handle: Proto's box decomposition into slabs."""

    def __init__(self, domain: px_box, box_size, ghost: int = 1, bc: int = PX_BC_PERIODIC,
                 nranks: int = 1, part: int = PX_PART_SLABS):
        h = ctypes.c_void_p()
        _check(lib().px_layout_create(domain, point(*box_size), ghost, bc, nranks, part,
                                      ctypes.byref(h)))
        self.h = h
        self.domain = domain
        self.ghost = ghost
        self.bc = bc
        self.nranks = nranks

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.px_layout_destroy(self.h)
            self.h = None

    @property
    def _as_parameter_(self):
        return self.h

    def num_boxes(self) -> int:
        n = ctypes.c_int32()
        _check(lib().px_layout_num_boxes(self.h, ctypes.byref(n)))
        return n.value

    def box(self, i: int):
        b, o = px_box(), ctypes.c_int32()
        _check(lib().px_layout_box(self.h, i, ctypes.byref(b), ctypes.byref(o)))
        return b, o.value

    def local(self, rank: int = 0) -> px_local_info:
        li = px_local_info()
        _check(lib().px_layout_local(self.h, rank, ctypes.byref(li)))
        return li

    def halo_plan(self, rank: int) -> list:
        """px_layout_halo_plan: the rank's y-ghost transfers in posting order."""
        ops = (px_halo_op * 4)()
        n = ctypes.c_int32()
        _check(lib().px_layout_halo_plan(self.h, rank, ops, ctypes.byref(n)))
        return [ops[i] for i in range(n.value)]

    def alloc(self, rank: int = 0, device=None):
        """Zero-filled float64 CUDA tensor sized for rank's ghosted slab."""
        import torch
        li = self.local(rank)
        return torch.zeros(li.alloc_elems, dtype=torch.float64, device=device or "cuda")

    def patch(self, rank: int, tensor) -> px_patch:
        p = px_patch()
        _check(lib().px_layout_patch(self.h, rank, ctypes.c_void_p(tensor.data_ptr()),
                                     ctypes.byref(p)))
        return p

    def view(self, rank: int, tensor, ghosts: bool = False):
        """(rows, cols) strided view of rank's owned cells (ghosts=True: ghosted box)."""
        li = self.local(rank)
        b = li.alloc if ghosts else li.owned
        off = li.patch_offset + (b.lo.c[0] - li.alloc.lo.c[0]) + (b.lo.c[1] - li.alloc.lo.c[1]) * li.ld
        return tensor.as_strided((b.hi.c[1] - b.lo.c[1] + 1, b.hi.c[0] - b.lo.c[0] + 1), (li.ld, 1), off)


def norm_buffer_len(region: px_box) -> int:
    return lib().px_norm_buffer_len(region)


def norm_buffer(region: px_box, device=None):
    import torch
    return torch.zeros(norm_buffer_len(region), dtype=torch.float64, device=device or "cuda")


def relax_params(h: float, lam: float, stencil: int = PX_LAPLACE_5PT) -> px_relax_params:
    return px_relax_params(stencil, 0, h, lam)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


# ---------------------------------------------------------------- kernels
def stencil_apply(stencil: int, scale: float, src: px_patch, dst: px_patch, dest_box: px_box,
                  stream=None):
    _check(lib().px_stencil_apply(stencil, scale, ctypes.byref(src), ctypes.byref(dst), dest_box,
                                  _stream(stream)))


def relax_step(p: px_relax_params, phi_in: px_patch, phi_out: px_patch, rhs: px_patch,
               region: px_box, norms=None, stream=None):
    _check(lib().px_relax_step(ctypes.byref(p), ctypes.byref(phi_in), ctypes.byref(phi_out),
                               ctypes.byref(rhs), region, _ptr(norms), _stream(stream)))


def relax_block(p: px_relax_params, k: int, phi_in: px_patch, phi_out: px_patch, rhs: px_patch,
                region: px_box, norms=None, stream=None):
    """px_relax_block: k sweeps in one pass (temporal blocking)."""
    _check(lib().px_relax_block(ctypes.byref(p), k, ctypes.byref(phi_in), ctypes.byref(phi_out),
                                ctypes.byref(rhs), region, _ptr(norms), _stream(stream)))


def residual_norm(p: px_relax_params, phi: px_patch, rhs: px_patch, region: px_box, norms,
                  stream=None):
    _check(lib().px_residual_norm(ctypes.byref(p), ctypes.byref(phi), ctypes.byref(rhs), region,
                                  _ptr(norms), _stream(stream)))


def mehrstellen_rhs(rho: px_patch, f: px_patch, region: px_box, stream=None):
    _check(lib().px_mehrstellen_rhs(ctypes.byref(rho), ctypes.byref(f), region, _stream(stream)))


def init_field(layout: Layout, rank: int, dst: px_patch, kind: int, seed: int = 0, k: int = 1,
               l: int = 1, stream=None):
    _check(lib().px_init_field(layout.h, rank, ctypes.byref(dst), kind, seed, k, l, _stream(stream)))


def fill_ghosts(layout: Layout, rank: int, phi: px_patch, stream=None):
    _check(lib().px_fill_ghosts(layout.h, rank, ctypes.byref(phi), _stream(stream)))


# ---------------------------------------------------------------- comm
class Comm:
    """Communicator (one process per GPU): NCCL (px_comm_create), or with
    uid=None peer memory only (px_comm_create_peer)."""

    def __init__(self, uid, nranks: int, rank: int, device: int):
        h = ctypes.c_void_p()
        if uid is None:
            _check(lib().px_comm_create_peer(nranks, rank, device, ctypes.byref(h)))
        else:
            _check(lib().px_comm_create(uid, nranks, rank, device, ctypes.byref(h)))
        self.h = h
        self.nranks, self.rank = nranks, rank

    def close(self):
        if getattr(self, "h", None):
            lib().px_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        if _lib is not None:
            self.close()


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().px_comm_unique_id(buf))
    return buf.raw


def comm_enable_p2p(comm: Comm, layout: Layout, rank: int, phi: px_patch, phi_scratch: px_patch):
    """px_comm_enable_p2p: fused halo push over peer memory for px_solve."""
    _check(lib().px_comm_enable_p2p(comm.h, layout.h, rank, ctypes.byref(phi), ctypes.byref(phi_scratch)))


P2P_BLOB_BYTES = 256  # PX_P2P_BLOB_BYTES


def comm_p2p_export(comm: Comm, layout: Layout, rank: int, phi: px_patch, phi_scratch: px_patch) -> bytes:
    """px_comm_p2p_export: register the solve buffers, return this rank's record."""
    buf = ctypes.create_string_buffer(P2P_BLOB_BYTES)
    _check(lib().px_comm_p2p_export(comm.h, layout.h, rank, ctypes.byref(phi), ctypes.byref(phi_scratch), buf))
    return buf.raw


def comm_p2p_import(comm: Comm, layout: Layout, records) -> None:
    """px_comm_p2p_import: records = every rank's export, in rank order."""
    blob = b"".join(bytes(r) for r in records)
    if len(blob) != P2P_BLOB_BYTES * comm.nranks:
        raise ValueError("need one record per rank")
    _check(lib().px_comm_p2p_import(comm.h, layout.h, blob))


def comm_allreduce_norms(comm: Comm, d_max, d_sum, n: int, stream=None):
    _check(lib().px_comm_allreduce_norms(comm.h, _ptr(d_max), _ptr(d_sum), n, _stream(stream)))


def exchange_ghosts(layout: Layout, comm: Comm | None, rank: int, phi: px_patch, stream=None):
    _check(lib().px_exchange_ghosts(layout.h, comm.h if comm else None, rank, ctypes.byref(phi),
                                    _stream(stream)))


def exchange_ghosts_local(layout: Layout, parts: list, stream=None):
    arr = (px_patch * len(parts))(*parts)
    _check(lib().px_exchange_ghosts_local(layout.h, arr, _stream(stream)))


# ---------------------------------------------------------------- solve
@dataclass
class SolveResult:
    norms: np.ndarray      # (n, 2): max|r|, sum r^2 per recorded iterate
    in_scratch: bool


def solve(layout: Layout, comm: Comm | None, rank: int, p: px_relax_params, nsweeps: int,
          norm_every: int, phi, phi_scratch, rhs, temporal_k: int = 1, use_graph: bool = False,
          cap: int | None = None, stream=None, keep_in_scratch: bool = True) -> SolveResult:
    """px_solve.  phi / phi_scratch / rhs: a px_patch, or a list of patches
    (one per rank of the layout) when comm is None and nranks > 1."""
    as_list = lambda v: v if isinstance(v, (list, tuple)) else [v]
    ph, sc, rh = as_list(phi), as_list(phi_scratch), as_list(rhs)
    n = len(ph)
    A = px_patch * n
    opts = px_solve_opts(nsweeps, norm_every, temporal_k, int(use_graph))
    if cap is None:
        cap = 0 if norm_every < 0 else ((nsweeps + norm_every - 1) // norm_every if norm_every > 0 else 0) + 1
    norms = np.zeros((max(cap, 1), 2), dtype=np.float64)
    nw, ins = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib().px_solve(layout.h, comm.h if comm else None, rank, ctypes.byref(p),
                          ctypes.byref(opts), A(*ph), A(*sc), A(*rh),
                          norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap,
                          ctypes.byref(nw), ctypes.byref(ins) if keep_in_scratch else None,
                          _stream(stream)))
    return SolveResult(norms[: nw.value].copy(), bool(ins.value))


def solve_async(layout: Layout, comm: Comm | None, rank: int, p: px_relax_params, nsweeps: int,
                norm_every: int, phi, phi_scratch, rhs, d_norms, temporal_k: int = 1, use_graph: bool = False,
                stream=None, keep_in_scratch: bool = True) -> tuple[int, bool]:
    """px_solve_async: as solve(), enqueued without a host round trip; the
    norms go to d_norms (a float64 cuda tensor of >= 2 * entries elements).
    Returns (entries written, in_scratch)."""
    as_list = lambda v: v if isinstance(v, (list, tuple)) else [v]
    ph, sc, rh = as_list(phi), as_list(phi_scratch), as_list(rhs)
    n = len(ph)
    A = px_patch * n
    opts = px_solve_opts(nsweeps, norm_every, temporal_k, int(use_graph))
    cap = d_norms.numel() // 2
    nw, ins = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib().px_solve_async(layout.h, comm.h if comm else None, rank, ctypes.byref(p),
                                ctypes.byref(opts), A(*ph), A(*sc), A(*rh),
                                ctypes.cast(d_norms.data_ptr(), ctypes.POINTER(ctypes.c_double)), cap,
                                ctypes.byref(nw), ctypes.byref(ins) if keep_in_scratch else None,
                                _stream(stream)))
    return nw.value, bool(ins.value)


def mg_solve(layout: Layout, p: px_relax_params, levels: int, ncycles: int, phi: px_patch,
             phi_scratch: px_patch, rhs: px_patch, nu1: int = 2, nu2: int = 2, nu_coarse: int = 8,
             use_graph: bool = False, stream=None) -> np.ndarray:
    """px_mg_solve: ncycles V(nu1, nu2)-cycles; the result is in phi.
    Returns norms[k] = (max|r|, sum r^2) after k cycles, k = 0..ncycles."""
    opts = px_mg_opts(levels, nu1, nu2, nu_coarse, ncycles, int(use_graph))
    cap = ncycles + 1
    norms = np.zeros((cap, 2), dtype=np.float64)
    nw = ctypes.c_int32(0)
    ph, sc, rh = px_patch(phi.data, phi.box, phi.ld), px_patch(phi_scratch.data, phi_scratch.box, phi_scratch.ld), \
        px_patch(rhs.data, rhs.box, rhs.ld)
    _check(lib().px_mg_solve(layout.h, ctypes.byref(p), ctypes.byref(opts), ctypes.byref(ph), ctypes.byref(sc),
                             ctypes.byref(rh), norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap,
                             ctypes.byref(nw), _stream(stream)))
    return norms[: nw.value].copy()


def solve_host(layout: Layout, p: px_relax_params, nsweeps: int, norm_every: int,
               phi0: np.ndarray, rho: np.ndarray, out: np.ndarray | None = None,
               use_graph: bool = False, stream=None, temporal_k: int = 1):
    """px_solve_host: numpy (n1, n0) float64 host arrays (pinned torch CPU
    tensors also accepted via .numpy()).  Returns (phi_N, norms)."""
    phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    if out is None:
        out = np.empty_like(phi0)
    cap = 0 if norm_every < 0 else ((nsweeps + norm_every - 1) // norm_every if norm_every > 0 else 0) + 1
    norms = np.zeros((max(cap, 1), 2), dtype=np.float64)
    nw = ctypes.c_int32(0)
    opts = px_solve_opts(nsweeps, norm_every, temporal_k, int(use_graph))
    _check(lib().px_solve_host(layout.h, ctypes.byref(p), ctypes.byref(opts),
                               phi0.ctypes.data_as(ctypes.c_void_p), rho.ctypes.data_as(ctypes.c_void_p),
                               out.ctypes.data_as(ctypes.c_void_p),
                               norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap,
                               ctypes.byref(nw), _stream(stream)))
    return out, norms[: nw.value].copy()


def solve_host_batch(layout: Layout, p: px_relax_params, nsweeps: int, norm_every: int,
                     rhos, outs, phi0s=None, use_graph: bool = True, stream=None, temporal_k: int = 1):
    """px_solve_host_batch: len(rhos) independent problems from host arrays,
    copies overlapped with the solves.  rhos/outs/phi0s: lists of (n1, n0)
    float64 numpy arrays (pinned torch CPU tensors via .numpy() for overlap);
    phi0s None (or None entries) = zero initial guess.  Returns the list of
    per-problem norm arrays."""
    n = len(rhos)
    if len(outs) != n or (phi0s is not None and len(phi0s) != n):
        raise ValueError("rhos, outs and phi0s must have the same length")
    keep = [np.ascontiguousarray(r, dtype=np.float64) for r in rhos]
    for o in outs:
        if not (o.flags.c_contiguous and o.dtype == np.float64):
            raise ValueError("outs must be C-contiguous float64 arrays")
    VP = ctypes.c_void_p * max(n, 1)
    a_rho = VP(*[r.ctypes.data for r in keep])
    a_out = VP(*[o.ctypes.data for o in outs])
    a_phi = None
    if phi0s is not None:
        keep0 = [None if q is None else np.ascontiguousarray(q, dtype=np.float64) for q in phi0s]
        a_phi = VP(*[None if q is None else q.ctypes.data for q in keep0])
    cap = 0 if norm_every < 0 else ((nsweeps + norm_every - 1) // norm_every if norm_every > 0 else 0) + 1
    norms = np.zeros((max(n, 1), max(cap, 1), 2), dtype=np.float64)
    nw = (ctypes.c_int32 * max(n, 1))()
    opts = px_solve_opts(nsweeps, norm_every, temporal_k, int(use_graph))
    _check(lib().px_solve_host_batch(layout.h, ctypes.byref(p), ctypes.byref(opts), n,
                                     ctypes.cast(a_phi, ctypes.c_void_p) if a_phi is not None else None,
                                     ctypes.cast(a_rho, ctypes.c_void_p), ctypes.cast(a_out, ctypes.c_void_p),
                                     norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap, nw,
                                     _stream(stream)))
    return [norms[i, : nw[i]].copy() for i in range(n)]


def release_cached():
    lib().px_release_cached()


def relax_variant(phi_in: px_patch, phi_out: px_patch, rhs: px_patch, region: px_box) -> int:
    """1 = TMA bulk-copy kernel, 0 = LDG streaming kernel, -1 = invalid."""
    return lib().px_relax_variant(ctypes.byref(phi_in), ctypes.byref(phi_out), ctypes.byref(rhs), region)


def stream_ceiling(a, b, c, variant: int = 0, stream=None):
    """K12 measurement helper: c = a + b (variant 0) or c = a (variant 1)."""
    _check(lib().px_stream_ceiling(_ptr(a), _ptr(b), _ptr(c), c.numel(), variant, _stream(stream)))


def pointwise_update(phi: px_patch, temp: px_patch, rhs: px_patch, lam: float, region: px_box, stream=None):
    """px_pointwise_update: Proto's unfused forallInPlace update (baseline)."""
    _check(lib().px_pointwise_update(ctypes.byref(phi), ctypes.byref(temp), ctypes.byref(rhs), lam, region,
                                     _stream(stream)))


def kernel_launch_count() -> int:
    return lib().px_kernel_launch_count()


def last_solve_kernels() -> str:
    """px_last_solve_kernels: the sweep kernels this thread's last solve enqueued."""
    return lib().px_last_solve_kernels().decode()


# ---------------------------------------------------------------------- 3D
class Grid3:
    """A 3D single-device field layout (px3_layout): allocation size and the
    view of cell (0,0,0) of caller-owned torch float64 tensors."""

    def __init__(self, n, ghost: int = 1):
        self.n = tuple(int(v) for v in n)
        self.ghost = int(ghost)
        ld, plane, org, tot = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().px3_layout((ctypes.c_int32 * 3)(*self.n), self.ghost, ctypes.byref(ld), ctypes.byref(plane),
                                ctypes.byref(org), ctypes.byref(tot)))
        self.ld, self.plane, self.origin, self.alloc_elems = ld.value, plane.value, org.value, tot.value

    def alloc(self, device=None):
        import torch
        return torch.zeros(self.alloc_elems, dtype=torch.float64, device=device or "cuda")

    def patch(self, t) -> px_patch3:
        return px_patch3(t.data_ptr() + 8 * self.origin, (ctypes.c_int32 * 3)(*self.n), self.ghost, self.ld,
                         self.plane)

    def view(self, t, ghosts: bool = False):
        """(n2[+2g], n1[+2g], n0[+2g]) strided view of the cells of t."""
        g = self.ghost if ghosts else 0
        n0, n1, n2 = self.n
        start = self.origin - g * (1 + self.ld + self.plane)
        return t.as_strided((n2 + 2 * g, n1 + 2 * g, n0 + 2 * g), (self.plane, self.ld, 1), start)


def norm_buffer3(device=None):
    import torch
    return torch.zeros(lib().px3_norm_buffer_len(), dtype=torch.float64, device=device or "cuda")


def init_field3(grid: Grid3, t, kind: int, seed: int = 0, stream=None, z0: int = 0):
    """px3_init_field (z0: the global index of the patch's first plane)."""
    p = grid.patch(t)
    _check(lib().px3_init_field(ctypes.byref(p), kind, seed, z0, _stream(stream)))


def fill_ghosts3(grid: Grid3, bc: int, t, stream=None):
    p = grid.patch(t)
    _check(lib().px3_fill_ghosts(bc, ctypes.byref(p), _stream(stream)))


def relax_step3(p: px_relax_params, grid: Grid3, phi_in, phi_out, rhs, norms=None, stream=None):
    a, b, r = grid.patch(phi_in), grid.patch(phi_out), grid.patch(rhs)
    _check(lib().px3_relax_step(ctypes.byref(p), ctypes.byref(a), ctypes.byref(b), ctypes.byref(r), _ptr(norms),
                                _stream(stream)))


def residual_norm3(p: px_relax_params, grid: Grid3, phi, rhs, norms, stream=None):
    a, r = grid.patch(phi), grid.patch(rhs)
    _check(lib().px3_residual_norm(ctypes.byref(p), ctypes.byref(a), ctypes.byref(r), _ptr(norms), _stream(stream)))


def solve3(grid: Grid3, bc: int, p: px_relax_params, nsweeps: int, norm_every: int, phi, phi_scratch, rhs,
           use_graph: bool = False, stream=None, keep_in_scratch: bool = True) -> SolveResult:
    """px3_solve on torch tensors allocated by grid.alloc()."""
    opts = px_solve_opts(nsweeps, norm_every, 1, int(use_graph))
    cap = 0 if norm_every < 0 else ((nsweeps + norm_every - 1) // norm_every if norm_every > 0 else 0) + 1
    norms = np.zeros((max(cap, 1), 2), dtype=np.float64)
    nw, ins = ctypes.c_int32(0), ctypes.c_int32(0)
    a, b, r = grid.patch(phi), grid.patch(phi_scratch), grid.patch(rhs)
    _check(lib().px3_solve(bc, ctypes.byref(p), ctypes.byref(opts), ctypes.byref(a), ctypes.byref(b), ctypes.byref(r),
                           norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), max(cap, 1), ctypes.byref(nw),
                           ctypes.byref(ins) if keep_in_scratch else None, _stream(stream)))
    return SolveResult(norms[: nw.value].copy(), bool(ins.value))


def solve3_host_batch(n, ghost: int, bc: int, p: px_relax_params, nsweeps: int, norm_every: int, rhos, outs,
                      phi0s=None, use_graph: bool = True, stream=None):
    """px3_solve_host_batch: len(rhos) independent 3D problems from host arrays
    (dense (n2, n1, n0) float64; pinned torch CPU tensors via .numpy() for
    overlap), copies overlapped with the solves.  phi0s None (or None entries)
    = zero initial guess.  Returns the list of per-problem norm arrays."""
    k = len(rhos)
    if len(outs) != k or (phi0s is not None and len(phi0s) != k):
        raise ValueError("rhos, outs and phi0s must have the same length")
    shape = (n[2], n[1], n[0])
    keep = [np.ascontiguousarray(r, dtype=np.float64) for r in rhos]
    for a in keep + list(outs) + [q for q in (phi0s or []) if q is not None]:
        if tuple(a.shape) != shape:
            raise ValueError(f"host arrays must have shape {shape}")
    for o in outs:
        if not (o.flags.c_contiguous and o.dtype == np.float64):
            raise ValueError("outs must be C-contiguous float64 arrays")
    VP = ctypes.c_void_p * max(k, 1)
    a_rho = VP(*[r.ctypes.data for r in keep])
    a_out = VP(*[o.ctypes.data for o in outs])
    a_phi = None
    if phi0s is not None:
        keep0 = [None if q is None else np.ascontiguousarray(q, dtype=np.float64) for q in phi0s]
        a_phi = VP(*[None if q is None else q.ctypes.data for q in keep0])
    cap = 0 if norm_every < 0 else ((nsweeps + norm_every - 1) // norm_every if norm_every > 0 else 0) + 1
    norms = np.zeros((max(k, 1), max(cap, 1), 2), dtype=np.float64)
    nw = (ctypes.c_int32 * max(k, 1))()
    opts = px_solve_opts(nsweeps, norm_every, 1, int(use_graph))
    nn = (ctypes.c_int32 * 3)(*n)
    _check(lib().px3_solve_host_batch(bc, ctypes.byref(p), ctypes.byref(opts), nn, ghost, k,
                                      ctypes.cast(a_phi, ctypes.c_void_p) if a_phi is not None else None,
                                      ctypes.cast(a_rho, ctypes.c_void_p), ctypes.cast(a_out, ctypes.c_void_p),
                                      norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), max(cap, 1), nw,
                                      _stream(stream)))
    return [norms[i, : nw[i]].copy() for i in range(k)]


def mehrstellen_rhs3(grid: Grid3, rho, f, stream=None):
    """px3_mehrstellen_rhs: f = ρ + S7(ρ)/12 (ρ's ghosts filled)."""
    a, b = grid.patch(rho), grid.patch(f)
    _check(lib().px3_mehrstellen_rhs(ctypes.byref(a), ctypes.byref(b), _stream(stream)))


def slab3(n2: int, nranks: int, rank: int):
    """px3_slab: the planes [z0, z1) rank owns of an n2-plane domain."""
    z0, z1 = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().px3_slab(n2, nranks, rank, ctypes.byref(z0), ctypes.byref(z1)))
    return z0.value, z1.value


def solve3_comm(comm, grid: Grid3, bc: int, p: px_relax_params, nsweeps: int, norm_every: int, phi, phi_scratch,
                rhs, use_graph: bool = False, stream=None, keep_in_scratch: bool = True) -> SolveResult:
    """px3_solve_comm: this rank's z-slab (grid.n[2] = its planes) of a domain split over comm."""
    opts = px_solve_opts(nsweeps, norm_every, 1, int(use_graph))
    cap = 0 if norm_every < 0 else ((nsweeps + norm_every - 1) // norm_every if norm_every > 0 else 0) + 1
    norms = np.zeros((max(cap, 1), 2), dtype=np.float64)
    nw, ins = ctypes.c_int32(0), ctypes.c_int32(0)
    a, b, r = grid.patch(phi), grid.patch(phi_scratch), grid.patch(rhs)
    _check(lib().px3_solve_comm(comm.h, bc, ctypes.byref(p), ctypes.byref(opts), ctypes.byref(a), ctypes.byref(b),
                                ctypes.byref(r), norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), max(cap, 1),
                                ctypes.byref(nw), ctypes.byref(ins) if keep_in_scratch else None, _stream(stream)))
    return SolveResult(norms[: nw.value].copy(), bool(ins.value))


def release3():
    lib().px3_release()
