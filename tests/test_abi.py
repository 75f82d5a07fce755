"""CPU tests of the C ABI: libprotox loads without a GPU, exports every
function include/protox.h declares, and its host logic (geometry, layout /
slab partitioner, halo plan, validation errors) is right.  No compute calls."""
import ctypes
import os
import re

import pytest

from paper_2307_07931_b200 import protox as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "protox.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(px3?_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_function():
    names = header_functions()
    assert len(names) >= 30
    L = P.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(P.EXPORTS)
    assert L.px_api_version() == 1


def test_status_strings():
    for s in range(9):
        assert P.lib().px_status_str(s).decode().startswith("PX_")


def test_box_geometry_fig_protox_constants():
    """Fig. ProtoX: a 64x64 box with one ghost layer."""
    b = P.box_grow(P.box(0, 0, 63, 63), 1)
    assert b.tuple() == (-1, -1, 64, 64) and P.box_size(b) == 66 * 66
    assert P.box_ordinal(b, P.point(0, 0)) == 67
    assert P.box_ordinal(b, P.point(1, 0)) == 68
    assert P.box_ordinal(b, P.point(0, 1)) == 133
    assert P.box_ordinal(b, P.point(-1, 0)) == 66
    assert P.box_ordinal(b, P.point(0, -1)) == 1
    with pytest.raises(P.PxError, match="PX_ERR_DOMAIN"):
        P.box_ordinal(b, P.point(65, 0))
    assert P.box_is_empty(P.box_grow(P.box(0, 0, 1, 1), -1))
    assert P.box_size(P.box_grow(P.box(0, 0, 1, 1), -1)) == 0
    assert P.box_intersect(P.box(0, 0, 3, 3), P.box(2, 2, 5, 5)).tuple() == (2, 2, 3, 3)
    assert P.box_is_empty(P.box_intersect(P.box(0, 0, 1, 1), P.box(5, 5, 6, 6)))


@pytest.mark.parametrize("n,box,nranks", [(16384, 256, 8), (16384, 256, 3), (32768, 256, 8),
                                          (150, 10, 4), (64, 64, 1)])
def test_layout_slabs_cover_domain(n, box, nranks):
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (box, box), 1, P.PX_BC_PERIODIC, nranks)
    assert lay.num_boxes() == (n // box) ** 2
    rows = []
    for r in range(nranks):
        li = lay.local(r)
        assert li.owned.lo.c[0] == 0 and li.owned.hi.c[0] == n - 1
        assert (li.owned.hi.c[1] - li.owned.lo.c[1] + 1) % box == 0
        rows.append((li.owned.lo.c[1], li.owned.hi.c[1]))
        assert li.ld % 16 == 0 and li.ld >= 16 + n + 1
        assert li.patch_offset == 15
        assert li.alloc_elems == li.ld * (li.owned.hi.c[1] - li.owned.lo.c[1] + 3)
        assert li.nbr_lo == (r - 1) % nranks and li.nbr_hi == (r + 1) % nranks
    assert rows[0][0] == 0 and rows[-1][1] == n - 1
    assert all(rows[i][1] + 1 == rows[i + 1][0] for i in range(nranks - 1))
    sizes = [b - a + 1 for a, b in rows]
    assert max(sizes) - min(sizes) <= box
    # box ownership agrees with the slabs
    for i in range(0, lay.num_boxes(), max(1, lay.num_boxes() // 97)):
        b, owner = lay.box(i)
        lo, hi = rows[owner]
        assert lo <= b.lo.c[1] and b.hi.c[1] <= hi


def test_layout_dirichlet_faces_have_no_neighbour():
    lay = P.Layout(P.box(0, 0, 255, 255), (64, 64), 1, P.PX_BC_DIRICHLET_CC, 4)
    assert lay.local(0).nbr_lo == -1 and lay.local(3).nbr_hi == -1
    assert lay.local(1).nbr_lo == 0 and lay.local(1).nbr_hi == 2


def test_halo_plan_pairs_match_in_posting_order():
    """The k-th send from a to b fills b's k-th receive from a, row-adjacent."""
    for nranks in (2, 3, 4, 8):
        for bc in (P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC):
            g = 2
            lay = P.Layout(P.box(0, 0, 99, 8 * 16 - 1), (20, 16), g, bc, nranks)
            plans = {r: lay.halo_plan(r) for r in range(nranks)}
            for r in range(nranks):
                li = lay.local(r)
                for k, op in enumerate(plans[r]):
                    assert op.count == (g - 1) * li.ld + (100 + 2 * g) and op.nrows == g
                    assert op.offset == (op.row - li.alloc.lo.c[1]) * li.ld
                    if not op.is_recv:
                        continue
                    kk = sum(1 for o in plans[r][:k] if o.is_recv and o.peer == op.peer)
                    sends = [o for o in plans[op.peer] if not o.is_recv and o.peer == r]
                    src = sends[kk]
                    # the ghost rows received are (periodic images of) the rows sent
                    assert (op.row - src.row) % (8 * 16) == 0
            if bc == P.PX_BC_DIRICHLET_CC:
                assert all(o.peer != nranks - 1 for o in plans[0] if o.row < 0)
    assert P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, P.PX_BC_PERIODIC, 1).halo_plan(0) == []


def test_layout_errors():
    with pytest.raises(P.PxError, match="PX_ERR_SHAPE"):
        P.Layout(P.box(0, 0, 99, 99), (64, 64))
    with pytest.raises(P.PxError, match="PX_ERR_ARG"):
        P.Layout(P.box(0, 0, 63, 63), (64, 64), 0)
    with pytest.raises(P.PxError, match="PX_ERR_SHAPE"):
        P.Layout(P.box(0, 0, 63, 63), (8, 8), 9)
    with pytest.raises(P.PxError, match="PX_ERR_ARG"):
        P.Layout(P.box(0, 0, 63, 63), (64, 32), 1, P.PX_BC_PERIODIC, 3)
    with pytest.raises(P.PxError, match="PX_ERR_SHAPE"):
        P.Layout(P.box(5, 5, 4, 4), (1, 1))
    with pytest.raises(P.PxError, match="PX_ERR_ARG"):
        P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, 7)
    lay = P.Layout(P.box(0, 0, 63, 63), (32, 32), 1, P.PX_BC_PERIODIC, 2)
    with pytest.raises(P.PxError, match="rank 2 out of range"):
        lay.local(2)
    with pytest.raises(P.PxError, match="PX_ERR_ARG"):
        lay.box(4)


def test_validation_rejects_bad_patches_before_any_launch():
    """Argument errors are detected on the host (no GPU touched)."""
    lay = P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, P.PX_BC_PERIODIC, 1)
    li = lay.local(0)
    fake = 1 << 40  # never dereferenced: validation fails first
    good = P.px_patch(fake + 8 * li.patch_offset, li.alloc, li.ld)
    prm = P.relax_params(1.0 / 64, 1e-5)
    # null data
    with pytest.raises(P.PxError, match="null data"):
        P.relax_step(prm, P.px_patch(None, li.alloc, li.ld), good, good, li.owned, stream=0)
    # odd ld
    with pytest.raises(P.PxError, match="PX_ERR_ALIGN"):
        P.relax_step(prm, P.px_patch(fake, li.alloc, 67), good, good, li.owned, stream=0)
    # stencil domain violation names the first point/tap in scan order
    small = P.px_patch(fake, P.box(0, 0, 63, 63), li.ld)
    with pytest.raises(P.PxError, match=r"i=\(0,0\) tap=\(-1,0\)"):
        P.relax_step(prm, small, good, good, li.owned, stream=0)
    with pytest.raises(P.PxError, match=r"i=\(1,1\) tap=\(0,1\)"):
        P.stencil_apply(0, 1.0, P.px_patch(fake, P.box(0, 0, 63, 1), li.ld), good, P.box(1, 1, 62, 1), stream=0)
    # bad stencil / h
    with pytest.raises(P.PxError, match="bad stencil"):
        P.relax_step(P.relax_params(1.0, 1.0, 7), good, good, good, li.owned, stream=0)
    with pytest.raises(P.PxError, match="h must be positive"):
        P.relax_step(P.relax_params(0.0, 1.0), good, good, good, li.owned, stream=0)
    # solve: temporal k beyond the ghost width, negative sweeps
    with pytest.raises(P.PxError):
        P.solve(lay, None, 0, prm, -1, 1, good, good, good, stream=0)


def test_norm_buffer_len_positive():
    assert P.norm_buffer_len(P.box(0, 0, 16383, 16383)) > 4
    assert P.norm_buffer_len(P.box(0, 0, 0, 0)) >= 6


def test_px3_layout_and_slabs_host_only():
    """3D host-side geometry without a GPU: the layout pitches (x origin at
    element 16, 16-aligned rows) and the z-slab partitioner."""
    g = P.Grid3((70, 37, 13), 1)
    assert g.ld % 16 == 0 and g.ld >= 70 + 32
    assert g.plane == g.ld * (37 + 2)
    assert g.origin == 16 + g.ld + g.plane
    assert g.alloc_elems == g.plane * (13 + 2)
    for world in (1, 2, 3, 8):
        spans = [P.slab3(512, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 512
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(P.PxError, match="planes"):
        P.slab3(2, 3, 0)
    with pytest.raises(P.PxError):
        P.slab3(16, 2, 2)
    with pytest.raises(P.PxError):
        P.Grid3((0, 4, 4), 1)
