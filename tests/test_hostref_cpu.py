"""The host re-run of the paper's CPU experiment (hostref/, SURVEY §8(f) rank
4) computes the method: the unfused Proto variant is bit-identical to the
oracle (same expression tree), the fused ProtoX transcription (Fig. ProtoX's
tree) agrees with it to rounding, for 1 and several OpenMP threads."""
import numpy as np
import pytest

import hostref
import oracle
from paper_2307_07931_b200 import inputs


@pytest.mark.parametrize("threads", [1, 3])
def test_unfused_bitwise_and_fused_to_rounding(threads):
    box, nb, N = 16, 4, 30
    n = box * nb
    h = 1.0 / n
    lam = h * h / 8
    rho = inputs.hash_field(n, n)
    p = oracle.Problem(n, n, h, lam, b0=box, b1=box, bc=oracle.BC_PERIODIC, nsweeps=N, norm_every=1)
    ref, rn = oracle.solve(p, np.zeros(p.gshape), oracle.ghosted(p, rho))
    ref = ref[1:-1, 1:-1]
    u, _, hu = hostref.run(0, box, nb, N, h, lam, rho, threads)
    assert np.array_equal(u.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(hu, rn[1:, 0])  # Proto records the post-update residual
    f, _, hf = hostref.run(1, box, nb, N, h, lam, rho, threads)
    assert np.max(np.abs(f - ref)) <= 1e-12 * np.max(np.abs(ref))
    np.testing.assert_allclose(hf, rn[:-1, 0], rtol=1e-12)  # fused: pre-update residual
