"""Race probes in place of compute-sanitizer (refused by the GPU pool,
profiles/sanitizer_r02.txt): every leaf kernel on small and large inputs,
run many times back to back, must give bitwise the same product -- a stage
released too early, a TMEM tile read before its MMAs retired or an epilogue
exchange overwritten shows up as a differing block (the round-1 K4 race was
~1 corrupted block in 40 launches)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster  # noqa: E402


def _inputs(which):
    if which == "cfg3x0":
        cfg = CONFIGS[3]
        h, _ = water_cluster(cfg.n_mol, seed=0)
        f = sp.build_from_dense(h, 32)
        x = sp.sp2_init(f, sp.gershgorin_bounds(f))
        return x, x, cfg.tau
    nb = 64 if which == "nb64" else 32
    da, db = decay_pair(1024, 0.1, (0, 1))
    return sp.build_from_dense(da, nb), sp.build_from_dense(db, nb), 1e-8


@pytest.mark.parametrize("which", ["cfg1", "nb64", "cfg3x0"])
@pytest.mark.parametrize("kernel", ["dmma", "ozaki", "exact"])
def test_repeated_products_bitwise(which, kernel):
    a, b, tau = _inputs(which)
    reps = 4 if kernel == "exact" else 30
    ref, _ = sp.multiply(a, b, tau, kernel=kernel)
    r0 = ref.blocks_device().clone()
    for _ in range(reps):
        c, _ = sp.multiply(a, b, tau, kernel=kernel)
        assert torch.equal(c.blocks_device(), r0)
    assert np.isfinite(sp.to_dense(ref)).all()
