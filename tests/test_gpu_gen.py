"""Config-5 generator: the device-built counter-based cluster Hamiltonian is
bitwise the host reference (synth.cluster_dense_cb)."""

import numpy as np
import pytest

from conftest import pyramid_flat

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import cluster_dense_cb, cluster_sites, device_cluster  # noqa: E402


@pytest.mark.parametrize("n_mol,nb", [(20, 16), (30, 64), (7, 4)])
def test_device_cluster_bitwise(n_mol, nb):
    cs = cluster_sites(n_mol, seed=11)
    h = cluster_dense_cb(cs)
    assert np.array_equal(h, h.T)
    x = device_cluster(cs, nb)
    ref = sp.build_from_dense(h, nb)
    assert np.array_equal(sp.to_dense(x), h)
    assert np.array_equal(x._block_keys, ref._block_keys)
    assert np.array_equal(pyramid_flat(x._tier_norms), pyramid_flat(ref._tier_norms))
    assert x.symmetric and ref.symmetric
    c1, s1 = sp.multiply(x, x, 1e-6)
    c2, s2 = sp.multiply(ref, ref, 1e-6)
    assert s1.counts_equal(s2)
    assert np.array_equal(sp.to_dense(c1), sp.to_dense(c2))
