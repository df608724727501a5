"""Full parity of the DEFAULT leaf kernel (kernel="auto": K4z, the INT8 digit
products, at Nb 32 and 64) against the CPU oracle run live on the box, at the
BASELINE configs 1-4.  The north-star contract: surviving task sets exact
(documented near-tau ties aside), C and the SP2 density matrix within a
relative Frobenius error of 1e-12, identical SP2 iteration counts.

* C of cfg1 (A.B), cfg2 (H.H) and cfg4 (X0^2) compared in full;
* final P of cfg3 / cfg4 (criterion ||X^2 - X||_F < 1e-6) compared in full to
  the oracle's own SP2 run (same iterations and branches);
* every SP2 iteration's task set on the default path compared (sha256 of the
  sorted task keys) with the reference's, from tests/golden (made by the
  reference, tests/golden/make_golden.py), together with the near-tau
  report (kernel.py:108) and the branch margin (sp2.py:97-99);
* the near-tau report itself checked against oracle.tie_log on constructed
  exact ties, for the dense cull, the tier walk and the symmetric path."""

import os

import numpy as np
import pytest

from conftest import golden, pyramid_flat
from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.sp2 import _native_step  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster  # noqa: E402

REL_FRO_TOL = 1e-12
THREADS = os.cpu_count() or 1


def rel_fro(x, ref):
    return np.linalg.norm(x - ref) / np.linalg.norm(ref)


def _keys(t, g):
    ti, tk, tj = t
    return np.sort((ti * g + tk) * g + tj)


def _check_product(a, b, oa, ob, tau, gd=None):
    c, st = sp.multiply(a, b, tau)                       # default kernel
    oc, ost, otasks = O.multiply(oa, ob, tau, threads=THREADS)
    assert st.visited == ost["visited"] and st.culled == ost["culled"]
    g = a.n_blocks
    assert np.array_equal(_keys(sp.leaf_tasks(a, b, tau), g), _keys(otasks, g))
    assert np.array_equal(c._block_keys, oc.keys)
    err = rel_fro(sp.to_dense(c), O.to_dense(oc))
    assert err <= REL_FRO_TOL, err
    near, margin = O.tie_log(oa.tier_norms, ob.tier_norms, tau, st.near_tau_ulps)
    assert list(st.near_tau) == near and st.tau_margin == margin
    if gd is not None:
        assert sum(st.near_tau) == int(gd["near_tau"])
        assert st.tau_margin == float(gd["tau_margin"])
    return st, err


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_product_full_c_default_kernel(name):
    gd = golden(name)
    cfg = CONFIGS[1 if name == "cfg1" else 2]
    if name == "cfg1":
        da, db = decay_pair(cfg.n, 0.1, (0, 1))
    else:
        da, _ = water_cluster(cfg.n_mol, seed=0)
        db = da
    a = sp.build_from_dense(da, cfg.block_size)
    b = a if db is da else sp.build_from_dense(db, cfg.block_size)
    oa = O.from_dense(da, cfg.block_size)
    ob = oa if db is da else O.from_dense(db, cfg.block_size)
    st, _ = _check_product(a, b, oa, ob, cfg.tau, gd)
    assert st.leaf_products == int(gd["leaf_products"])


def test_cfg4_x0_square_full_c_default_kernel():
    cfg = CONFIGS[4]
    h, _ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x0 = sp.sp2_init(f, sp.gershgorin_bounds(f))
    of = O.from_dense(h, cfg.block_size)
    ox0 = O.sp2_init(of, O.gershgorin_bounds(of))
    assert np.array_equal(pyramid_flat(x0._tier_norms), pyramid_flat(ox0.tier_norms))
    st, _ = _check_product(x0, x0, ox0, ox0, cfg.tau)
    assert st.symmetric and st.leaf_products == int(golden("cfg4_sp2")["leaf_products"][0])


@pytest.mark.parametrize("cfg_index", [3, 4])
def test_sp2_full_p_default_kernel_vs_live_oracle(cfg_index):
    cfg = CONFIGS[cfg_index]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    p, st = sp.sp2_solve(sp.build_from_dense(h, cfg.block_size), n_occ, cfg.tau,
                         criterion="fro", fro_tol=1e-6)
    r = O.sp2_solve(O.from_dense(h, cfg.block_size), n_occ, cfg.tau, threads=THREADS,
                    criterion="fro", fro_tol=1e-6)
    assert st.converged and r.converged
    assert st.iteration == r.iterations
    assert st.branch_history == r.branches
    assert list(st.leaf_products) == list(r.leaf_products)
    ref = O.to_dense(r.x)
    err = rel_fro(sp.to_dense(p), ref)
    assert err <= REL_FRO_TOL, err
    # the branch rule's margins: same decisions with margins far above the
    # trace rounding (the converging multiply's branch is discarded)
    bm, rbm = np.array(st.branch_margins), np.array(r.branch_margins)
    assert np.array_equal(np.sign(bm[:-1]), np.sign(rbm[:-1]))
    assert np.min(np.abs(rbm[:-1])) > 1e-7
    assert np.max(np.abs(bm - rbm)) < 1e-9
    assert len(st.wall_seconds_per_iteration) == len(st.leaf_products)
    assert all(w > 0 for w in st.wall_seconds_per_iteration)


@pytest.mark.parametrize("name,cfg_index", [("cfg3_sp2", 3), ("cfg4_sp2", 4)])
def test_sp2_task_set_of_every_iteration_equals_reference(name, cfg_index):
    gd = golden(name)
    cfg = CONFIGS[cfg_index]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    n_mult = len(gd["task_sha256"])
    for k in range(n_mult):
        ti, tk, tj = sp.leaf_tasks(x, x, cfg.tau)
        assert O.task_sha256(ti, tk, tj, x.n_blocks) == bytes(gd["task_sha256"][k]).hex(), k
        x_next, branch, t_x, t_sq, idem, stats = _native_step(x, n_occ, cfg.tau, "auto", True)
        assert stats.leaf_products == int(gd["leaf_products"][k])
        # no tested product within 64 ulps of tau on either side
        assert sum(stats.near_tau) == int(gd["near_tau"][k]) == 0
        assert np.isinf(stats.tau_margin) == np.isinf(gd["tau_margin"][k])
        bm = abs((2.0 * t_x - t_sq) - n_occ) - abs(t_sq - n_occ)
        assert abs(bm - float(gd["branch_margin"][k])) < 1e-9
        if idem < 1e-6:
            assert k == n_mult - 1
            break
        assert (branch == sp.SQUARE) == bool(gd["branches"][k])
        x = x_next
    else:
        pytest.fail("did not converge within the reference's multiply count")


# -- the near-tau report on constructed ties ----------------------------------

def _tied_pair(rng, n, nb):
    a = rng.standard_normal((n, n))
    a[np.abs(a) < 0.9] = 0.0
    return a


@pytest.mark.parametrize("mode", ["dense", "walk", "sym"])
def test_near_tau_report_matches_oracle_on_exact_ties(rng, mode):
    nb = 4
    da = _tied_pair(rng, 48, nb)
    if mode == "sym":
        da = np.triu(da) + np.triu(da, 1).T
        db = da
    else:
        db = _tied_pair(rng, 48, nb)
    a = sp.build_from_dense(da, nb)
    b = a if db is da else sp.build_from_dense(db, nb)
    oa = O.from_dense(da, nb)
    ob = oa if db is da else O.from_dense(db, nb)
    leaf_a, leaf_b = oa.tier_norms[-1], ob.tier_norms[-1]
    # tau = an actual leaf product (an exact tie), and one ulp either side
    p = float(leaf_a[1, 2] * leaf_b[2, 3])
    assert p > 0
    for tau in (p, np.nextafter(p, 0), np.nextafter(p, np.inf), p * (1 + 1e-9)):
        if mode == "walk":
            sp.set_dense_cull(False)
        try:
            c, st = sp.multiply(a, b, tau, kernel="exact")
            cs = sp.convolution_census(a, b, tau)
        finally:
            sp.set_dense_cull(True)
        near, margin = O.tie_log(oa.tier_norms, ob.tier_norms, tau, st.near_tau_ulps)
        assert list(st.near_tau) == near and st.tau_margin == margin, (tau, st.near_tau, near)
        assert list(cs.near_tau) == near
        if tau in (p, np.nextafter(p, 0), np.nextafter(p, np.inf)):
            assert sum(near) >= 1 and margin <= 2 ** -50
        oc, ost, _ = O.multiply(oa, ob, tau)
        assert st.visited == ost["visited"]
        assert np.array_equal(sp.to_dense(c), O.to_dense(oc))
    # the band width is a setting
    sp.set_near_tau_ulps(0)
    try:
        _, st0 = sp.multiply(a, b, p, kernel="exact")
        assert list(st0.near_tau) == O.tie_log(oa.tier_norms, ob.tier_norms, p, 0)[0]
        assert st0.near_tau_ulps == 0
    finally:
        sp.set_near_tau_ulps(64)
