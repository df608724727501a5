"""SpAMM on the GPU vs the reference semantics (kernel.py): the reference's
own kernel tests ported to the new API, golden-fixture parity, the compiled
seam gemm_batch, and properties at full config sizes.

Tolerances (BASELINE north_star): surviving task set exact; C within a
relative Frobenius error of 1e-12 (DMMA rounding differs from the
reference's unfused i-k-j loop); the "exact" leaf kernel is bitwise."""

import os

import numpy as np
import pytest
import torch

from conftest import golden, pyramid_flat
from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster  # noqa: E402

REL_FRO_TOL = 1e-12


def rel_fro(x, ref):
    den = np.linalg.norm(ref)
    return np.linalg.norm(x - ref) / den if den > 0 else np.linalg.norm(x)


# -- leaf_gemm (kernel.py:80-93) ------------------------------------------------

def test_leaf_gemm_known_answers(rng):
    c = np.zeros((4, 4))
    sp.leaf_gemm(np.eye(4), np.eye(4), c)
    assert np.array_equal(c, np.eye(4))
    a, b = np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0], [7.0, 8.0]])
    c = np.zeros((2, 2))
    out = sp.leaf_gemm(a, b, c)
    assert np.array_equal(out, golden("small_cases")["hand_example"]) and out is c
    a, b, c0 = (rng.standard_normal((16, 16)) for _ in range(3))
    assert np.array_equal(sp.leaf_gemm(a, b, c0.copy()), O.leaf_gemm(a, b, c0.copy()))
    with pytest.raises(ValueError):
        sp.leaf_gemm(np.eye(4), np.eye(3), np.zeros((4, 4)))


# -- multiply correctness (reference test_kernel.py) ----------------------------

def test_identity_multiply_is_exact(rng):
    dense = rng.standard_normal((24, 24))
    x = sp.build_from_dense(dense, block_size=4)
    c, stats = sp.multiply(sp.identity(24, 4), x, 0.0)
    assert np.array_equal(sp.to_dense(c), dense)
    assert stats.leaf_products == x.stored_leaf_count


@pytest.mark.parametrize("nb", [4, 8, 16, 32, 64])
def test_multiply_matches_dense(rng, nb):
    n = 3 * nb + 5
    da, db = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    c, _ = sp.multiply(sp.build_from_dense(da, nb), sp.build_from_dense(db, nb), 0.0)
    ref = np.einsum("ik,kj->ij", da, db)
    assert np.abs(sp.to_dense(c) - ref).max() <= 1e-13 * np.linalg.norm(da) * np.linalg.norm(db)


def test_root_occlusion(rng):
    a = sp.build_from_dense(rng.standard_normal((16, 16)), block_size=4)
    c, stats = sp.multiply(a, a, a.norm() * a.norm() + 1.0)
    assert np.array_equal(sp.to_dense(c), np.zeros((16, 16)))
    assert stats.leaf_products == 0 and all(v == 0 for v in stats.visited)
    assert stats.culled[0] == 1 and c.stored_leaf_count == 0


def test_error_nonincreasing_as_tau_decreases():
    n = 128
    idx = np.arange(n)
    u = np.random.default_rng(2).uniform(0.5, 1.0, (n, n))
    dense = 0.6 ** np.abs(idx[:, None] - idx[None, :]) * (np.triu(u) + np.triu(u, 1).T)
    tree = sp.build_from_dense(dense, block_size=8)
    ref = np.einsum("ik,kj->ij", dense, dense)
    errors = [np.abs(sp.to_dense(sp.multiply(tree, tree, tau)[0]) - ref).max()
              for tau in (1e-4, 1e-6, 1e-8, 1e-10, 0.0)]
    assert all(e1 >= e2 - 1e-18 for e1, e2 in zip(errors, errors[1:]))
    assert errors[-1] <= 1e-13 * tree.norm() ** 2


def test_census_equals_multiply_counts_and_recursion(rng):
    dense = rng.standard_normal((32, 32))
    dense[np.abs(dense) < 0.8] = 0.0
    tree = sp.build_from_dense(dense, block_size=4)
    for tau in (0.0, 1e-3, 0.5, 5.0):
        census = sp.convolution_census(tree, tree, tau)
        _, stats = sp.multiply(tree, tree, tau)
        assert census.counts_equal(stats) and census.flop_estimate == stats.flop_estimate
        ot = O.from_dense(dense, 4)
        v, c, i, _, _ = O.sweep(ot.tier_norms, ot.tier_norms, tau)
        assert census.visited == tuple(v) and census.culled == tuple(c)
        assert census.leaf_products == len(i)


def test_dense_and_diagonal_census():
    tree = sp.build_from_dense(np.full((16, 16), 1.0), block_size=4)
    stats = sp.convolution_census(tree, tree, 0.0)
    assert stats.visited == (1, 8, 64) and stats.leaf_products == 8 ** tree.depth
    diag = sp.build_from_dense(np.diag(np.arange(1.0, 17.0)), block_size=4)
    assert sp.convolution_census(diag, diag, 0.0).leaf_products == diag.stored_leaf_count


def test_stats_structural_invariants():
    n = 64
    idx = np.arange(n)
    dense = 0.5 ** np.abs(idx[:, None] - idx[None, :])
    tree = sp.build_from_dense(dense, block_size=4)
    leaf = tree._tier_norms[-1]
    tau = leaf[leaf > 0].min() ** 2 * 10
    stats = sp.convolution_census(tree, tree, tau)
    for t, (v, c) in enumerate(zip(stats.visited, stats.culled)):
        assert v + c <= 8 ** t
        if t:
            assert stats.visited[t] <= 8 * stats.visited[t - 1]
    assert stats.flop_estimate == stats.leaf_products * 2 * 4 ** 3 and sum(stats.culled) > 0


def test_mode_chunk_and_run_to_run_determinism(rng):
    da, db = rng.standard_normal((48, 48)), rng.standard_normal((48, 48))
    for chunk in (8, 16, 64):
        a = sp.build_from_dense(da, block_size=4, chunk_size=chunk)
        b = sp.build_from_dense(db, block_size=4, chunk_size=chunk)
        for tau in (0.0, 1e-2):
            serial, s_stats = sp.multiply(a, b, tau, mode="serial")
            for workers in (2, 8):
                tasked, t_stats = sp.multiply(a, b, tau, mode="tasked", workers=workers)
                assert np.array_equal(sp.to_dense(serial), sp.to_dense(tasked))
                assert s_stats.counts_equal(t_stats)
            c3, _ = sp.multiply(a, b, tau, mode="tasked", deterministic=False, workers=4)
            assert np.array_equal(sp.to_dense(serial), sp.to_dense(c3))


def test_multiply_validation():
    a, b = sp.build_from_dense(np.eye(8), 2), sp.build_from_dense(np.eye(16), 2)
    with pytest.raises(ValueError):
        sp.multiply(a, b, 0.0)
    for bad in (-1.0, float("inf"), float("nan")):
        with pytest.raises(ValueError):
            sp.multiply(a, a, bad)
    with pytest.raises(ValueError):
        sp.multiply(a, a, 0.0, mode="parallel")
    with pytest.raises(ValueError):
        sp.multiply(a, a, 0.0, mode="tasked", workers=0)
    with pytest.raises(ValueError):
        sp.multiply(a, a, 0.0, kernel="dmma")  # Nb = 2 has no DMMA tiling


def test_linear_scaling_trend():
    counts = []
    for n in (256, 512, 1024):
        idx = np.arange(n)
        u = np.random.default_rng(11).uniform(0.5, 1.0, (n, n))
        d = 0.7 ** np.abs(idx[:, None] - idx[None, :]) * (np.triu(u) + np.triu(u, 1).T)
        tree = sp.build_from_dense(d, block_size=16)
        counts.append(sp.convolution_census(tree, tree, 1e-8).leaf_products)
    ratios = [b / a for a, b in zip(counts, counts[1:])]
    assert all(1.5 <= r <= 3.0 for r in ratios), ratios


def test_stats_json_schema(rng):
    a = sp.build_from_dense(rng.standard_normal((16, 16)), block_size=4)
    payload = sp.multiply(a, a, 1e-2)[1].to_json_dict()
    assert set(payload) == {"tau", "tiers", "leaf_products", "flop_estimate", "wall_seconds"}
    assert payload["tiers"][0].keys() == {"t", "visited", "culled"} and payload["tau"] == 1e-2


# -- golden fixtures (reference outputs) ---------------------------------------

def test_golden_small_cases():
    g = golden("small_cases")
    for idx in range(int(g["n_small"])):
        nb = int(g[f"s{idx}_nb"])
        a, b = sp.build_from_dense(g[f"s{idx}_a"], nb), sp.build_from_dense(g[f"s{idx}_b"], nb)
        for tau in (0.0, 1e-2, 1.0):
            key = f"s{idx}_t{tau:g}"
            ce, st = sp.multiply(a, b, tau, kernel="exact")
            assert st.visited == tuple(g[key + "_visited"]) and st.culled == tuple(g[key + "_culled"])
            assert np.array_equal(sp.to_dense(ce), g[key + "_c"]), key
            assert np.array_equal(pyramid_flat(ce._tier_norms), g[key + "_cpyr"]), key
            assert sp.trace(ce) == float(g[key + "_trace"])
            c, _ = sp.multiply(a, b, tau)
            assert rel_fro(sp.to_dense(c), g[key + "_c"]) <= REL_FRO_TOL


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_golden_product_configs(name):
    gd = golden(name)
    cfg = CONFIGS[1 if name == "cfg1" else 2]
    if name == "cfg1":
        da, db = decay_pair(cfg.n, 0.1, (0, 1))
    else:
        da, _ = water_cluster(cfg.n_mol, seed=0)
        db = da
    a, b = sp.build_from_dense(da, cfg.block_size), sp.build_from_dense(db, cfg.block_size)
    ti, tk, tj = sp.leaf_tasks(a, b, cfg.tau)
    g = a.n_blocks
    assert np.array_equal(np.sort((ti * g + tk) * g + tj), gd["task_keys"])   # exact task set
    c, st = sp.multiply(a, b, cfg.tau)
    assert st.visited == tuple(gd["visited"]) and st.culled == tuple(gd["culled"])
    assert st.flop_estimate == int(gd["flop_estimate"])
    assert np.array_equal(c._block_keys, gd["c_keys"])
    pos = np.searchsorted(c._block_keys, gd["c_sample_keys"])
    assert rel_fro(c._block_data[pos], gd["c_sample_blocks"]) <= REL_FRO_TOL
    leaf = c._tier_norms[-1]
    ref_leaf = gd["c_pyramid"][-leaf.size:].reshape(leaf.shape)
    assert rel_fro(leaf, ref_leaf) <= REL_FRO_TOL
    assert abs(sp.trace(c) - float(gd["c_trace"])) <= 1e-12 * abs(float(gd["c_trace"]))
    ce, _ = sp.multiply(a, b, cfg.tau, kernel="exact")
    assert np.array_equal(pyramid_flat(ce._tier_norms), gd["c_pyramid"])
    assert sp.trace(ce) == float(gd["c_trace"])
    assert np.array_equal(ce._block_data[pos], gd["c_sample_blocks"])


# -- the compiled seam gemm_batch (kernel.py:74-77) -----------------------------

@pytest.mark.parametrize("nb", [2, 8, 32, 64])
def test_gemm_batch_seam(rng, nb):
    m_a, m_b, m_c = 9, 7, 5
    a = rng.standard_normal((m_a, nb, nb))
    b = rng.standard_normal((m_b, nb, nb))
    c0 = rng.standard_normal((m_c, nb, nb))
    n = 40
    c_pos = np.sort(rng.integers(0, m_c, n))
    c_pos = np.array([3, 0, 4, 1, 2])[c_pos]      # contiguous runs, not ascending
    a_pos, b_pos = rng.integers(0, m_a, n), rng.integers(0, m_b, n)
    ref = c0.copy()
    O.gemm_batch(a_pos, b_pos, c_pos, a, b, ref, threads=1)
    dev = lambda x, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(x), dtype=dt).cuda()
    for kern in ("exact", "auto"):
        if kern == "auto" and nb not in (8, 16, 32, 64):
            continue
        out = dev(c0)
        sp.gemm_batch(dev(a_pos, torch.int64), dev(b_pos, torch.int64), dev(c_pos, torch.int64),
                      dev(a), dev(b), out, kernel=kern)
        got = out.cpu().numpy()
        if kern == "exact":
            assert np.array_equal(got, ref)
        else:
            assert rel_fro(got, ref) <= REL_FRO_TOL


# -- symmetric SpAMM (X*X with X == X^T) -------------------------------------------

def _sym(rng, n, thr=0.0):
    d = rng.standard_normal((n, n))
    d = np.triu(d) + np.triu(d, 1).T
    d[np.abs(d) < thr] = 0.0
    return d


@pytest.mark.parametrize("nb,kernel", [(4, "exact"), (8, "auto"), (32, "auto"), (32, "exact"),
                                       (64, "auto"), (64, "exact")])
def test_symmetric_path_bitwise_equals_full(rng, nb, kernel):
    d = _sym(rng, 5 * nb + 7, 0.7)
    x = sp.build_from_dense(d, nb)
    assert x.symmetric
    for tau in (0.0, 0.3, 3.0):
        c_sym, st_sym = sp.multiply(x, x, tau, kernel=kernel)
        sp.set_symmetric_products(False)
        try:
            c_full, st_full = sp.multiply(x, x, tau, kernel=kernel)
        finally:
            sp.set_symmetric_products(True)
        assert st_sym.symmetric and not st_full.symmetric
        assert st_sym.counts_equal(st_full) and st_sym.flop_estimate == st_full.flop_estimate
        assert st_sym.executed_products <= st_full.executed_products
        assert np.array_equal(sp.to_dense(c_sym), sp.to_dense(c_full))
        assert np.array_equal(pyramid_flat(c_sym._tier_norms), pyramid_flat(c_full._tier_norms))
        assert c_sym.symmetric
        cs = sp.convolution_census(x, x, tau)
        assert cs.counts_equal(st_full)


def test_symmetric_flag_propagation(rng):
    d = _sym(rng, 40)
    x = sp.build_from_dense(d, 8)
    assert x.symmetric and sp.identity(40, 8).symmetric
    assert sp.add_scaled(2.0, x, -1.0, sp.identity(40, 8)).symmetric
    a = sp.build_from_dense(rng.standard_normal((40, 40)), 8)
    assert not a.symmetric
    _, st = sp.multiply(a, a, 0.0)
    assert not st.symmetric and st.executed_products == st.leaf_products
    _, st = sp.multiply(x, sp.add_scaled(1.0, x, 0.0, x), 0.0)   # equal but distinct operands
    assert not st.symmetric


def test_symmetric_tie_falls_back_to_full_cull(rng):
    """Block norms of X_ik and X_ki^T are summed in different orders; if tau
    splits a mirror pair the survivor set is not symmetric and the full path
    must run (bitwise the non-symmetric result, symmetric=False)."""
    nb = 4
    for attempt in range(50):
        d = _sym(rng, 32)
        x = sp.build_from_dense(d, nb)
        leaf = x._tier_norms[-1]
        g = leaf.shape[0]
        found = None
        for i in range(g):
            for j in range(i + 1, g):
                for k in range(g):
                    p, q = leaf[i, k] * leaf[k, j], leaf[j, k] * leaf[k, i]
                    if p != q:
                        found = min(p, q)
                        break
                if found:
                    break
            if found:
                break
        if found:
            break
    assert found, "no ulp-asymmetric norm product found"
    c_sym, st = sp.multiply(x, x, found)
    assert not st.symmetric
    sp.set_symmetric_products(False)
    try:
        c_full, st_full = sp.multiply(x, x, found)
    finally:
        sp.set_symmetric_products(True)
    assert st.counts_equal(st_full)
    assert np.array_equal(sp.to_dense(c_sym), sp.to_dense(c_full))
    ox = O.from_dense(d, nb)
    v, c, *_ = O.sweep(ox.tier_norms, ox.tier_norms, found)
    assert st.visited == tuple(v) and st.culled == tuple(c)


# -- full-size properties --------------------------------------------------------

def test_cfg4_x0_square_task_set_and_properties():
    cfg = CONFIGS[4]
    h, _ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x0 = sp.sp2_init(f, sp.gershgorin_bounds(f))
    of = O.from_dense(h, cfg.block_size)
    ox0 = O.sp2_init(of, O.gershgorin_bounds(of))
    assert np.array_equal(pyramid_flat(x0._tier_norms), pyramid_flat(ox0.tier_norms))
    ti, tk, tj = sp.leaf_tasks(x0, x0, cfg.tau)
    v, _, oi, ok, oj = O.sweep(ox0.tier_norms, ox0.tier_norms, cfg.tau)
    g = x0.n_blocks
    assert np.array_equal(np.sort((ti * g + tk) * g + tj), np.sort((oi * g + ok) * g + oj))
    c, st = sp.multiply(x0, x0, cfg.tau)
    assert st.visited == tuple(v)
    assert sp.verify_norms(c)[0]
    # linearity in the scale of one operand (exact: scaling by 2 is exact)
    x2 = sp.add_scaled(2.0, x0, 0.0, x0)
    c2, st2 = sp.multiply(x0, x2, 2 * cfg.tau)
    assert st2.leaf_products == st.leaf_products
    assert np.array_equal(sp.to_dense(c2), 2 * sp.to_dense(c))
    # run-to-run bitwise determinism at full size
    c3, _ = sp.multiply(x0, x0, cfg.tau)
    assert torch.equal(c.blocks_device(), c3.blocks_device())


# -- dense cull (depth <= 8) == tier walk ---------------------------------------

def _walk(fn):
    sp.set_dense_cull(False)
    try:
        return fn()
    finally:
        sp.set_dense_cull(True)


@pytest.mark.parametrize("case", ["sym", "pair", "sparse", "single", "deep", "nan"])
def test_dense_cull_equals_tier_walk_and_reference(rng, case):
    """The dense cull (every leaf triple tested with its ancestor chain) gives
    the tier walk's task list (same order), counters and C, and the
    reference _sweep's counters -- including a NaN block, where a parent's
    NaN norm culls finite children (the reason the chain is tested)."""
    nb = 4
    if case == "sym":
        da = _sym(rng, 61, 0.7)
        db = da
    elif case == "pair":
        da, db = rng.standard_normal((61, 61)), rng.standard_normal((61, 61))
    elif case == "sparse":
        da = rng.standard_normal((64, 64))
        da[np.abs(da) < 1.2] = 0.0
        db = da.T.copy()
    elif case == "single":
        nb, da = 8, rng.standard_normal((7, 7))
        db = da
    elif case == "deep":                       # depth 8: G = 256 with Nb = 1
        nb = 1
        da = _sym(rng, 200, 0.3)
        db = da
    else:
        da = _sym(rng, 48, 0.5)
        da[9, 30] = np.nan
        db = da
    a = sp.build_from_dense(da, nb)
    b = a if db is da else sp.build_from_dense(db, nb)
    oa, ob = O.from_dense(da, nb), O.from_dense(db, nb)
    norms = np.concatenate([t.ravel() for t in a._tier_norms])
    fin = norms[np.isfinite(norms) & (norms > 0)]
    for tau in (0.0, float(np.median(fin) ** 2), float(fin.max() ** 2) * 0.99, 1e300):
        c_d, st_d = sp.multiply(a, b, tau, kernel="exact")
        c_w, st_w = _walk(lambda: sp.multiply(a, b, tau, kernel="exact"))
        assert st_d.counts_equal(st_w)
        v, cu, ti, *_ = O.sweep(oa.tier_norms, ob.tier_norms, tau)
        assert st_d.visited == tuple(v) and st_d.culled == tuple(cu)
        assert st_d.leaf_products == len(ti)
        assert np.array_equal(sp.to_dense(c_d), sp.to_dense(c_w), equal_nan=True)
        t_d = sp.leaf_tasks(a, b, tau)
        t_w = _walk(lambda: sp.leaf_tasks(a, b, tau))
        assert all(np.array_equal(x, y) for x, y in zip(t_d, t_w))
        cs = sp.convolution_census(a, b, tau)
        assert cs.counts_equal(st_d)


# -- determinism (regression: a K4 stage-refill race once corrupted ~1 block
#    in 40 launches at Nb = 32; results must be bitwise run-to-run) -----------

@pytest.mark.parametrize("cfg_index", [3, 4])
def test_products_bitwise_repeatable(cfg_index):
    import torch
    cfg = CONFIGS[cfg_index]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    for _ in range(6):
        x, _ = sp.sp2_step(x, n_occ, cfg.tau)
    ref = None
    for _ in range(40 if cfg_index == 3 else 12):
        c, _ = sp.multiply(x, x, cfg.tau)
        d = c.blocks_device().clone()
        if ref is None:
            ref = d
        else:
            assert torch.equal(d, ref)
