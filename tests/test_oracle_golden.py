"""Pin the CPU oracle to the reference's own outputs (golden fixtures made by
tests/golden/make_golden.py from the reference package).  CPU only."""

import os

import numpy as np
import pytest

from conftest import golden, pyramid_flat
from oracle import spamm_oracle as O
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, hilbert_keys_3d, water_cluster


def test_numpy_einsum_order_self_check():
    O.self_check_numpy()


def test_leaf_norm_recipe_matches_einsum(rng):
    for nb in (1, 2, 4, 8, 32, 64):
        blk = rng.standard_normal((20, nb, nb)) * np.exp(rng.standard_normal((20, 1, 1)) * 6)
        assert np.array_equal(O.leaf_norms2_recipe(blk), np.einsum("tij,tij->t", blk, blk))


def test_pairwise_sum_matches_numpy(rng):
    for n in (1, 5, 8, 13, 100, 128, 129, 750, 3750):
        a = np.abs(rng.standard_normal(n)) * np.exp(rng.standard_normal(n) * 3)
        assert O.pairwise_sum(a) == a.sum()


def test_known_answers():
    g = golden("small_cases")
    c = O.leaf_gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0], [7.0, 8.0]]),
                    np.zeros((2, 2)))
    assert np.array_equal(c, g["hand_example"])
    tree = O.from_dense(np.full((16, 16), 1.0), 4)
    visited, _, _, _, _ = O.sweep(tree.tier_norms, tree.tier_norms, 0.0)
    assert tuple(visited) == tuple(g["dense_census_visited"]) == (1, 8, 64)


def test_small_cases_bitwise():
    g = golden("small_cases")
    for idx in range(int(g["n_small"])):
        nb = int(g[f"s{idx}_nb"])
        a = O.from_dense(g[f"s{idx}_a"], nb)
        b = O.from_dense(g[f"s{idx}_b"], nb)
        assert np.array_equal(pyramid_flat(a.tier_norms), g[f"s{idx}_apyr"])
        for tau in (0.0, 1e-2, 1.0):
            key = f"s{idx}_t{tau:g}"
            c, st, _ = O.multiply(a, b, tau, threads=2)
            assert np.array_equal(O.to_dense(c), g[key + "_c"]), key
            assert st["visited"] == tuple(g[key + "_visited"])
            assert st["culled"] == tuple(g[key + "_culled"])
            assert np.array_equal(pyramid_flat(c.tier_norms), g[key + "_cpyr"])
            assert O.trace(c) == float(g[key + "_trace"])
        s = O.add_scaled(0.3, a, -1.7, b)
        assert np.array_equal(O.to_dense(s), g[f"s{idx}_add"])
        assert np.array_equal(pyramid_flat(s.tier_norms), g[f"s{idx}_addpyr"])


def _task_keys(ti, tk, tj, g):
    return np.sort((ti * g + tk) * g + tj)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_product_configs_bitwise(name):
    gd = golden(name)
    cfg = CONFIGS[1 if name == "cfg1" else 2]
    if name == "cfg1":
        da, db = decay_pair(cfg.n, 0.1, (0, 1))
    else:
        da, _ = water_cluster(cfg.n_mol, seed=0)
        db = da
    a, b = O.from_dense(da, cfg.block_size), O.from_dense(db, cfg.block_size)
    assert np.array_equal(pyramid_flat(a.tier_norms), gd["a_pyramid"])
    assert np.array_equal(pyramid_flat(b.tier_norms), gd["b_pyramid"])
    c, st, (ti, tk, tj) = O.multiply(a, b, cfg.tau, threads=os.cpu_count())
    assert st["visited"] == tuple(gd["visited"]) and st["culled"] == tuple(gd["culled"])
    assert np.array_equal(_task_keys(ti, tk, tj, a.n_blocks), gd["task_keys"])
    near, margin = O.tie_log(a.tier_norms, b.tier_norms, cfg.tau)
    assert sum(near) == int(gd["near_tau"]) and margin == float(gd["tau_margin"])
    assert np.array_equal(c.keys, gd["c_keys"])
    assert np.array_equal(pyramid_flat(c.tier_norms), gd["c_pyramid"])
    assert O.trace(c) == float(gd["c_trace"])
    pos = np.searchsorted(c.keys, gd["c_sample_keys"])
    assert np.array_equal(c.data[pos], gd["c_sample_blocks"])


def test_cfg2_gershgorin_bitwise():
    gb = golden("cfg2_bounds")
    h, n_occ = water_cluster(CONFIGS[2].n_mol, seed=0)
    lo, hi = O.gershgorin_bounds(O.from_dense(h, 32))
    assert (lo, hi) == (float(gb["eps_min"]), float(gb["eps_max"]))
    assert n_occ == int(gb["n_occ"])


def test_cfg3_sp2_bitwise():
    gd = golden("cfg3_sp2")
    cfg = CONFIGS[3]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = O.from_dense(h, cfg.block_size)
    assert np.array_equal(pyramid_flat(f.tier_norms), gd["f_pyramid"])
    res = O.sp2_solve(f, n_occ, cfg.tau, threads=os.cpu_count(), criterion="fro",
                      record_tasks=True)
    assert res.iterations == int(gd["iterations"]) and res.converged
    # every multiply's task set (sha256 of the sorted keys) and tie log
    assert [bytes.fromhex(h) for h in res.task_sha256] == [bytes(d) for d in gd["task_sha256"]]
    assert [n for n, _ in res.tie_logs] == list(gd["near_tau"])
    assert np.array_equal(np.array([m for _, m in res.tie_logs]), gd["tau_margin"])
    assert np.array_equal(np.array(res.branch_margins), gd["branch_margin"])
    assert [b == O.SQUARE for b in res.branches] == list(gd["branches"])
    assert np.array_equal(np.array(res.trace_history), gd["traces"])
    assert np.array_equal(np.array(res.idem_history), gd["idem"])
    assert np.array_equal(pyramid_flat(res.x.tier_norms), gd["p_pyramid"])


def test_inputs_bit_identical_to_golden():
    """The generators are host independent (synth.py): same bytes everywhere."""
    from paper_1403_7458_b200.synth import input_digest
    da, db = decay_pair(1024, 0.1, (0, 1))
    assert input_digest(da, db) == str(golden("cfg1")["input_sha256"])
    h2, _ = water_cluster(CONFIGS[2].n_mol, seed=0)
    assert input_digest(h2, h2) == str(golden("cfg2")["input_sha256"])
    for name, ci in (("cfg3_sp2", 3), ("cfg4_sp2", 4)):
        h, _ = water_cluster(CONFIGS[ci].n_mol, seed=0)
        assert input_digest(h) == str(golden(name)["input_sha256"]), name


def test_hilbert_keys_match_reference_vectors():
    gd = golden("hilbert")
    assert np.array_equal(hilbert_keys_3d(gd["cells"], 10), gd["keys"])
    assert np.array_equal(hilbert_keys_3d(gd["small"], 2), gd["small_keys"])
