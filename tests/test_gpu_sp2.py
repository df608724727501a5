"""SP2 on the GPU vs the reference (sp2.py) and its golden runs.

Contract (BASELINE north_star): identical iteration count and branch
sequence; density matrix within relative Frobenius 1e-12; with the exact leaf
kernel the whole run is bitwise identical to the reference."""

import numpy as np
import pytest

from conftest import golden, pyramid_flat
from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, water_cluster  # noqa: E402

REL_FRO_TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_gershgorin_bitwise_cfg2():
    gb = golden("cfg2_bounds")
    h, _ = water_cluster(CONFIGS[2].n_mol, seed=0)
    b = sp.gershgorin_bounds(sp.build_from_dense(h, 32))
    assert (b.eps_min, b.eps_max) == (float(gb["eps_min"]), float(gb["eps_max"]))


def test_gershgorin_rejects_asymmetric(rng):
    d = rng.standard_normal((20, 20))
    with pytest.raises(ValueError, match="not symmetric"):
        sp.gershgorin_bounds(sp.build_from_dense(d, 4))


def test_sp2_validation():
    f = sp.build_from_dense(np.diag(np.arange(1.0, 9.0)), 4)
    for bad in (0, 8, -1):
        with pytest.raises(ValueError):
            sp.sp2_solve(f, bad, 1e-8)
    with pytest.raises(ValueError):
        sp.sp2_init(f, sp.SpectralBounds(1.0, 1.0))


@pytest.mark.parametrize("nb,kernel", [(16, "exact"), (16, "auto"), (8, "auto"), (4, "exact")])
def test_sp2_trace_criterion_vs_oracle(nb, kernel):
    h, n_occ = water_cluster(12, seed=3)
    p, st = sp.sp2_solve(sp.build_from_dense(h, nb), n_occ, 1e-9, kernel=kernel)
    r = O.sp2_solve(O.from_dense(h, nb), n_occ, 1e-9, threads=4)
    assert st.iteration == r.iterations and st.converged == r.converged
    assert st.branch_history == r.branches
    ref = O.to_dense(r.x)
    if kernel == "exact":
        assert st.trace_history == r.trace_history
        assert np.array_equal(sp.to_dense(p), ref)
    else:
        assert rel(sp.to_dense(p), ref) <= REL_FRO_TOL


def test_sp2_step_branches():
    h, n_occ = water_cluster(8, seed=1)
    x = sp.sp2_init(sp.build_from_dense(h, 8), sp.gershgorin_bounds(sp.build_from_dense(h, 8)))
    ox = O.sp2_init(O.from_dense(h, 8), O.gershgorin_bounds(O.from_dense(h, 8)))
    for _ in range(4):
        x, br = sp.sp2_step(x, n_occ, 1e-10, kernel="exact")
        ox, obr, *_ = O.sp2_step(ox, n_occ, 1e-10)
        assert br == obr
        assert np.array_equal(sp.to_dense(x), O.to_dense(ox))


@pytest.mark.parametrize("name,cfg_index", [("cfg3_sp2", 3), ("cfg4_sp2", 4)])
def test_sp2_baseline_configs(name, cfg_index):
    """BASELINE cfg3 / cfg4: ||X^2-X||_F < 1e-6 with SpAMM tau on every X^2."""
    from paper_1403_7458_b200.synth import input_digest
    gd = golden(name)
    cfg = CONFIGS[cfg_index]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    assert input_digest(h) == str(gd["input_sha256"]), "generator not host independent"
    f = sp.build_from_dense(h, cfg.block_size)
    assert np.array_equal(pyramid_flat(f._tier_norms), gd["f_pyramid"])
    b = sp.gershgorin_bounds(f)
    assert (b.eps_min, b.eps_max) == (float(gd["eps_min"]), float(gd["eps_max"]))
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6)
    assert st.converged and st.iteration == int(gd["iterations"])
    assert [br == sp.SQUARE for br in st.branch_history] == list(gd["branches"])
    assert list(st.leaf_products) == list(gd["leaf_products"])   # task sets: exact counts
    assert np.allclose(st.trace_history, gd["traces"], rtol=1e-12, atol=0)
    leaf = p._tier_norms[-1]
    ref_leaf = gd["p_pyramid"][-leaf.size:].reshape(leaf.shape)
    assert rel(leaf, ref_leaf) <= REL_FRO_TOL
    assert abs(sp.trace(p) - float(gd["p_trace"])) <= 1e-12 * float(gd["p_trace"])
    assert abs(sp.trace(p) - n_occ) < 1e-3
    # exact leaf kernel: the whole SP2 trajectory is bitwise the reference's
    pe, ste = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6, kernel="exact")
    assert ste.iteration == int(gd["iterations"])
    assert np.array_equal(np.array(ste.trace_history), gd["traces"])
    assert np.array_equal(np.array(ste.idempotency_history), gd["idem"])
    assert np.array_equal(pyramid_flat(pe._tier_norms), gd["p_pyramid"])
    assert np.array_equal(pe._block_keys, gd["p_keys"])


@pytest.mark.parametrize("nb", [8, 32, 64])
def test_fused_update_bitwise_equals_add_scaled(rng, nb):
    """K6 fused pass == add_scaled(2,X,-1,X2) and add_scaled(1,X2,-1,X).norm()."""
    from paper_1403_7458_b200.sp2 import _update
    n = 5 * nb + 3
    d = rng.standard_normal((n, n))
    d[np.abs(d) < 1.0] = 0.0
    d[: nb, nb: 2 * nb] = 0.0             # a block present in X only after squaring
    x = sp.build_from_dense(d, nb)
    x2, _ = sp.multiply(x, x, 0.5)
    e, idem = _update(x, x2, True, True)
    ref_e = sp.add_scaled(2.0, x, -1.0, x2)
    assert np.array_equal(sp.to_dense(e), sp.to_dense(ref_e))
    assert np.array_equal(pyramid_flat(e._tier_norms), pyramid_flat(ref_e._tier_norms))
    assert np.array_equal(e._block_keys, ref_e._block_keys)
    assert idem == sp.add_scaled(1.0, x2, -1.0, x).norm()
    oe = O.add_scaled(2.0, O.from_dense(d, nb), -1.0, O.from_dense(sp.to_dense(x2), nb))
    assert np.array_equal(sp.to_dense(e), O.to_dense(oe))
    # X == X2: the expansion cancels to X exactly, the idempotency error is 0
    z, idem0 = _update(x, x, True, True)
    assert idem0 == 0.0 and np.array_equal(sp.to_dense(z), d)


@pytest.mark.parametrize("kernel", ["auto", "exact"])
def test_sp2_step_with_exactly_cancelling_blocks(rng, kernel):
    """X = [[I, M], [M^T, -I]] (+ a small tail) makes (X^2)_01 = M - M = 0
    exactly: the native step's lazily pruned X^2 / 2X - X^2 must match the
    reference's eagerly pruned ones (keys, data, pyramid, traces)."""
    nb = 16
    m = rng.standard_normal((2 * nb, 2 * nb))
    n = 4 * nb
    x = np.zeros((n, n))
    x[: 2 * nb, : 2 * nb] = np.eye(2 * nb)
    x[2 * nb:, 2 * nb:] = -np.eye(2 * nb)
    x[: 2 * nb, 2 * nb:] = m
    x[2 * nb:, : 2 * nb] = m.T
    dx = sp.build_from_dense(x, nb)
    ox = O.from_dense(x, nb)
    for n_occ in (10, -10):           # one SQUARE, one EXPAND step (t_x = 0)
        nxt, br = sp.sp2_step(dx, n_occ, 0.0, kernel=kernel)
        onxt, obr, *_ = O.sp2_step(ox, n_occ, 0.0)
        assert br == obr
        assert np.array_equal(nxt._block_keys, onxt.keys)      # exact cancellation pruned
        assert nxt.stored_leaf_count == len(onxt.keys)
        if kernel == "exact":
            assert np.array_equal(sp.to_dense(nxt), O.to_dense(onxt))
            assert np.array_equal(pyramid_flat(nxt._tier_norms), pyramid_flat(onxt.tier_norms))
        else:
            assert rel(sp.to_dense(nxt), O.to_dense(onxt)) <= REL_FRO_TOL


def test_idempotency_and_energy_error():
    h, n_occ = water_cluster(10, seed=4)
    f = sp.build_from_dense(h, 16)
    p, st = sp.sp2_solve(f, n_occ, 0.0)
    assert st.converged
    assert sp.idempotency_error(p) < 1e-6
    of = O.from_dense(h, 16)
    assert abs(sp.energy_error(f, p, p)) == 0.0
    w, v = np.linalg.eigh(h)
    proj = v[:, :n_occ] @ v[:, :n_occ].T
    assert np.linalg.norm(sp.to_dense(p) - proj) < 1e-6
    assert of.n_native == h.shape[0]


_TF_CODE = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
out = {}
for ci, crit, max_iter in ((3, "fro", 100), (4, "fro", 100), (4, "trace", 100), (4, "fro", 7),
                           (4, "fro", 1), (3, "trace", 5)):
    cfg = CONFIGS[ci]
    h, n = water_cluster(cfg.n_mol, seed=0)
    kw = dict(criterion=crit, max_iter=max_iter)
    if crit == "trace":
        kw["idem_tol"] = 1e-7
    p, st = sp.sp2_solve(sp.build_from_dense(h, cfg.block_size), n, cfg.tau, **kw)
    d = sp.to_dense(p)
    key = f"{ci}-{crit}-{max_iter}"
    np.save(sys.argv[1] + key + ".npy", d)
    out[key] = dict(it=st.iteration, conv=st.converged, br=[str(b) for b in st.branch_history],
                    tr=[float(v).hex() for v in st.trace_history],
                    idem=[float(v).hex() for v in (st.idempotency_history or [])],
                    leaf=[int(v) for v in st.leaf_products],
                    bm=[float(v).hex() for v in st.branch_margins],
                    near=[int(v) for v in st.near_tau_history])
json.dump(out, open(sys.argv[1] + "meta.json", "w"))
"""


def test_trace_first_loop_bitwise_equals_previous_loop(tmp_path):
    """The trace-first SP2 loop (branch from tr X^2 before any norm pass; the
    residual read one host sync later, a converged step's next product
    dropped) gives bitwise the same P, iteration count, branches, traces,
    residuals and per-multiply survivor counts as the loop that finalises X^2
    before the branch (SPAMM_SP2_TF=0) -- converged runs with both criteria
    and runs cut by max_iter."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        base = str(tmp_path / f"tf{flag}_")
        env = dict(os.environ, SPAMM_SP2_TF=flag)
        subprocess.run([sys.executable, "-c", _TF_CODE % root, base], env=env, check=True,
                       timeout=900)
        res[flag] = (base, json.load(open(base + "meta.json")))
    (b0, m0), (b1, m1) = res["0"], res["1"]
    assert m0 == m1
    for key in m0:
        assert np.array_equal(np.load(b0 + key + ".npy"), np.load(b1 + key + ".npy")), key
