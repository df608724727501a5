"""Generate golden fixtures by running the REFERENCE implementation.

Run once in the build container (the reference is importable from
/root/reference/pkg/src there; it does not exist on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are re-created from paper_1403_7458_b200.synth (seeded numpy), so the
fixtures only store reference OUTPUTS (norm pyramids, counters, sorted task
keys, per-block C norms, traces, SP2 histories) plus full operands for the
small cases.  Everything is written to tests/golden/*.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import hashlib  # noqa: E402

import spamm  # noqa: E402  (the reference)

from oracle import spamm_oracle as O  # noqa: E402  (tie_log helper only)
from spamm import sp2 as ref_sp2  # noqa: E402

from paper_1403_7458_b200.synth import (CONFIGS, decay_pair, input_digest,  # noqa: E402
                                        water_cluster)


def pyramid_flat(tree):
    return np.concatenate([t.reshape(-1) for t in tree._tier_norms])


def task_keys(a, b, tau):
    _, _, i, k, j = spamm.kernel._sweep(a._tier_norms, b._tier_norms, tau)
    g = a.n_blocks
    return np.sort((i * g + k) * g + j).astype(np.int64)


def task_digest(a, b, tau):
    """sha256 of the reference's sorted leaf task keys ((i G + k) G + j, int64
    little-endian) -- the exact task set, kernel.py:96-122."""
    return np.frombuffer(hashlib.sha256(task_keys(a, b, tau).astype("<i8").tobytes()).digest(),
                         dtype=np.uint8)


def tie_log(a, b, tau):
    """Near-tau products (64 ulps) per tier and the smallest relative margin of
    a tested product, on the REFERENCE's pyramids (oracle.tie_log restates the
    candidate expansion of kernel.py:96-122)."""
    near, margin = O.tie_log(a._tier_norms, b._tier_norms, tau, 64)
    return int(sum(near)), margin


def product_case(name, da, db, nb, tau, sample_blocks=8):
    a = spamm.build_from_dense(da, nb)
    b = spamm.build_from_dense(db, nb)
    c, st = spamm.multiply(a, b, tau, mode="tasked", workers=os.cpu_count())
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(len(c._block_keys), size=min(sample_blocks, len(c._block_keys)),
                              replace=False))
    out = dict(
        nb=nb, tau=tau, n=da.shape[0],
        a_pyramid=pyramid_flat(a), b_pyramid=pyramid_flat(b),
        a_stored=a.stored_leaf_count, b_stored=b.stored_leaf_count,
        visited=np.array(st.visited), culled=np.array(st.culled),
        leaf_products=st.leaf_products, flop_estimate=st.flop_estimate,
        task_keys=task_keys(a, b, tau),
        near_tau=tie_log(a, b, tau)[0], tau_margin=tie_log(a, b, tau)[1],
        c_keys=c._block_keys, c_pyramid=pyramid_flat(c), c_trace=spamm.trace(c),
        c_sample_keys=c._block_keys[pick], c_sample_blocks=c._block_data[pick],
        a_trace=spamm.trace(a), input_sha256=input_digest(da, db),
    )
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "leaf_products", st.leaf_products, "visited", st.visited, flush=True)
    return a


def sp2_fro_case(name, h, nb, n_occ, tau, fro_tol=1e-6, max_iter=100):
    """BASELINE's ||X^2-X||_F < tol loop built from reference primitives (sp2.py)."""
    f = spamm.build_from_dense(h, nb)
    bounds = spamm.gershgorin_bounds(f)
    x = spamm.sp2_init(f, bounds)
    traces, branches, idem, leaf = [spamm.trace(x)], [], [], []
    digests, near, margin, bmargin = [], [], [], []
    it = 0
    converged = False
    for _ in range(max_iter):
        # sp2._step (sp2.py:92-101), spelled out so X^2 is also available for
        # the idempotency test.
        x_sq, st = spamm.multiply(x, x, tau, mode="tasked", workers=os.cpu_count())
        leaf.append(st.leaf_products)
        digests.append(task_digest(x, x, tau))
        nt, mg = tie_log(x, x, tau)
        near.append(nt)
        margin.append(mg)
        t_x, t_sq = spamm.trace(x), spamm.trace(x_sq)
        t_ex = 2.0 * t_x - t_sq
        bmargin.append(abs(t_ex - n_occ) - abs(t_sq - n_occ))
        branch = ref_sp2.SQUARE if abs(t_sq - n_occ) <= abs(t_ex - n_occ) else ref_sp2.EXPAND
        e = spamm.add_scaled(1.0, x_sq, -1.0, x).norm()
        idem.append(e)
        if e < fro_tol:
            converged = True
            break
        x = x_sq if branch == ref_sp2.SQUARE else spamm.add_scaled(2.0, x, -1.0, x_sq)
        it += 1
        traces.append(spamm.trace(x))
        branches.append(branch)
        print(name, it, branch, e, flush=True)
    out = dict(nb=nb, tau=tau, n_occ=n_occ, eps_min=bounds.eps_min, eps_max=bounds.eps_max,
               f_pyramid=pyramid_flat(f), x0_pyramid=None, iterations=it, converged=converged,
               traces=np.array(traces), branches=np.array([b == "SQUARE" for b in branches]),
               idem=np.array(idem), leaf_products=np.array(leaf),
               task_sha256=np.array(digests), near_tau=np.array(near), tau_margin=np.array(margin),
               branch_margin=np.array(bmargin),
               p_pyramid=pyramid_flat(x), p_trace=spamm.trace(x), p_keys=x._block_keys,
               input_sha256=input_digest(h))
    out.pop("x0_pyramid")
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def small_cases():
    rng = np.random.default_rng(12345)
    cases = {}
    for idx, (n, nb, thr) in enumerate([(48, 4, 0.0), (37, 4, 0.8), (100, 8, 0.5), (64, 16, 0.0),
                                        (7, 2, 0.0), (1, 1, 0.0), (96, 32, 1.2), (130, 64, 1.5)]):
        da = rng.standard_normal((n, n))
        db = rng.standard_normal((n, n))
        da[np.abs(da) < thr] = 0.0
        db[np.abs(db) < thr] = 0.0
        a = spamm.build_from_dense(da, nb)
        b = spamm.build_from_dense(db, nb)
        for tau in (0.0, 1e-2, 1.0):
            c, st = spamm.multiply(a, b, tau)
            key = f"s{idx}_t{tau:g}"
            cases[key + "_c"] = spamm.to_dense(c)
            cases[key + "_visited"] = np.array(st.visited)
            cases[key + "_culled"] = np.array(st.culled)
            cases[key + "_cpyr"] = pyramid_flat(c)
            cases[key + "_trace"] = np.array(spamm.trace(c))
        cases[f"s{idx}_a"] = da
        cases[f"s{idx}_b"] = db
        cases[f"s{idx}_nb"] = np.array(nb)
        cases[f"s{idx}_apyr"] = pyramid_flat(a)
        s = spamm.add_scaled(0.3, a, -1.7, b)
        cases[f"s{idx}_add"] = spamm.to_dense(s)
        cases[f"s{idx}_addpyr"] = pyramid_flat(s)
    cases["n_small"] = np.array(8)
    # known answers from the reference's own tests (test_kernel.py:18-24, 115-119)
    c = np.zeros((2, 2))
    spamm.leaf_gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0], [7.0, 8.0]]), c)
    cases["hand_example"] = c
    tree = spamm.build_from_dense(np.full((16, 16), 1.0), block_size=4)
    cases["dense_census_visited"] = np.array(spamm.convolution_census(tree, tree, 0.0).visited)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **cases)
    print("small cases", len(cases))


def hilbert_vectors():
    rng = np.random.default_rng(5)
    cells = rng.integers(0, 1 << 10, size=(200, 3))
    keys = np.array([spamm.hilbert_index(c, 10) for c in cells], dtype=np.int64)
    small = np.array([[i, j, k] for i in range(4) for j in range(4) for k in range(4)])
    skeys = np.array([spamm.hilbert_index(c, 2) for c in small], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "hilbert.npz"), cells=cells, keys=keys, small=small,
                        small_keys=skeys)


def main():
    which = sys.argv[1:] or ["small", "hilbert", "cfg1", "cfg2", "cfg3", "cfg4"]
    if "small" in which:
        small_cases()
    if "hilbert" in which:
        hilbert_vectors()
    if "cfg1" in which:
        cfg = CONFIGS[1]
        da, db = decay_pair(cfg.n, 0.1, (0, 1))
        product_case("cfg1", da, db, cfg.block_size, cfg.tau)
    if "cfg2" in which:
        cfg = CONFIGS[2]
        h, n_occ = water_cluster(cfg.n_mol, seed=0)
        product_case("cfg2", h, h, cfg.block_size, cfg.tau)
        f = spamm.build_from_dense(h, cfg.block_size)
        b = spamm.gershgorin_bounds(f)
        np.savez_compressed(os.path.join(HERE, "cfg2_bounds.npz"), eps_min=b.eps_min,
                            eps_max=b.eps_max, n_occ=n_occ)
    if "cfg3" in which:
        cfg = CONFIGS[3]
        h, n_occ = water_cluster(cfg.n_mol, seed=0)
        sp2_fro_case("cfg3_sp2", h, cfg.block_size, n_occ, cfg.tau)
    if "cfg4" in which:
        cfg = CONFIGS[4]
        h, n_occ = water_cluster(cfg.n_mol, seed=0)
        sp2_fro_case("cfg4_sp2", h, cfg.block_size, n_occ, cfg.tau)


if __name__ == "__main__":
    main()
