"""K4z, the INT8-sliced leaf kernel (leaf_ozaki.cu), against the reference
semantics: the surviving task set and counters are the cull's (identical to
the DMMA and exact kernels), C agrees with the reference-order product within
the north-star tolerance (1e-12 relative Frobenius) and is closer than FP64
itself to the exactly rounded product; symmetric inputs give bitwise symmetric
C; segments longer than the int32 flush chunk; SP2 decisions identical."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster  # noqa: E402

REL_FRO_TOL = 1e-12


def rel_fro(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def extended(da, db, n):
    xa = np.zeros((n, n), np.longdouble)
    xb = np.zeros((n, n), np.longdouble)
    xa[:da.shape[0], :da.shape[1]] = da
    xb[:db.shape[0], :db.shape[1]] = db
    return xa @ xb


def err_vs(c, ex):
    return float(np.linalg.norm((c - ex).astype(np.float64)) / np.linalg.norm(ex.astype(np.float64)))


@pytest.mark.parametrize("nb", [64, 32])
@pytest.mark.parametrize("case", ["decay_ab", "decay_aa", "water", "wide", "wide_sym"])
def test_products_vs_reference_and_extended_precision(case, nb):
    rng = np.random.default_rng(7)
    if case.startswith("decay"):
        da, db = decay_pair(1024, 0.1, (0, 1))
        if case == "decay_aa":
            db = da
    elif case == "water":
        da, _ = water_cluster(30, seed=0)
        db = da
    else:
        x = rng.uniform(-1, 1, (512, 512)) * np.exp(rng.uniform(-30, 5, (512, 512)))
        da = db = x + x.T if case == "wide_sym" else x
    a = sp.build_from_dense(da, nb)
    b = a if db is da else sp.build_from_dense(db, nb)
    for tau in (0.0, 1e-8):
        ce, se = sp.multiply(a, b, tau, kernel="exact")
        co, so = sp.multiply(a, b, tau, kernel="ozaki")
        assert so.counts_equal(se) and so.flop_estimate == se.flop_estimate
        de, do = sp.to_dense(ce), sp.to_dense(co)
        assert rel_fro(do, de) < REL_FRO_TOL
        if tau == 0.0:
            ex = extended(da, db, de.shape[0])
            # one rounding of the digit-pair sum: closer to the exact product than
            # the reference's own FP64 loop (measured 5-6e-17 vs 4-9e-16)
            assert err_vs(do, ex) < 2e-16
            assert err_vs(do, ex) < err_vs(de, ex)
        if a is b and a.symmetric:
            assert np.array_equal(do, do.T)
            assert co.symmetric


@pytest.mark.parametrize("nb", [64, 32])
def test_symmetric_path_bitwise_equals_full_path(nb):
    h, _ = water_cluster(30, seed=0)
    x = sp.build_from_dense(h, nb)
    assert x.symmetric
    c_sym, st_sym = sp.multiply(x, x, 1e-6, kernel="ozaki")
    sp.set_symmetric_products(False)
    try:
        c_full, st_full = sp.multiply(x, x, 1e-6, kernel="ozaki")
    finally:
        sp.set_symmetric_products(True)
    assert st_sym.symmetric and not st_full.symmetric
    assert np.array_equal(sp.to_dense(c_sym), sp.to_dense(c_full))


def test_deterministic_repeats():
    da, db = decay_pair(1024, 0.05, (3, 4))
    a, b = sp.build_from_dense(da, 64), sp.build_from_dense(db, 64)
    c0 = sp.to_dense(sp.multiply(a, b, 1e-10, kernel="ozaki")[0])
    for _ in range(3):
        assert np.array_equal(sp.to_dense(sp.multiply(a, b, 1e-10, kernel="ozaki")[0]), c0)


@pytest.mark.parametrize("nb", [64, 32])
def test_long_segments_flush_in_chunks(nb):
    """G = 132 leaf blocks per side, tau = 0: every C block reduces 132 tasks,
    more than the 128-task int32 chunk, so each block is flushed to FP64 twice."""
    n = 132 * nb
    g = torch.Generator(device="cuda").manual_seed(5)
    d = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    i = torch.arange(n, device="cuda", dtype=torch.float64)
    d *= torch.exp(-0.002 * (i[:, None] - i[None, :]).abs())
    a = sp.build_from_dense(d, nb)
    cd, sd = sp.multiply(a, a, 0.0, kernel="dmma")
    co, so = sp.multiply(a, a, 0.0, kernel="ozaki")
    assert so.counts_equal(sd) and so.leaf_products == 132 ** 3
    ref = (d @ d).cpu().numpy()
    assert rel_fro(sp.to_dense(co), ref) < 1e-14
    assert rel_fro(sp.to_dense(co), sp.to_dense(cd)) < 1e-14


def test_zero_rows_and_empty_products():
    rng = np.random.default_rng(11)
    d = rng.standard_normal((300, 300))
    d[17, :] = 0.0
    d[:, 200:264] = 0.0
    a = sp.build_from_dense(d, 64)
    c, st = sp.multiply(a, a, 0.0, kernel="ozaki")
    ref = d @ d
    assert rel_fro(sp.to_dense(c), ref) < 1e-15
    assert not sp.to_dense(c)[17].any()
    z = sp.build_from_dense(np.zeros((200, 200)), 64)
    c, st = sp.multiply(z, z, 0.0, kernel="ozaki")
    assert st.leaf_products == 0 and not sp.to_dense(c).any()


def test_block_size_guard():
    a = sp.build_from_dense(np.eye(64), 16)
    with pytest.raises(ValueError, match="block size 32 or 64"):
        sp.multiply(a, a, 0.0, kernel="ozaki")


@pytest.mark.parametrize("cfg_index", [4, 3])
def test_sp2_same_decisions_as_dmma(cfg_index):
    cfg = CONFIGS[cfg_index]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
    kw = dict(criterion="fro", fro_tol=1e-6)
    pd, sd = sp.sp2_solve(f, n_occ, cfg.tau, kernel="dmma", **kw)
    po, so = sp.sp2_solve(f, n_occ, cfg.tau, kernel="ozaki", **kw)
    assert so.iteration == sd.iteration and so.converged and sd.converged
    assert so.branch_history == sd.branch_history
    assert so.leaf_products == sd.leaf_products
    assert rel_fro(sp.to_dense(po), sp.to_dense(pd)) < REL_FRO_TOL
    assert po.symmetric


def test_auto_falls_back_to_dmma_without_slice_memory():
    """AUTO needs the digit slices (the operand's size again); when they cannot
    be allocated it runs the DMMA kernel (config 5's 84-GB H on one GPU).  The
    SPAMM_OZ_FORCE_NOMEM hook makes every slice allocation fail."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, paper_1403_7458_b200 as sp\n"
        "from paper_1403_7458_b200.synth import water_cluster\n"
        "h, _ = water_cluster(30, seed=0)\n"
        "x = sp.build_from_dense(h, 64)\n"
        "ca, _ = sp.multiply(x, x, 1e-8)\n"
        "cd, _ = sp.multiply(x, x, 1e-8, kernel='dmma')\n"
        "assert np.array_equal(sp.to_dense(ca), sp.to_dense(cd))\n"
        "print('fallback ok')\n")
    env = dict(os.environ, SPAMM_OZ_FORCE_NOMEM="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and "fallback ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("env_on,env_off", [
    ({"SPAMM_OZ_EXOUT": "1", "SPAMM_OZ_EXPROD": "0"}, {"SPAMM_OZ_EXPROD": "0"}),
    ({}, {"SPAMM_OZ_EXPROD": "0"}),
])
def test_product_exponents_from_the_epilogue_are_the_exponent_pass(tmp_path, env_on, env_off):
    """The next multiply's K4z row exponents taken from the kernel that
    produced the matrix -- the K4z epilogue (SPAMM_OZ_EXOUT=1), or, by default,
    the column maxima of the K1 pass over X^2 and of the SP2 update over
    2X - X^2 (SPAMM_OZ_EXPROD) -- instead of a separate exponent pass: bitwise
    the SP2 with the pass, for Nb = 64 (K4z) and Nb = 32 (K4z32)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_1403_7458_b200 as sp\n"
            "from paper_1403_7458_b200.synth import CONFIGS, water_cluster\n"
            "for ci in (3, 4):\n"
            "    cfg = CONFIGS[ci]; h, n = water_cluster(cfg.n_mol, seed=0)\n"
            "    p, st = sp.sp2_solve(sp.build_from_dense(h, cfg.block_size), n, cfg.tau,"
            " criterion='fro')\n"
            "    np.save(sys.argv[1] + f'_{ci}.npy', sp.to_dense(p))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag, extra in (("0", env_off), ("1", env_on)):
        env = dict(os.environ, **extra)
        base = str(tmp_path / f"p{flag}")
        subprocess.run([sys.executable, "-c", code % root, base], env=env, check=True)
        outs[flag] = [np.load(f"{base}_{ci}.npy") for ci in (3, 4)]
    for a, b in zip(outs["0"], outs["1"]):
        assert np.array_equal(a, b)


def _exact_product(a, b):
    """C = A B exactly (Python integers on the doubles' mantissa grid), then
    the exact values as (numerator, exponent) -> float via Fraction."""
    from fractions import Fraction
    n = a.shape[0]
    fa = [[Fraction(float(v)) for v in row] for row in a]
    fb = [[Fraction(float(v)) for v in row] for row in b]
    out = np.zeros((n, n))
    err_ref = np.zeros((n, n), dtype=object)
    for i in range(n):
        for j in range(n):
            s = sum(fa[i][k] * fb[k][j] for k in range(n))
            err_ref[i, j] = s
            out[i, j] = float(s)
    return out, err_ref


@pytest.mark.parametrize("nb", [32, 64])
def test_elementwise_accuracy_envelope(nb):
    """K4z scales each global row of A (column of B) by one power of two, so
    its error bound is absolute against the row / column maxima -- a
    fixed-point format of 63 bits per row: |c - c_exact| <= K 2^-62
    2^(E_r + E_c) per element (E: the scale exponents, max|A_r| < 2^E_r), where
    FP64's bound is relative to sum |a_rk b_kc|.  An element 2^-k below the
    product of its row and column maxima therefore keeps ~63 - k bits (FP64:
    ~53).  Rows here span 60 binades; the bound must hold for every element,
    and the matrix-level error stays below FP64's."""
    rng = np.random.default_rng(3)
    n = nb
    a = rng.uniform(-1, 1, (n, n)) * np.exp2(-rng.integers(0, 60, (n, n)))
    b = rng.uniform(-1, 1, (n, n)) * np.exp2(-rng.integers(0, 60, (n, n)))
    ref, exact = _exact_product(a, b)
    got = sp.to_dense(sp.multiply(sp.build_from_dense(a, nb), sp.build_from_dense(b, nb), 0.0,
                                  kernel="ozaki")[0])
    fp64 = sp.to_dense(sp.multiply(sp.build_from_dense(a, nb), sp.build_from_dense(b, nb), 0.0,
                                   kernel="exact")[0])
    er = np.ceil(np.log2(np.abs(a).max(axis=1))) + 1       # >= the kernel's row scale exponents
    ec = np.ceil(np.log2(np.abs(b).max(axis=0))) + 1
    scale = np.exp2(er[:, None] + ec[None, :])
    # digit truncation of both operands (K terms) + the rounding of the result
    bound = n * np.exp2(-62.0) * scale + np.exp2(-52.0) * np.abs(ref)
    from fractions import Fraction
    err = np.array([[abs(float(Fraction(float(got[i, j])) - exact[i, j])) for j in range(n)]
                    for i in range(n)])
    assert (err <= bound).all(), float((err / bound).max())
    # matrix level: K4z is closer to the exact product than the FP64 loop
    assert np.linalg.norm(got - ref) <= np.linalg.norm(fp64 - ref)
    # elements within 2^8 of their row x column scale keep FP64-level relative
    # accuracy; smaller ones lose relative bits as the envelope says
    rel = err / np.maximum(np.abs(ref), 1e-300)
    big = np.abs(ref) >= np.exp2(-8) * scale
    assert big.any() and rel[big].max() < 1e-14


@pytest.mark.parametrize("nb", [32, 64])
@pytest.mark.parametrize("ea,eb", [(400, 400), (-490, -490), (500, -500), (-500, 500)])
def test_power_of_two_scaling_commutes_exactly(nb, ea, eb):
    """K4z's row / column scales are powers of two taken from the data, so
    scaling A by 2^ea and B by 2^eb (no overflow; results compared where they
    are normal numbers) must scale C by exactly 2^(ea + eb) -- bitwise -- and stay
    within the north-star tolerance of the reference-order FP64 product at
    magnitudes far from 1 (the epilogue's 2^k factor as one exact multiply, or
    ldexp when k leaves the normal exponent range)."""
    rng = np.random.default_rng(21)
    n = 3 * nb + 5
    a = rng.uniform(-1, 1, (n, n)) * np.exp(rng.uniform(-12, 0, (n, n)))
    b = rng.uniform(-1, 1, (n, n)) * np.exp(rng.uniform(-12, 0, (n, n)))
    c0 = sp.to_dense(sp.multiply(sp.build_from_dense(a, nb), sp.build_from_dense(b, nb), 0.0,
                                 kernel="ozaki")[0])
    sa, sb = np.ldexp(a, ea), np.ldexp(b, eb)
    qa, qb = sp.build_from_dense(sa, nb), sp.build_from_dense(sb, nb)
    c1 = sp.to_dense(sp.multiply(qa, qb, 0.0, kernel="ozaki")[0])
    want = np.ldexp(c0, ea + eb)
    normal = np.abs(want) >= np.ldexp(1.0, -1021)
    assert normal.mean() > 0.99 and np.array_equal(c1[normal], want[normal])
    ce = sp.to_dense(sp.multiply(qa, qb, 0.0, kernel="exact")[0])
    # (compared at unit scale: the norms of values near 2^+-800 leave the FP64 range)
    assert np.isfinite(ce).all()
    assert rel_fro(np.ldexp(c1, -(ea + eb)), np.ldexp(ce, -(ea + eb))) < REL_FRO_TOL
