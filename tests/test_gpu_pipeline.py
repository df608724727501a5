"""pipeline.sp2_solve_many: transfers overlapped with compute, results bitwise
the one-at-a-time path (build_from_dense -> sp2_solve -> to_dense)."""

import numpy as np
import pytest
import torch

import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.pipeline import sp2_solve_many
from paper_1403_7458_b200.synth import water_cluster


def _problems(sizes_seeds):
    return [water_cluster(n_mol, seed) for n_mol, seed in sizes_seeds]


@pytest.mark.gpu
@pytest.mark.parametrize("count", [1, 2, 5])
def test_solve_many_bitwise_single_path(count):
    probs = _problems([(12, s) for s in range(count)])
    hs = [h for h, _ in probs]
    occ = [o for _, o in probs]
    ps, states = sp2_solve_many(hs, occ, 1e-7, block_size=16, criterion="fro")
    assert len(ps) == len(states) == count
    for (h, o), p, st in zip(probs, ps, states):
        f = sp.build_from_dense(h, 16)
        p_ref, st_ref = sp.sp2_solve(f, o, 1e-7, criterion="fro")
        assert st.iteration == st_ref.iteration and st.branch_history == st_ref.branch_history
        assert np.array_equal(p.numpy(), sp.to_dense(p_ref))


@pytest.mark.gpu
def test_solve_many_custom_solver_and_out():
    probs = _problems([(10, 3), (10, 4), (10, 5)])
    hs = [torch.from_numpy(h) for h, _ in probs]          # host tensors, not pinned
    out = [torch.empty_like(h).pin_memory() for h in hs]
    calls = []

    def solver(f, occ):
        calls.append(occ)
        return sp.sp2_solve(f, occ, 0.0)

    hooks = []
    ps, _ = sp2_solve_many(hs, [o for _, o in probs], 0.0, 16, solver=solver, out=out,
                           before_each=hooks.append)
    assert calls == [o for _, o in probs] and hooks == [0, 1, 2]
    assert all(p is o for p, o in zip(ps, out))
    for (h, o), p in zip(probs, ps):
        p_ref, _ = sp.sp2_solve(sp.build_from_dense(h, 16), o, 0.0)
        assert np.array_equal(p.numpy(), sp.to_dense(p_ref))


def test_solve_many_argument_errors():
    h = np.eye(8)
    assert sp2_solve_many([], 2, 0.0) == ([], [])
    with pytest.raises(ValueError, match="must be 8x8"):
        sp2_solve_many([h, np.eye(9)], 2, 0.0)
    with pytest.raises(ValueError, match="one per Hamiltonian"):
        sp2_solve_many([h, h], [2, 3, 4], 0.0)
    with pytest.raises(ValueError, match="out: one tensor"):
        sp2_solve_many([h, h], 2, 0.0, out=[None])
