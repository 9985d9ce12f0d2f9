"""CPU checks of the parity rules themselves (tests/_parity.py): the residual-history rule
must FAIL on a deliberately perturbed history (the old check could not fail)."""
import numpy as np
import pytest

import gen
import oracle
from _parity import assert_hist_agree, cycle_layout


def _run(restart, orth=0, tol=1e-8):
    p = gen.make_config("C2", nx=14, ny=12, nz=4)
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=60, orth=orth)
    return M.solve(p["rhs"], tol=tol, restart=restart)


def test_cycle_layout():
    assert cycle_layout(5, 30, 6) == ["est"] * 5 + ["true"]
    assert cycle_layout(7, 3, 10) == ["est"] * 3 + ["true"] + ["est"] * 3 + ["true"] + ["est", "true"]


@pytest.mark.parametrize("restart", [30, 5])
def test_history_rule_accepts_same_run_and_rejects_perturbation(restart):
    o = _run(restart)
    assert len(o["hist"]) == o["iters"] + -(-o["iters"] // restart)      # estimates + cycle ends
    k = assert_hist_agree(o["hist"], o["iters"], o["hist"], o["iters"], restart)
    assert k == len(o["hist"])
    for pos in (0, len(o["hist"]) // 2, len(o["hist"]) - 2):
        h = o["hist"].copy()
        h[pos] *= 1 + 2e-6
        with pytest.raises(AssertionError):
            assert_hist_agree(h, o["iters"], o["hist"], o["iters"], restart)


def test_history_rule_cgs2_vs_dcgs2_vs_mgs():
    """The oracle's three orthogonalisations build the same basis in exact arithmetic:
    their histories satisfy the rule against each other (restarted runs included)."""
    for restart in (30, 5):
        ref = _run(restart, orth=0)
        for orth in (1, 2):
            o = _run(restart, orth=orth)
            assert abs(o["iters"] - ref["iters"]) <= 1
            assert_hist_agree(o["hist"], o["iters"], ref["hist"], ref["iters"], restart)


def test_history_rule_iteration_mismatch_compares_shared_cycles():
    ref = _run(5)
    it = ref["iters"]
    # a run one iteration shorter: drop the last estimate of the final cycle
    last_cycle = it % 5 or 5
    h = list(ref["hist"][:-(last_cycle + 1)]) + list(ref["hist"][-(last_cycle + 1):-2]) + [ref["hist"][-1]]
    k = assert_hist_agree(np.array(h), it - 1, ref["hist"], it, 5)
    assert k == len(ref["hist"]) - (last_cycle + 1)
    h2 = np.array(h)
    h2[1] *= 1.01
    with pytest.raises(AssertionError):
        assert_hist_agree(h2, it - 1, ref["hist"], it, 5)
