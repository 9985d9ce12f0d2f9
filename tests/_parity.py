"""Shared parity checks of the test suite (no method arithmetic): the residual-history rule
of SURVEY §8(c)-15 ("history agrees to 1e-6 relative while > 1e-10")."""
import numpy as np


def cycle_layout(iters, restart, hist_len):
    """Positions of the Arnoldi estimates / cycle-end true residuals in a history of a
    GMRES(restart) run with `iters` Arnoldi steps that ended by convergence or maxit:
    every cycle but the last has `restart` estimates followed by one true residual."""
    kinds = []
    left = iters
    while left > 0 and len(kinds) < hist_len:
        k = min(restart, left)
        kinds += ["est"] * k + ["true"]
        left -= k
    return kinds[:hist_len]


def assert_hist_agree(h, it, ref, it_ref, restart, rtol=1e-6, floor=1e-10):
    """Entry-by-entry comparison of two residual histories over their common aligned part.
    With equal iteration counts the layouts are identical and every entry is compared; with
    counts differing by one, the shorter run's LAST cycle (whose length differs) is left out
    and the rest compared.  Entries are compared while both exceed `floor`."""
    h = np.asarray(h, float)
    ref = np.asarray(ref, float)
    la = cycle_layout(it, restart, len(h))
    lb = cycle_layout(it_ref, restart, len(ref))
    k = min(len(h), len(ref))
    if it != it_ref:
        # aligned prefix: whole cycles shared by both layouts
        last_end = 0
        for i in range(k):
            if la[i] == "true" and lb[i] == "true":
                last_end = i + 1
            if la[i] != lb[i]:
                break
        k = last_end
    assert k > 0 or min(it, it_ref) == 0, "no comparable history entries"
    assert la[:k] == lb[:k], "history layouts differ"
    for i in range(k):
        a, c = h[i], ref[i]
        if a > floor and c > floor:
            assert abs(a - c) <= rtol * c, (i, la[i], a, c, abs(a - c) / c)
    return k
