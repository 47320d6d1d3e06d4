"""Helpers shared by the parity tests (label matching, oracle stepping)."""
import numpy as np


def matched_agreement(a: np.ndarray, b: np.ndarray):
    """Fraction of points whose labels agree after an optimal one-to-one cluster matching
    (contingency table + Hungarian assignment), and the matching (a-id -> b-id)."""
    from scipy.optimize import linear_sum_assignment
    ka, kb = int(a.max()) + 1, int(b.max()) + 1
    cont = np.bincount(a.astype(np.int64) * kb + b, minlength=ka * kb).reshape(ka, kb)
    r, c = linear_sum_assignment(-cont)
    return cont[r, c].sum() / len(a), dict(zip(r.tolist(), c.tolist()))


def oracle_states(X, h, steps, mode=1):
    """The oracle's build state followed by `steps` iterate_once states."""
    from oracle import oracle as O
    keys, cnt, cen, _ = O.build_grid(X, h, mode)
    states = [(keys, cnt, cen)]
    for _ in range(steps):
        r = O.iterate_once(keys, cnt, cen, h)
        keys, cnt, cen = r["keys"], r["counts"], r["centroids"]
        states.append((keys, cnt, cen))
        if r["converged"] or not r["changed"]:
            break
    return states
