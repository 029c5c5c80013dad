"""Shared parity helpers for the GPU tests (comparisons against the oracle /
golden fixtures). Tolerances are the north-star contract: O, dQ, dK, dV
within max-abs 2e-2 and rel-L2 1e-2 of the reference on the same inputs;
routing bit-exact except documented score ties within 1e-6."""

import numpy as np

MAX_ABS = 2e-2
REL_L2 = 1e-2
TIE_TOL = 1e-6


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def assert_close(got, ref, what, max_abs=MAX_ABS, rel=REL_L2):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.all(np.isfinite(got)), f"{what}: non-finite values"
    err = float(np.abs(got - ref).max()) if got.size else 0.0
    r = rel_l2(got, ref) if got.size else 0.0
    assert err <= max_abs and r <= rel, f"{what}: max-abs {err:.3e} (tol {max_abs}), rel-L2 {r:.3e} (tol {rel})"
    return err, r


def unexcused_routing_rows(Q, cents, got, ref, B, k, tol=TIE_TOL):
    """Rows whose selected sets differ and the difference is NOT a near-tie.

    A row is excused when every block in the symmetric difference of the two
    sets scores (f64, unscaled q . centroid) within `tol` of the k-th best
    past-block score, i.e. the two selections are both valid top-k sets up to
    the score resolution.
    """
    Q = np.asarray(Q, dtype=np.float64)
    cents = np.asarray(cents, dtype=np.float64)
    got = np.asarray(got)
    ref = np.asarray(ref)
    bad = []
    diff_rows = np.nonzero(np.any(got != ref, axis=1))[0]
    for i in diff_rows:
        own = i // B
        sg = set(int(x) for x in got[i] if x >= 0)
        sr = set(int(x) for x in ref[i] if x >= 0)
        if own not in sg:
            bad.append(int(i))
            continue
        if own <= k or len(sg) != len(sr):
            bad.append(int(i))
            continue
        scores = Q[i] @ cents[:own].T
        kth = np.sort(scores)[::-1][k - 1]
        if any(abs(scores[j] - kth) > tol for j in sg ^ sr):
            bad.append(int(i))
    return bad, len(diff_rows)


def bf16_round(x):
    import torch
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()
