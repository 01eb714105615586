"""Index-set comparison for the floating-point scorers (SnapKV), bounded by the measured score error.

If every device score is within eps (absolute) of the oracle's, an index can be in the device's top-k and not in the
oracle's (or the reverse) only if its oracle score lies within 2 eps of the oracle's k-th score:
  i in got \\ want:  want[i] <= kth, and want[i] >= got[i] - eps >= (k-th largest got) - eps >= kth - 2 eps
                    (the k oracle winners all have got >= kth - eps);
  j in want \\ got:  want[j] >= kth, and want[j] <= got[j] + eps <= (k-th largest got) + eps <= kth + 2 eps
                    (some device winner is an oracle loser, so the k-th largest got <= kth + eps).
So once the device's index set is exactly the top-k of the device's own scores under (score desc, index asc) -- the
reference's order (prefill.cpp:240-253), asserted here -- every index difference from the oracle's set is explained
by the measured score error alone (eps, which the callers bound by their rtol and report); the band assertion is the
consistency check of that argument, not a separate tolerance.  Test infrastructure only.
"""
import numpy as np


def top_k_set(scores, k):
    order = np.lexsort((np.arange(len(scores)), -np.asarray(scores, dtype=np.float64)))
    return set(order[:k].tolist())


def error_bounded_ties(got_idx, got_scores, want_scores, k):
    """Returns (n differing indices, eps, band).  Raises AssertionError when the device's set is not the top-k of
    its own scores or when a differing index lies outside the error-derived band."""
    got_scores = np.asarray(got_scores, dtype=np.float64)
    want_scores = np.asarray(want_scores, dtype=np.float64)
    got = set(np.asarray(got_idx).tolist())
    assert got == top_k_set(got_scores, k), "device index set is not the top-k of the device's own scores"
    want = top_k_set(want_scores, k)
    kth = min(want_scores[i] for i in want)
    eps = float(np.max(np.abs(got_scores - want_scores))) if len(got_scores) else 0.0
    band = 2 * eps * (1 + 1e-12) + 1e-300
    diff = got ^ want
    outside = [i for i in diff if abs(want_scores[i] - kth) > band]
    assert not outside, f"{len(outside)} index differences outside the 2-eps band (eps {eps:.3g}, kth {kth:.6g})"
    return len(diff), eps, band
