"""Exact-identity check F = B - (I - P) H on EVERY row, for
PageRank P = dQ (p_ji = d / #out_i): an independent numpy SpMV -- the in-edge sum
of (d/#out_i) H_i per row -- accumulated with np.bincount over column chunks of
about 2^27 edges, so a 1.6e9-edge graph needs a few GB of temporaries.  Test-side
code: shares nothing with oracle/ or the CUDA path."""
import numpy as np


def pagerank_push_sum(n, cp, ri, H, d, chunk_edges=1 << 27):
    """(P H)_j = sum over edges i -> j of (d / #out_i) H_i, and the same sum of |.|."""
    cp = np.asarray(cp, dtype=np.int64)
    deg = np.diff(cp)
    x = np.where(deg > 0, d / np.maximum(deg, 1), 0.0) * H
    acc = np.zeros(n)
    c0 = 0
    while c0 < n:
        c1 = int(np.searchsorted(cp, cp[c0] + chunk_edges, side="right")) - 1
        c1 = min(n, max(c1, c0 + 1))
        e0, e1 = int(cp[c0]), int(cp[c1])
        if e1 > e0:
            acc += np.bincount(ri[e0:e1], weights=np.repeat(x[c0:c1], deg[c0:c1]), minlength=n)
        c0 = c1
    return acc


def identity_residual(n, cp, ri, H, F, b, d):
    """max_j |F_j - (B_j - H_j + (P H)_j)| / (|B_j| + |H_j| + (P H)_j) over all rows
    (H >= 0 for PageRank, so (P H)_j is its own absolute sum), and the row where it
    is largest."""
    acc = pagerank_push_sum(n, cp, ri, H, d)
    err = np.abs(F - (b - H + acc))
    err /= np.abs(b) + np.abs(H) + acc
    j = int(np.argmax(err))
    return float(err[j]), j
