"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference's QTT study
(/root/reference/proj/include/latsum/qtt.hpp), the checker for csrc/qtt.cu.

The reference factorises with Eigen's BDCSVD, which this image does not have (so
oracle/_ref cannot build qtt.hpp); numpy's LAPACK SVD stands in for it. Parity for the QTT
row is therefore pinned to this restatement and to the reference's own test laws
(proj/tests/test_qtt.cpp), not to a run of the reference itself.
"""
from __future__ import annotations

import math

import numpy as np


def _keep(sigma: np.ndarray, thresh: float) -> int:
    """qtt.hpp:63-69: smallest r whose discarded tail has Frobenius norm <= thresh, >= 1."""
    keep = len(sigma)
    tail = 0.0
    for i in range(len(sigma) - 1, -1, -1):
        tail += sigma[i] * sigma[i]
        if math.sqrt(tail) > thresh:
            break
        keep = i
    return max(keep, 1)


def qtt_compress(v: np.ndarray, eps: float):
    """qtt.hpp:49-86: returns (cores, per-level singular values)."""
    N = len(v)
    L = int(round(math.log2(N)))
    assert 1 << L == N and N >= 2 and eps > 0
    delta = eps * float(np.linalg.norm(v)) / math.sqrt(max(L - 1, 1))
    carry = np.array(v, dtype=np.float64)
    r_prev, rest = 1, N
    cores, sigmas = [], []
    for _ in range(L - 1):
        M = carry.reshape((2 * r_prev, rest // 2), order="F")  # column-major reinterpretation
        U, s, Vt = np.linalg.svd(M, full_matrices=False)
        keep = _keep(s, delta)
        cores.append(U[:, :keep])
        sigmas.append(s)
        nxt = (s[:keep, None] * Vt[:keep, :])
        rest //= 2
        r_prev = keep
        carry = nxt.reshape(-1, order="F")
    cores.append(carry.reshape((2 * r_prev, 1), order="F"))
    return cores, sigmas


def qtt_reconstruct(cores) -> np.ndarray:
    """qtt.hpp:89-107."""
    w = cores[0]
    for core in cores[1:]:
        r = core.shape[0] // 2
        w = np.vstack([w @ core[:r], w @ core[r:]])
    return w[:, 0]


def unfolding_rank_profile(v: np.ndarray, eps: float) -> list[int]:
    """qtt.hpp:131-152."""
    N = len(v)
    L = int(round(math.log2(N)))
    thresh = eps * float(np.linalg.norm(v))
    out = []
    for k in range(1, L):
        s = np.linalg.svd(np.asarray(v).reshape((1 << k, 1 << (L - k)), order="F"), compute_uv=False)
        out.append(_keep(s, thresh))
    return out
