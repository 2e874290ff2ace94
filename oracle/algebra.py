"""Synchronization matrices in fp64 (TEST INFRASTRUCTURE ONLY; see oracle/__init__).

PAPER.md §3.1-§3.3:
  * X = [x_1 ... x_n] in R^{N x n}; one averaging step is X_{k+1} = X_k W_k
  * pairwise W: W_ii = W_ij = W_ji = W_jj = 1/2, W_uu = 1 otherwise
  * P-Reduce matrix F^G: F_ij = 1/|G| for i, j in G; F_uu = 1 for u not in G
  * doubly stochastic; (F^G)^T F^G = F^G
"""
import numpy as np


def pairwise_matrix(n, i, j):
    """AD-PSGD pairwise synchronization matrix W^k."""
    if i == j or not (0 <= i < n and 0 <= j < n):
        raise ValueError("pairwise_matrix needs two distinct workers in range")
    W = np.eye(n, dtype=np.float64)
    W[i, i] = W[i, j] = W[j, i] = W[j, j] = 0.5
    return W


def group_matrix(n, members):
    """F^G: 1/|G| on the G x G block, identity elsewhere."""
    G = sorted(set(int(m) for m in members))
    if not G or G[0] < 0 or G[-1] >= n:
        raise ValueError("group members out of range")
    F = np.eye(n, dtype=np.float64)
    for i in G:
        for j in G:
            F[i, j] = 1.0 / len(G)
    return F


def apply(X, W):
    """X·W (averaging term only). X is N x n, one column per worker."""
    return np.asarray(X, dtype=np.float64) @ np.asarray(W, dtype=np.float64)


def doubly_stochastic_deviation(W):
    """max |row sum - 1|, |col sum - 1|."""
    W = np.asarray(W, dtype=np.float64)
    return max(np.abs(W.sum(axis=0) - 1).max(), np.abs(W.sum(axis=1) - 1).max())
