"""Pins for oracle.algebra against the paper's worked examples and closed forms (§3)."""
import itertools

import numpy as np
import pytest

from oracle import algebra as A
from conftest import golden_matrix


def _as_float(M):
    return np.array([[float(v) for v in row] for row in M])


def test_group_matrix_paper_example_034():
    # fig:adpsgd_preduce
    assert np.array_equal(A.group_matrix(5, [0, 3, 4]), _as_float(golden_matrix("fg_group_034_n5.txt")))


def test_pairwise_matrix_paper_example_03():
    # fig:adpsgd_1pair
    assert np.array_equal(A.pairwise_matrix(5, 0, 3), _as_float(golden_matrix("w_pair_03_n5.txt")))


def test_fused_pair_product_paper_example():
    # fig:adpsgd_2pairs: W_fused = W(0,3) W(4,3)
    Wf = A.pairwise_matrix(5, 0, 3) @ A.pairwise_matrix(5, 4, 3)
    assert np.array_equal(Wf, _as_float(golden_matrix("w_fused_03_43_n5.txt")))
    # and it is NOT an F^G: the relaxation of P:548-556 is a different matrix
    assert not np.allclose(Wf, A.group_matrix(5, [0, 3, 4]))


def test_k2_group_matrix_is_pairwise():
    # "The group in AD-PSGD of size 2 ... becomes a special case"
    for i, j in itertools.combinations(range(6), 2):
        assert np.array_equal(A.group_matrix(6, [i, j]), A.pairwise_matrix(6, i, j))


@pytest.mark.parametrize("n", [1, 2, 5, 8, 16])
def test_doubly_stochastic_and_projection(n):
    rng = np.random.default_rng(n)
    for _ in range(20):
        k = int(rng.integers(1, n + 1))
        G = sorted(rng.choice(n, size=k, replace=False).tolist())
        F = A.group_matrix(n, G)
        assert A.doubly_stochastic_deviation(F) < 1e-12
        assert np.allclose(F.T @ F, F, atol=1e-12, rtol=0)
        assert np.array_equal(F, F.T)
        assert np.all((F >= 0) & (F <= 1))


def test_permutation_is_not_idempotent_negative_control():
    P = np.eye(4)[[1, 0, 2, 3]]
    assert A.doubly_stochastic_deviation(P) == 0
    assert not np.allclose(P.T @ P, P)


def test_special_groups():
    assert np.array_equal(A.group_matrix(4, [2]), np.eye(4))        # singleton = identity
    assert np.allclose(A.group_matrix(4, range(4)), np.full((4, 4), 0.25))  # G = all


def test_apply_mean_of_columns():
    # columns (0), (6), (3) averaged over G = {0,1,2} -> all (3)
    X = np.array([[0.0, 6.0, 3.0]])
    assert np.array_equal(A.apply(X, A.group_matrix(3, [0, 1, 2])), np.array([[3.0, 3.0, 3.0]]))


def test_disjoint_groups_commute_exactly():
    # non-conflicting F^G's can run concurrently
    F1, F2 = A.group_matrix(7, [0, 2, 5]), A.group_matrix(7, [1, 3])
    assert np.array_equal(F1 @ F2, F2 @ F1)
    # overlapping groups do not (conflicts must be serialized)
    F3 = A.group_matrix(7, [2, 3])
    assert not np.allclose(F1 @ F3, F3 @ F1)


def test_errors():
    with pytest.raises(ValueError):
        A.pairwise_matrix(4, 1, 1)
    with pytest.raises(ValueError):
        A.group_matrix(4, [4])
