"""Pins of the projection oracle (oracle/proj.py) to definitions outside itself."""
import numpy as np

from oracle.proj import gemm, qkv_projection


def test_gemm_triple_loop():
    rng = np.random.default_rng(1)
    A, B = rng.standard_normal((5, 7)), rng.standard_normal((4, 7))
    Y = gemm(A, B)
    for i in range(5):
        for j in range(4):
            s = 0.0
            for k in range(7):
                s += A[i, k] * B[j, k]
            assert abs(Y[i, j] - s) < 1e-12


def test_qkv_block_structure():
    # W = [I; 2I; 3I] (H = E): Q = X, K = 2X, V = 3X, reshaped [rows, heads, head_dim]
    h, d = 2, 3
    E = h * d
    X = np.arange(4 * E, dtype=np.float64).reshape(4, E)
    W = np.concatenate([np.eye(E), 2 * np.eye(E), 3 * np.eye(E)])
    Q, K, V = qkv_projection(X, W, h, d)
    assert Q.shape == (4, h, d)
    assert np.array_equal(Q.reshape(4, E), X) and np.array_equal(K.reshape(4, E), 2 * X)
    assert np.array_equal(V.reshape(4, E), 3 * X)
    # head j of Q is columns [j d, (j+1) d) of X W_q^T
    assert np.array_equal(Q[:, 1, :], X[:, d:2 * d])


def test_qkv_rows_independent():
    # the projection acts row by row (each rank can project its own shard, Alg. 1 l.1)
    rng = np.random.default_rng(2)
    X, W = rng.standard_normal((6, 8)), rng.standard_normal((12, 8))
    full = qkv_projection(X, W, 2, 2)
    part = qkv_projection(X[3:], W, 2, 2)
    for a, b in zip(full, part):
        assert np.allclose(a[3:], b, atol=0, rtol=0)
