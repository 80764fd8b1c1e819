"""fp64 oracle of the QKV projection that precedes the team all-gather (Alg. 1
l.1 "AllGather_QKVmatmul").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's step is Q, K, V = (X W_q, X W_k, X W_v) on each rank's shard, gathered over
the team.  With W stored as nn.Linear does ([out, in], y = x W^T) and the three weights
stacked [W_q; W_k; W_v] into one [3E, H] matrix, the projection is one product
Y = X W^T whose column blocks [0, E), [E, 2E), [2E, 3E) are Q, K, V.  The all-gather
only moves these values (pinned by the schedule tests), so the oracle is the product.
Pinned in tests/test_oracle_proj.py by an explicit triple loop on tiny inputs and by the
block structure of the stacked weight.
"""
import numpy as np


def qkv_projection(X, W, heads, head_dim):
    """X fp64 [rows, H], W fp64 [3 heads head_dim, H] -> (Q, K, V) fp64 [rows, heads, head_dim]."""
    E = heads * head_dim
    assert W.shape[0] == 3 * E and W.shape[1] == X.shape[1]
    Y = np.asarray(X, dtype=np.float64) @ np.asarray(W, dtype=np.float64).T
    return tuple(Y[:, i * E:(i + 1) * E].reshape(-1, heads, head_dim) for i in range(3))


def gemm(A, B):
    """Y = A B^T in fp64 (the plain GEMM the projection is made of)."""
    return np.asarray(A, dtype=np.float64) @ np.asarray(B, dtype=np.float64).T
