"""Edge cases of the reference's Dataset contract (src/dataset.cpp:28-56) and of ragged sparse data,
through the C ABI against the oracle: empty / one-column shards are rejected like the reference's
validate(); CSR rows with no nonzeros, rows longer than a warp's index chunk, untouched columns,
duplicate entries (summed, setFromTriplets semantics) and the class-count bounds of the sparse
nonzero-group passes (C - 1 = 32 on them, 33 on the generic path)."""
import numpy as np
import pytest

import oracle
from util import rel

pytestmark = pytest.mark.gpu

TOL = 1e-12


def test_dataset_validation(nadmm):
    with pytest.raises(nadmm.ConfigError):  # n >= 1 (src/dataset.cpp:31-34)
        nadmm.Dataset.dense(np.zeros((0, 3)), np.zeros(0, np.int32), 2)
    with pytest.raises(nadmm.ConfigError):  # p >= 1
        nadmm.Dataset.dense(np.zeros((2, 0)), [1, 2], 2)
    with pytest.raises(nadmm.ConfigError):  # label count == rows
        nadmm.Dataset.dense(np.zeros((3, 2)), [1, 2], 2)
    with pytest.raises(nadmm.DataError):  # non-finite sparse value
        nadmm.Dataset.sparse([0, 1, 2], [0, 1], [1.0, np.inf], [1, 2], 2, 3)
    with pytest.raises(nadmm.DataError):  # label out of range
        nadmm.Dataset.sparse([0, 1, 2], [0, 1], [1.0, 2.0], [1, 3], 2, 3)
    with pytest.raises(nadmm.ConfigError):
        nadmm.Dataset.sparse([0], [], [], np.zeros(0, np.int32), 2, 3)


def ragged_csr(rng, n, p):
    """Row lengths 0, 1, 31, 32, 33, 100, p (full row) and random; the last columns never used."""
    lengths = [0, 1, 31, 32, 33, 100, p, 0, 5]
    lengths += list(rng.integers(0, 60, size=n - len(lengths)))
    used = p - 7  # columns [used, p) stay empty (empty CSC columns)
    indptr, indices, vals = [0], [], []
    for L in lengths:
        L = min(L, used) if L != p else used
        cols = np.sort(rng.choice(used, size=L, replace=False))
        indices.extend(cols.tolist())
        vals.extend(rng.normal(size=L).tolist())
        indptr.append(len(indices))
    return np.array(indptr, np.int64), np.array(indices, np.int32), np.array(vals)


@pytest.mark.parametrize("C", [2, 10, 33, 34])
def test_ragged_sparse_matches_oracle(nadmm, port, C):
    rng = np.random.default_rng(C)
    n, p = 240, 300
    ip, ix, vv = ragged_csr(rng, n, p)
    y = (np.arange(n) % C + 1).astype(np.int32)
    ds = nadmm.Dataset.sparse(ip, ix, vv, y, C, p)
    sh = oracle.Shard(labels=y, C_=C, csr=(ip, ix, vv), p=p)
    w = rng.normal(size=sh.d) * 0.3
    v = rng.normal(size=sh.d)
    lw = port.loss(sh, w, 1e-3)
    assert abs(nadmm.loss(ds, w, 1e-3) - lw) <= TOL * abs(lw)
    assert rel(nadmm.gradient(ds, w, 1e-3), port.gradient(sh, w, 1e-3)) <= TOL
    assert rel(nadmm.hessian_vec(ds, w, v, 1e-3), port.hessian_vec(sh, w, v, 1e-3)) <= TOL
    np.testing.assert_array_equal(nadmm.predict(ds, w), port.predict(sh, w))
    # the empty rows' logits are all zero: their predictions follow the reference tie rule
    assert nadmm.predict(ds, w)[0] == port.predict(sh, w)[0]
    # the empty columns get only the ridge term in the gradient
    g = nadmm.gradient(ds, w, 1e-3).reshape(C - 1, p)
    np.testing.assert_allclose(g[:, -7:], 1e-3 * w.reshape(C - 1, p)[:, -7:], rtol=1e-14, atol=0)


@pytest.mark.parametrize("C", list(range(2, 34)))
def test_sparse_every_class_count(nadmm, port, C):
    """Every class count the CSR lane path takes (K = C - 1 <= 32): both word widths (32-byte words when
    K rounds up to a multiple of 4 without extra padding, else 16-byte), one or two rows per warp, a
    lane group per CSC column; odd n so the last warp's second row is past the end; ragged rows with
    empty rows / columns (kernels_sparse.cu; src/dataset.cpp:69-85, src/softmax.cpp:51-139)."""
    rng = np.random.default_rng(100 + C)
    n, p = 37, 61
    ip, ix, vv = ragged_csr(rng, n, p)
    y = (np.arange(n) % C + 1).astype(np.int32)
    ds = nadmm.Dataset.sparse(ip, ix, vv, y, C, p)
    sh = oracle.Shard(labels=y, C_=C, csr=(ip, ix, vv), p=p)
    w = rng.normal(size=sh.d) * 0.3
    v = rng.normal(size=sh.d)
    lw = port.loss(sh, w, 1e-3)
    assert abs(nadmm.loss(ds, w, 1e-3) - lw) <= TOL * abs(lw)
    assert rel(nadmm.gradient(ds, w, 1e-3), port.gradient(sh, w, 1e-3)) <= TOL
    assert rel(nadmm.hessian_vec(ds, w, v, 1e-3), port.hessian_vec(sh, w, v, 1e-3)) <= TOL
    np.testing.assert_array_equal(nadmm.predict(ds, w), port.predict(sh, w))


def test_duplicate_entries_are_summed(nadmm):
    rng = np.random.default_rng(3)
    n, p, C = 50, 40, 5
    ip, ix, vv = ragged_csr(rng, n, p)
    y = (np.arange(n) % C + 1).astype(np.int32)
    # split every value into two entries of the same column, listed in reverse column order
    ip2, ix2, vv2 = [0], [], []
    for i in range(n):
        cols, vals = ix[ip[i]:ip[i + 1]], vv[ip[i]:ip[i + 1]]
        for c, x in zip(cols[::-1], vals[::-1]):
            ix2 += [c, c]
            vv2 += [0.25 * x, 0.75 * x]
        ip2.append(len(ix2))
    a = nadmm.Dataset.sparse(ip, ix, vv, y, C, p)
    b = nadmm.Dataset.sparse(np.array(ip2, np.int64), np.array(ix2, np.int32), np.array(vv2), y, C, p)
    w = rng.normal(size=(C - 1) * p) * 0.3
    v = rng.normal(size=(C - 1) * p)
    assert rel(nadmm.hessian_vec(b, w, v, 0.0), nadmm.hessian_vec(a, w, v, 0.0)) <= 1e-14
    assert abs(nadmm.loss(b, w, 0.0) - nadmm.loss(a, w, 0.0)) <= 1e-14 * abs(nadmm.loss(a, w, 0.0))


@pytest.mark.parametrize("n,p,C", [(1, 1, 2), (1, 3072, 10), (7, 1, 10), (8, 3072, 10), (9, 784, 10)])
def test_tiny_dense_shapes(nadmm, port, n, p, C):
    """One-row / one-feature shards and shards smaller than one row tile of the fused passes."""
    rng = np.random.default_rng(n * 1000 + p)
    # the suite's conditioning convention (features scaled by 1/sqrt(p), as test_dense_model_ops):
    # unscaled 3,072-feature rows give logits of ~17 and a near one-hot softmax, where Hv's
    # P o a - P (P^T a) cancels and any change of summation order shows at ~1e-11
    X = rng.normal(size=(n, p)) / np.sqrt(p)
    y = (np.arange(n) % C + 1).astype(np.int32)
    ds = nadmm.Dataset.dense(X, y, C)
    sh = oracle.Shard(X, y, C)
    w = rng.normal(size=sh.d)
    v = rng.normal(size=sh.d)
    lw = port.loss(sh, w, 1e-3)
    assert abs(nadmm.loss(ds, w, 1e-3) - lw) <= TOL * abs(lw)
    assert rel(nadmm.gradient(ds, w, 1e-3), port.gradient(sh, w, 1e-3)) <= TOL
    assert rel(nadmm.hessian_vec(ds, w, v, 1e-3), port.hessian_vec(sh, w, v, 1e-3)) <= TOL
    np.testing.assert_array_equal(nadmm.predict(ds, w), port.predict(sh, w))
