import numpy as np


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / den)


def random_dense(rng, n, p, C, scale=1.0):
    X = rng.normal(size=(n, p)) * scale
    y = (np.arange(n) % C + 1).astype(np.int32)
    rng.shuffle(y)
    return X, y


def random_csr(rng, n, p, C, density=0.3):
    indptr = [0]
    indices, vals = [], []
    for i in range(n):
        cols = np.sort(rng.choice(p, size=max(1, int(density * p)), replace=False))
        indices.extend(cols.tolist())
        vals.extend(rng.normal(size=len(cols)).tolist())
        indptr.append(len(indices))
    y = (np.arange(n) % C + 1).astype(np.int32)
    return np.array(indptr, np.int64), np.array(indices, np.int32), np.array(vals), y
