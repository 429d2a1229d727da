"""Generate the golden fixtures from the REFERENCE's own code (oracle/_ref: /root/reference/proj
sources built against oracle/eigen_shim). Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

The .npz files are committed so the pins travel to machines without /root/reference."""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import oracle  # noqa: E402

ref = oracle.ref()
assert ref is not None, "oracle/_ref not built"


def model_case(name, n, p, C, lam, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n, p)) * scale
    y = (np.arange(n) % C + 1).astype(np.int32)
    rng.shuffle(y)
    sh = oracle.Shard(X, y, C)
    rd = ref.dataset(sh)
    w, v = rng.normal(size=sh.d) * 0.5, rng.normal(size=sh.d)
    np.savez_compressed(HERE / f"{name}.npz", meta=json.dumps({"kind": "model", "C": C, "lam": lam}), X=X, y=y, w=w,
                        v=v, loss=rd.loss(w, lam), grad=rd.gradient(w, lam), hv=rd.hessian_vec(w, v, lam),
                        pred=rd.predict(w))


def newton_case(name, n, p, C, lam, seed):
    Xtr, ytr, _, _ = ref.generate_synthetic(n, p, C, 3.0, 1.0, seed)
    sh = oracle.Shard(Xtr, ytr, C)
    cfg = [1e-4, 10, 1e-4, 0.5, 10, 1e-8, 5]
    r = ref.dataset(sh).newton_solve(lam, np.zeros(sh.d), cfg=cfg)
    np.savez_compressed(HERE / f"{name}.npz", meta=json.dumps({"kind": "newton", "C": C, "lam": lam, "cfg": cfg}),
                        X=Xtr, y=ytr, x=r["x"], cg_iters=np.array([t["cg_iters"] for t in r["trace"]]))


def synthetic_case(name, args):
    Xtr, ytr, Xte, yte = ref.generate_synthetic(*args)
    np.savez_compressed(HERE / f"{name}.npz", meta=json.dumps({"kind": "synthetic", "args": list(args)}), Xtr=Xtr,
                        yte=yte)


model_case("model_small_c4", 60, 7, 4, 0.0, 1)
model_case("model_mnistlike_c10", 300, 784, 10, 1e-3, 2, scale=1 / 28)
model_case("model_binary_c2", 500, 28, 2, 1e-3, 3)
newton_case("newton_c5", 600, 20, 5, 1e-3, 4)
synthetic_case("synthetic_small", (200, 9, 4, 3.0, 1.0, 0))
print("golden fixtures written to", HERE)
