"""Accuracy of the operator product H.V against an FP64 numpy restatement of
the Matern-3/2 ARD kernel (max error relative to each column's max |H.V|),
for the tensor-core Gram distances (GPK_TGRAM=1) vs the FP32 loops (=0)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402


def dense_h(X, ls, s2, sig2):
    Z = X / ls
    r2 = np.maximum((Z * Z).sum(1)[:, None] + (Z * Z).sum(1)[None, :] - 2 * Z @ Z.T, 0)
    r = np.sqrt(r2)
    K = s2 * (1 + np.sqrt(3) * r) * np.exp(-np.sqrt(3) * r)
    return K + sig2 * np.eye(len(X))


def main():
    ctx = G.Context(0)
    for n, d, m, ell, uniform in [(2048, 26, 65, 1.0, False), (2048, 26, 65, 4.0, False), (2048, 11, 65, 1.0, False),
                                  (2048, 20, 65, 3.0, False), (2048, 8, 17, 1.0, False), (4096, 3, 65, 0.2, True)]:
        rng = np.random.default_rng(n + d)
        X = rng.uniform(-1, 1, (n, d)) if uniform else rng.standard_normal((n, d))
        X = X.astype(np.float32).astype(np.float64)
        ls = np.full(d, ell)
        raw = np.array([G.gpiter.softplus_inverse(v) for v in list(ls) + [1.3, 0.1]])
        op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
        V = np.asfortranarray(rng.standard_normal((n, m)))
        out = op.apply(V)
        ref = dense_h(X, ls, 1.3 ** 2, 0.01) @ V
        err = np.max(np.abs(out - ref) / np.max(np.abs(ref), axis=0))
        print(json.dumps({"tgram": os.environ.get("GPK_TGRAM", "1"), "n": n, "d": d, "m": m, "ell": ell,
                          "max_err_rel_colmax": float(err)}), flush=True)


if __name__ == "__main__":
    main()
